"""Print the main sections of an ncu report's details page (speed of light, scheduler,
warp state, launch, occupancy).   python tools/ncu_details.py report.ncu-rep"""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
si, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
keep = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
        "Scheduler Statistics", "Warp State Statistics", "Launch Statistics", "Occupancy")
for x in rows[1:]:
    if len(x) > vi and x[si] in keep:
        print("%-32s %-52s %-12s %s" % (x[si], x[mi], x[ui], x[vi]))
