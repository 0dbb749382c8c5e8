"""Summarise an ncu --set full report of the edge kernel into a small JSON
(profiles/ncu_edge_kernel.json, read by bench.py for roofline.traffic).

  python tools/ncu_summary.py report.ncu-rep config out.json
"""
import csv
import json
import subprocess
import sys

rep, config, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}


def get(name):
    i = h.index(name)
    return float(v[i].replace(",", "")) * scale.get(units[i], 1.0)


want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
d = {"config": config, "report": rep, "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
for w in want:
    try:
        d[w] = get(w)
    except ValueError:
        pass
d["dram_bytes_per_launch"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
d["note"] = ("ncu --set full --clock-control none, one launch (cold L2, serialised): traffic is the per-launch "
             "DRAM bytes; time under the profiler is not a bench value")
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
