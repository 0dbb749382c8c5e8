"""Per-source-line instructions executed and stall samples from an ncu report
(cuda,sass source page).
  python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout.splitlines()
fname, hdr, res = None, None, []
for line in out:
    row = next(csv.reader([line]))
    if row and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        continue
    if hdr and len(row) > 8 and row[0].isdigit():
        try:
            ins = int(row[hdr.index("Instructions Executed")] or 0)
            smp = int(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        res.append((ins, smp, fname, row[0], row[1][:90]))
ti = sum(r[0] for r in res) or 1
ts = sum(r[1] for r in res) or 1
print("warp instructions %d, stall samples %d" % (ti, ts))
for ins, smp, f, l, src in sorted(res, reverse=True)[:top]:
    print("%5.1f%% inst %5.1f%% samples  %s:%s  %s" % (100 * ins / ti, 100 * smp / ts, f, l, src))
