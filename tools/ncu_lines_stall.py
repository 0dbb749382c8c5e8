"""Per-source-line stall breakdown (one stall reason) from an ncu report.
  python tools/ncu_lines_stall.py report.ncu-rep stall_long_sb [top]"""
import csv
import subprocess
import sys

rep, reason = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
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
            v = int(row[hdr.index(reason)] or 0)
        except (ValueError, IndexError):
            continue
        res.append((v, fname, row[0], row[1][:90]))
tot = sum(r[0] for r in res) or 1
for v, f, l, src in sorted(res, reverse=True)[:top]:
    print("%5.1f%% %s:%s  %s" % (100 * v / tot, f, l, src))
