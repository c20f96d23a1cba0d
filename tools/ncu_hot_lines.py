"""Top source lines of an ncu report by warp-stall samples.

usage: python tools/ncu_hot_lines.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = "?", None, []
for x in csv.reader(io.StringIO(txt)):
    if len(x) >= 2 and x[0] == "File Name":
        fname = x[1].split("/")[-1]
        continue
    if x and x[0] == "Line No":
        hdr = {k: i for i, k in enumerate(x)}
        continue
    if hdr and x and x[0] not in ("",) and len(x) >= 8:
        ks = [k for k in hdr if k.startswith("Warp Stall Sampling (All")][0]
        ki = [k for k in hdr if k.startswith("Instructions Executed")][0]
        try:
            rows.append((fname, x[0], float(x[hdr[ks]] or 0), float(x[hdr[ki]] or 0), x[1]))
        except ValueError:
            pass
tot = sum(r[2] for r in rows) or 1
toti = sum(r[3] for r in rows) or 1
for f, ln, s, i, src in sorted(rows, key=lambda r: -r[2])[:top]:
    print(f"{f}:{ln:>5} stall {100 * s / tot:5.1f}%  inst {100 * i / toti:5.1f}%  {src.strip()[:90]}")
