"""Top CUDA source lines of an ncu report by warp stall samples (needs a
capture with --import-source on and a -lineinfo build).

    python tools/ncu_hot.py REPORT.ncu-rep [N]
"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
if rep.endswith(".csv"):  # source page exported on the GPU box
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
items, path, col = [], "", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        col = r.index("Warp Stall Sampling (All Samples)")
        continue
    if col is None or len(r) <= col or not r[0]:
        continue
    try:
        v = float(r[col] or 0)
    except ValueError:
        continue
    if v > 0:
        items.append((v, f"{path}:{r[0]}", r[1].strip()[:100]))
tot = sum(v for v, _, _ in items) or 1.0
for v, where, src in sorted(items, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {where:<18} {src}")
