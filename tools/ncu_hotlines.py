"""Top source lines by warp-stall samples for one kernel of an ncu report.
    python tools/ncu_hotlines.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, agg, src = None, collections.Counter(), {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No" or r[0] == "":
        continue
    key = (cur_file, int(r[0]))
    src[key] = r[1]
    try:
        agg[key] += int(r[4])
    except ValueError:
        pass
tot = sum(agg.values()) or 1
for k, v in agg.most_common(n):
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]}  {src[k][:110]}")
