"""Split an ncu source-page CSV (exported on the GPU box) into phases by
line ranges of one source file.
    python tools/ncu_phases.py SRC.csv FILE name:first_line ...  (ranges end at the next start)"""
import collections
import csv
import os
import sys

src, fname = sys.argv[1], sys.argv[2]
marks = sorted((int(a.split(":")[1]), a.split(":")[0]) for a in sys.argv[3:])
rows = list(csv.reader(open(src)))
path, col, coli = None, None, None
st, ins = collections.Counter(), collections.Counter()


def fl(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        col = r.index("Warp Stall Sampling (All Samples)")
        coli = r.index("Instructions Executed")
        continue
    if col is None or len(r) <= col or not r[0].isdigit():
        continue
    ln = int(r[0])
    name = "other files" if path != fname else "before"
    if path == fname:
        for m, nm in marks:
            if ln >= m:
                name = nm
    st[name] += fl(r[col])
    ins[name] += fl(r[coli])
ts, ti = sum(st.values()) or 1, sum(ins.values()) or 1
for k, v in st.most_common():
    print(f"{100 * v / ts:5.1f}% stalls {100 * ins[k] / ti:5.1f}% instr  {k}")
