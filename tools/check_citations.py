"""List reference citations (`file.py:NNN`) that point past the end of the
cited reference file. Build container only (reads /root/reference)."""
import os
import re
import sys

REF = "/root/reference/pkg/src/srsim"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
files = {}
for d, _, fs in os.walk(REF):
    for f in fs:
        if f.endswith(".py"):
            rel = os.path.relpath(os.path.join(d, f), REF)
            n = sum(1 for _ in open(os.path.join(d, f)))
            files.setdefault(f, []).append((rel, n))
            files.setdefault(rel, []).append((rel, n))
pat = re.compile(r"((?:[\w]+/)*[\w]+\.py):(\d+)(?:[-–](\d+))?")
bad = 0
for d, _, fs in os.walk(ROOT):
    if any(x in d for x in (".git", "gpurun_out", "__pycache__", "build", "exp")):
        continue
    for f in fs:
        if not f.endswith((".py", ".md", ".cu", ".cuh", ".h")) or f in ("check_citations.py",):
            continue
        p = os.path.join(d, f)
        for ln, line in enumerate(open(p, errors="ignore"), 1):
            for m in pat.finditer(line):
                name = m.group(1)
                key = name if name in files else os.path.basename(name)
                if key not in files:
                    continue
                cands = files[key]
                lines = [int(m.group(2))] + ([int(m.group(3))] if m.group(3) else [])
                if all(any(x > n for _, n in cands) for x in lines) or any(
                        all(x > n for _, n in cands) for x in lines):
                    bad += 1
                    print(f"{os.path.relpath(p, ROOT)}:{ln}: {m.group(0)} (ref {cands})")
print(bad, "out-of-range citations", file=sys.stderr)
