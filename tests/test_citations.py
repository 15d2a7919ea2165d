"""Every `file.py:N` (or `file.py:N-M`) citation of a reference file in the
repo's sources and docs points inside that file. Runs where the reference
checkout exists (this container), skips elsewhere (the GPU box)."""
import glob
import os
import re

import pytest

REF = "/root/reference"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CITE = re.compile(r"((?:[\w.]+/)*\w+\.py):(\d+)(?:-(\d+))?")
SKIP_DIRS = ("gpurun_out", "baseline", ".git", "tests/golden", "profiles")
SKIP_FILES = ("VERDICT.md", "ADVICE.md")


def _ref_lengths():
    out = {}
    for p in glob.glob(os.path.join(REF, "**", "*.py"), recursive=True):
        with open(p, errors="replace") as fh:
            out[os.path.relpath(p, REF)] = sum(1 for _ in fh)
    return out


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference checkout not present")
def test_reference_citations_in_range():
    lens = _ref_lengths()
    bad, n = [], 0
    for p in glob.glob(os.path.join(ROOT, "**", "*"), recursive=True):
        rel = os.path.relpath(p, ROOT)
        if (not os.path.isfile(p) or rel.startswith(SKIP_DIRS) or os.path.basename(p) in SKIP_FILES
                or not p.endswith((".py", ".md", ".cu", ".cuh", ".h", ".c", ".sh"))):
            continue
        with open(p, errors="replace") as fh:
            text = fh.read()
        for m in CITE.finditer(text):
            path = m.group(1)
            cands = [L for r, L in lens.items() if r == path or r.endswith("/" + path)]
            if not cands:
                continue  # not a reference file (a repo file or a third-party one)
            n += 1
            hi = int(m.group(3) or m.group(2))
            if hi > max(cands):
                bad.append(f"{rel}: {m.group(0)} (file has {max(cands)} lines)")
    assert n > 100, n
    assert not bad, "\n".join(bad[:40])
