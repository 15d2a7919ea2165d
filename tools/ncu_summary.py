"""Summarise ncu outputs into a markdown file under profiles/.

    python tools/ncu_summary.py LAUNCHES.csv [REPORT.ncu-rep] OUT.md [title]

LAUNCHES.csv: `ncu --metrics gpu__time_duration.sum --csv --log-file` output
(per-launch, cold-cache, serialised: compare shares, not absolutes).
REPORT: an `ncu --set full -o` report; raw metrics of each captured launch.
"""

import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        name = r[ki].split("(")[0].split("<")[0].strip()
        agg[name][0] += 1
        agg[name][1] += v
    return agg


RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for m in RAW:
            d[m] = r[h.index(m)] if m in h else "-"
        res.append(d)
    return res


def main():
    a = sys.argv[1:]
    lpath = a[0]
    rep = a[1] if len(a) > 2 and a[1].endswith(".ncu-rep") else None
    out = a[2] if rep else a[1]
    title = (a[3] if rep and len(a) > 3 else (a[2] if not rep and len(a) > 2 else "ncu summary"))
    agg = launches(lpath)
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {title}", "", f"Launch list: `{lpath}` — {sum(v[0] for v in agg.values())} launches, "
             f"{tot / 1e3:.1f} ms total (ncu serialised, cold cache: read shares, not absolutes).", "",
             "| kernel | launches | total µs | share | µs/launch |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {t:.1f} | {100 * t / tot:.1f}% | {t / n:.2f} |")
    if rep:
        lines += ["", f"Full captures: `{rep}`", "",
                  "| kernel | time (µs) | DRAM read B | DRAM write B | mem % | SM % | fp64 pipe % | warps active % | regs | grid | block |",
                  "|---|---|---|---|---|---|---|---|---|---|---|"]
        for d in raw(rep):
            lines.append("| " + " | ".join([d["kernel"]] + [d[m] for m in RAW]) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
