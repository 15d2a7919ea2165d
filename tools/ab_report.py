"""Summarise tools/ab_libs.sh outputs: python tools/ab_report.py LIB..."""
import glob
import json
import re
import sys

for lib in sys.argv[1:]:
    for f in sorted(glob.glob(f"gpurun_out/ab_{lib}_*.json")):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except (ValueError, IndexError):
            print(f, "no line")
            continue
        st = d.get("step_ms", [])
        print(f"{lib:22s} {d['ms_per_step']:7.3f} ms/step {d['value']:9.0f}/s iters {d['results']['newton_iters_timed']} "
              f"sha {d['results']['state_sha16']} steps {st}")
    try:
        for line in open(f"gpurun_out/abp_{lib}.err"):
            if "timed profile" in line:
                m = re.match(r"\[timed profile\]\s+(\S+)\s+([\d.]+) ms\s+(\d+) launches\s+([\d.]+)", line)
                if m and float(m.group(2)) > 1.0:
                    print(f"    {m.group(1):14s} {m.group(2):>8s} ms {m.group(3):>5s} x {m.group(4):>7s} us")
    except OSError:
        pass
