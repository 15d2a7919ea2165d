"""Sum ncu counters of one kernel over every launch of bench.py's timed
window into profiles/r2_window_<kernel>.json (read by bench.roofline_block).

Capture (on the GPU box, after the same bench command exited 0 without ncu):

    ncu --set full --clock-control none --nvtx --nvtx-include "bench_timed/" \
        -k regex:k_env_newton_rest -o gpurun_out/window \
        python bench.py --no-cpu --window-only --steps 20 --warmup 3

Summarise (here):

    python tools/ncu_window.py gpurun_out/window.ncu-rep fused_step 1024 0 3 20 strong
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
         "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def main():
    rep, kernel, envs, seed, warmup, steps, scaling = sys.argv[1:8]
    if rep.endswith(".csv"):  # raw page exported on the GPU box (the .ncu-rep is too big to bring back)
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]

    def num(r, name):
        i = h.index(name)
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)

    tot = {"dadd": 0.0, "dmul": 0.0, "dfma": 0.0, "dram": 0.0, "t": 0.0, "pipe_t": 0.0, "sm_t": 0.0,
           "warps_t": 0.0}
    n = 0
    regs = None
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        n += 1
        t = num(r, "gpu__time_duration.sum")
        tot["t"] += t
        tot["dadd"] += num(r, "sm__sass_thread_inst_executed_op_dadd_pred_on.sum")
        tot["dmul"] += num(r, "sm__sass_thread_inst_executed_op_dmul_pred_on.sum")
        tot["dfma"] += num(r, "sm__sass_thread_inst_executed_op_dfma_pred_on.sum")
        tot["dram"] += num(r, "dram__bytes_read.sum") + num(r, "dram__bytes_write.sum")
        tot["pipe_t"] += t * num(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        tot["sm_t"] += t * num(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed")
        tot["warps_t"] += t * num(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
        regs = num(r, "launch__registers_per_thread")
    out = {"kernel": kernel, "envs": int(envs), "seed": int(seed), "warmup": int(warmup),
           "steps": int(steps), "scaling": scaling, "launches": n,
           "source": f"ncu --set full --clock-control none --nvtx --nvtx-include bench_timed/ ({rep})",
           "fp64_flops": tot["dadd"] + tot["dmul"] + 2 * tot["dfma"],
           "dadd": tot["dadd"], "dmul": tot["dmul"], "dfma": tot["dfma"], "dram_bytes": tot["dram"],
           "duration_s_under_ncu": tot["t"],
           "fp64_pipe_active_pct": tot["pipe_t"] / tot["t"] if tot["t"] else None,
           "sm_throughput_pct": tot["sm_t"] / tot["t"] if tot["t"] else None,
           "warps_active_pct": tot["warps_t"] / tot["t"] if tot["t"] else None,
           "registers_per_thread": regs}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "profiles", f"r2_window_{kernel}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
