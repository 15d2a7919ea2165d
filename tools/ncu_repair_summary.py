"""Summarise an ncu --set full capture of k_repair_retract into the JSON
bench.py reads for the config-4 roofline (profiles/r1e_repair_ncu.json).

    python tools/ncu_repair_summary.py gpurun_out/repair_retract.ncu-rep ENVS SEED OUT.json [HAND]

REPORT may also be the raw-page CSV exported on the GPU box (`ncu -i … --page raw --csv`).
"""
import csv
import io
import json
import subprocess
import sys

rep, envs, seed, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
hand = sys.argv[5] if len(sys.argv) > 5 else "pj"
if rep.endswith(".csv"):
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
m = {n: (u, x) for n, u, x in zip(h, units, v)}


def num(name, scale_units=True):
    u, x = m[name]
    x = float(x.replace(",", ""))
    if scale_units:
        x *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u, 1.0)
    return x


dadd = num("sm__sass_thread_inst_executed_op_dadd_pred_on.sum")
dmul = num("sm__sass_thread_inst_executed_op_dmul_pred_on.sum")
dfma = num("sm__sass_thread_inst_executed_op_dfma_pred_on.sum")
summary = {
    "kernel": "k_repair_retract", "envs": envs, "seed": seed, "hand": hand,
    "source": f"ncu --set full --clock-control none, one launch ({rep})",
    "duration_s_under_ncu": num("gpu__time_duration.sum"),
    "fp64_flops": dadd + dmul + 2 * dfma, "dadd": dadd, "dmul": dmul, "dfma": dfma,
    "dram_bytes_read": num("dram__bytes_read.sum"), "dram_bytes_write": num("dram__bytes_write.sum"),
    "fp64_pipe_active_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "threads_per_inst": num("smsp__thread_inst_executed_per_inst_executed.ratio"),
    "registers_per_thread": num("launch__registers_per_thread"),
}
with open(out, "w") as fh:
    json.dump(summary, fh, indent=1)
print(json.dumps(summary, indent=1))
