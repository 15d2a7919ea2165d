"""Sub-phase SM cycles of the batched dense solve (k_dense_solve) on the
config-3 batch, per env solve (GPU only):
    IPC_FUSED_TIMERS=1 IPC_FUSED=0 IPC_TAIL=0 IPC_LOOP_GRAPH=0 python tools/dense_phases.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_05945_b200 import workloads as WL  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig  # noqa: E402
from paper_2311_05945_b200.world import GpuWorld  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
scenes, grippers, half, poses = WL.grasp_batch(1024, seed=0)
sched = WL.schedule(grippers, half, poses, K)
w = GpuWorld(scenes)
w.upload_schedule(sched)
cfg = SolverConfig()
for k in range(K):
    t0 = w.fused_timers()
    reps = w.step_scheduled(cfg, k)
    t1 = w.fused_timers()
    solves = sum(r.newton_iters for r in reps)
    d = {n: (t1[n] - t0[n]) / max(solves, 1) / 1965.0 for n in t1 if n.startswith("dense_")}
    print(f"step {k}: {solves} env solves, us per env solve (SM cycles at 1965 MHz): "
          + " ".join(f"{n[6:]} {v:.1f}" for n, v in d.items()), flush=True)
