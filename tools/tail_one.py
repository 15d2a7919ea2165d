"""Replay the slowest contact-onset env of config 3 alone for a few steps
(profiling helper; GPU only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_05945_b200 import workloads as WL  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig  # noqa: E402
from paper_2311_05945_b200.world import GpuWorld  # noqa: E402

e, n_env, step = 630, 1024, 3
scenes, grippers, half, poses = WL.grasp_batch(e + 1, seed=0)
sched = WL.schedule(grippers, half, poses, step + 1)
n_links = len(sched[0]) // ((e + 1) * 12)
sub = sched.reshape(step + 1, e + 1, n_links * 12)[:, e].copy()
w = GpuWorld([scenes[e]])
w.upload_schedule(sub.reshape(step + 1, -1))
cfg = SolverConfig()
for k in range(step + 1):
    w.step_scheduled(cfg, k, want_reports=False)
w.sync()
print("done")
