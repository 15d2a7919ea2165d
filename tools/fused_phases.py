"""Per-phase SM cycles of the fused per-env step (GPU only; the timers are
on when the world is created with IPC_FUSED_TIMERS=1).

    IPC_FUSED_TIMERS=1 IPC_FUSED=1 python tools/fused_phases.py [env] [steps]

Replays one env of the config-3 batch alone (default env 630 — the
contact-onset env that needs 271 Newton iterations at step 3) and prints
cycles per Newton iteration by phase, then the same for the whole batch.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_05945_b200 import workloads as WL  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig  # noqa: E402
from paper_2311_05945_b200.world import GpuWorld  # noqa: E402


def phases(w, st0, st1, t0, t1, label):
    it = st1["fused_env_iters"] - st0["fused_env_iters"]
    ls = st1["fused_ls_trials"] - st0["fused_ls_trials"]
    d = {k: t1[k] - t0[k] for k in t1}
    items = {}
    for kind in ("pt", "ee", "body", "fr"):
        n = d.pop(f"{kind}_items", 0)
        cyc = d.pop(f"{kind}_cycles", 0)
        d.pop(f"{kind}_max", 0)
        items[kind] = {"per_iter": n / max(it, 1), "mean_us": cyc / max(n, 1) / 1965.0,
                       "max_us_cumulative": t1[f"{kind}_max"] / 1965.0}
    sub = {k: d.pop(k) / max(it, 1) for k in list(d) if k.startswith("dense_")}
    tot = sum(d.values())
    out = {"label": label, "newton_iters": it, "ls_trials": ls,
           "cycles_per_iter": {k: v / max(it, 1) for k, v in d.items()},
           "share": {k: v / max(tot, 1) for k, v in d.items()},
           "us_per_iter_at_1965MHz": tot / max(it, 1) / 1965.0, "items": items,
           "dense_sub_cycles_per_iter": sub}
    print(json.dumps(out), flush=True)


def main():
    e = int(sys.argv[1]) if len(sys.argv) > 1 else 630
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg = SolverConfig()
    n_env = 1024
    scenes, grippers, half, poses = WL.grasp_batch(n_env, seed=0)
    sched = WL.schedule(grippers, half, poses, steps)
    nl = len(sched[0]) // (n_env * 12)
    sub = sched.reshape(steps, n_env, nl * 12)[:, e].copy()
    one = GpuWorld([WL.grasp_batch(n_env, seed=0, select=[e])[0][0]])
    one.set_fused(True)
    one.upload_schedule(sub.reshape(steps, -1))
    for k in range(steps):
        st0, t0 = one.stats(), one.fused_timers()
        r = one.step_scheduled(cfg, k)[0]
        phases(one, st0, one.stats(), t0, one.fused_timers(), f"env {e} step {k} newton {r.newton_iters}")
    w = GpuWorld(scenes)
    w.set_fused(True)
    w.upload_schedule(sched)
    for k in range(steps):
        st0, t0 = w.stats(), w.fused_timers()
        reps = w.step_scheduled(cfg, k)
        it = np.array([r.newton_iters for r in reps])
        phases(w, st0, w.stats(), t0, w.fused_timers(),
               f"batch step {k} newton mean {it.mean():.2f} max {it.max()}")


if __name__ == "__main__":
    main()
