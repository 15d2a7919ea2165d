"""Isolate the contact-onset tail of config 3: find the envs that need the
most Newton iterations at a given step of the 1024-env batch, then replay the
slowest one alone and print its per-kernel breakdown (GPU only)."""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2311_05945_b200 import workloads as WL  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig  # noqa: E402
from paper_2311_05945_b200.world import GpuWorld  # noqa: E402


def main(n_env=1024, step=3, seed=0):
    cfg = SolverConfig()
    scenes, grippers, half, poses = WL.grasp_batch(n_env, seed=seed)
    sched = WL.schedule(grippers, half, poses, step + 1)
    world = GpuWorld(scenes)
    world.upload_schedule(sched)
    for k in range(step):
        world.step_scheduled(cfg, k, want_reports=False)
    reps = world.step_scheduled(cfg, step)
    it = np.array([r.newton_iters for r in reps])
    order = np.argsort(-it)
    print("slowest envs", [(int(i), int(it[i])) for i in order[:8]], flush=True)
    e = int(order[0])
    # replay env e alone (its scene object is rebuilt from the same stream)
    scenes, grippers, half, poses = WL.grasp_batch(n_env, seed=seed)
    one = GpuWorld([scenes[e]])
    n_links = len(sched[0]) // (n_env * 12)
    sub = sched.reshape(step + 1, n_env, n_links * 12)[:, e].copy()
    one.upload_schedule(sub.reshape(step + 1, -1))
    for k in range(step):
        one.step_scheduled(cfg, k, want_reports=False)
    print("candidates before step: pt %d ee %d ground %d" % (len(one.candidates(0, 0)), len(one.candidates(0, 1)),
                                                           len(one.candidates(0, 2))), flush=True)
    one.profile(True)
    st0 = one.stats()
    one.mark(0)
    t0 = time.perf_counter()
    r = one.step_scheduled(cfg, step)[0]
    one.mark(1)
    dt = time.perf_counter() - t0
    st1 = one.stats()
    prof, launches = one.profile_read()
    d = {k: st1[k] - st0[k] for k in st1}
    print(f"env {e}: dof {scenes[e].state.n_dof}, newton {r.newton_iters}, {1e3 * dt:.1f} ms wall, "
          f"{one.elapsed_ms(0, 1):.1f} ms device, launches {launches}, {d}", flush=True)
    print("candidates after step: pt %d ee %d ground %d" % (len(one.candidates(0, 0)), len(one.candidates(0, 1)),
                                                          len(one.candidates(0, 2))))
    for name, (ms, c) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:14]:
        print(f"  {name:14s} {ms:9.2f} ms {c:6d} launches {1e3 * ms / max(c, 1):9.1f} us/launch")
    ft = one.fused_timers()
    tot = sum(ft.values())
    if tot:
        print("  fused phases (us per Newton iteration at 1.9 GHz):",
              {k: round(v / 1.9e3 / max(r.newton_iters, 1), 1) for k, v in ft.items()})
    per_it = 1e3 * one.elapsed_ms(0, 1) / max(r.newton_iters, 1)
    print(f"  per Newton iteration: {per_it:.0f} us", flush=True)


if __name__ == "__main__":
    main(step=int(sys.argv[1]) if len(sys.argv) > 1 else 3)
