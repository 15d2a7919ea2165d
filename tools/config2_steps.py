import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2311_05945_b200 import workloads as WL
from paper_2311_05945_b200.solver import SolverConfig, engine_of, step
sc, g, cube = WL.soft_grasp(12)
cfg = SolverConfig()
for k in range(30):
    g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
    w = engine_of(sc)
    st0 = w.stats() if w else None
    t0 = time.perf_counter()
    _, rep = step(sc, cfg)
    dt = time.perf_counter() - t0
    st1 = engine_of(sc).stats()
    d = {kk: st1[kk] - st0[kk] for kk in st1} if st0 else {}
    print(k, f"{dt*1e3:.1f} ms newton {rep.newton_iters} al {rep.al_outer}", d.get("pcg_iters"), d.get("ls_rounds"), flush=True)
