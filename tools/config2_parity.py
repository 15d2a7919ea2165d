"""Config-2 (10,368-tet soft grasp) GPU trajectory vs the reference golden,
per step: Newton / AL counts, PCG iterations, and the worst DoF error split
by block (soft vertices, each affine body). GPU only.

    IPC_PCG_AFF=0|1 IPC_PCG_RTOL=1e-12 python tools/config2_parity.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2311_05945_b200 import data_path  # noqa: E402
from paper_2311_05945_b200.bodies import Material, SoftBody  # noqa: E402
from paper_2311_05945_b200.mesh import box_tet  # noqa: E402
from paper_2311_05945_b200.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose  # noqa: E402
from paper_2311_05945_b200.solver import SolverConfig, engine_of, step  # noqa: E402

CUBE_Y = 0.02515


def main():
    z = dict(np.load(os.path.join(ROOT, "tests", "golden", "traj_soft_grasp_c2.npz")))
    g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
    d = int(z["divisions"])
    obj = SoftBody(box_tet(0.05, d, center=(0.0, CUBE_Y, 0.0)),
                   Material(youngs_modulus=1e5, poisson_ratio=0.3, density=500.0))
    q0 = float(z["q0"])
    sc = build_grasp_scene(obj, g, top_down_pose((0.0, CUBE_Y, 0.0)), [q0, q0], mu=0.5)
    blocks = [(b.body.name or ("soft" if not b.is_affine else "aff"), b.offset, b.dof)
              for b in sc.state.blocks]
    cfg = SolverConfig()
    for k in range(len(z["x"])):
        g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
        st0 = engine_of(sc).stats() if k else None
        t0 = time.perf_counter()
        _, rep = step(sc, cfg)
        wall_ms = 1e3 * (time.perf_counter() - t0)
        st1 = engine_of(sc).stats()
        x = sc.state.gather()
        scale = np.abs(z["x"][k]).max()
        err = {name: float(np.abs(x[o:o + n] - z["x"][k][o:o + n]).max() / scale)
               for name, o, n in blocks}
        out = {"step": k, "wall_ms": wall_ms, "newton": [rep.newton_iters, int(z["newton_iters"][k])],
               "al": [rep.al_outer, int(z["al_outer"][k])],
               "pcg_iters": st1["pcg_iters"] - (st0["pcg_iters"] if st0 else 0),
               "max_rel": max(err.values()), "by_block": err,
               "min_dist": [rep.min_dist_after, float(z["min_dist"][k])]}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
