"""Cross-check of the CPU baseline: the reference's own step (srsim, jax
mapped onto torch.func by tests/golden/_jaxshim) against the oracle port on
the same 40-step rigid pinch (mu = 0.5, the golden traj_pinch_steps run),
one core each, build container only:

    python tools/ref_vs_port_timing.py [steps]

Prints per-step wall ms of both and checks the port's states against the
reference's (same Newton counts, DoFs within 1e-8)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "tests", "golden", "_jaxshim"), "/root/reference/pkg/src"):
    sys.path.insert(0, p)

import srsim.bodies as RB  # noqa: E402
import srsim.geometry.mesh as RM  # noqa: E402
import srsim.robot as RR  # noqa: E402
from srsim.data import data_path as rdata  # noqa: E402
from srsim.solver import SolverConfig as RCfg, step as rstep  # noqa: E402

from oracle import stepper as S  # noqa: E402
from paper_2311_05945_b200 import data_path  # noqa: E402
from paper_2311_05945_b200.bodies import AffineBody  # noqa: E402
from paper_2311_05945_b200.mesh import box_surface  # noqa: E402
from paper_2311_05945_b200.robot import Gripper, build_grasp_scene, parse_urdf, top_down_pose  # noqa: E402

CY = 0.02515
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40

rg = RR.Gripper(RR.parse_urdf(rdata("pj_gripper.urdf")))
ro = RB.AffineBody(RM.box_surface(0.05, center=(0.0, CY, 0.0)), density=500.0)
rsc = RR.build_grasp_scene(ro, rg, RR.top_down_pose((0.0, CY, 0.0)), [0.0, 0.0], mu=0.5)
g = Gripper(parse_urdf(data_path("pj_gripper.urdf")))
o = AffineBody(box_surface(0.05, center=(0.0, CY, 0.0)), density=500.0)
sc = build_grasp_scene(o, g, top_down_pose((0.0, CY, 0.0)), [0.0, 0.0], mu=0.5)
lay = S.Layout(sc)

t_ref, t_port, worst, same = 0.0, 0.0, 0.0, True
for k in range(n):
    rg.set_targets(joint_values=np.minimum(rg.joint_values + 1e-3, 0.0262))
    g.set_targets(joint_values=np.minimum(g.joint_values + 1e-3, 0.0262))
    t0 = time.perf_counter()
    _, rr = rstep(rsc, RCfg())
    t1 = time.perf_counter()
    pr = S.step(sc, S.Config(), lay)
    t2 = time.perf_counter()
    t_ref += t1 - t0
    t_port += t2 - t1
    xr, xp = rsc.state.gather(), sc.state.gather()
    worst = max(worst, float(np.abs(xr - xp).max() / np.abs(xr).max()))
    same &= rr.newton_iters == pr.newton_iters
out = {"scene": f"rigid pinch, mu 0.5, {n} steps, one core",
       "reference_ms_per_step": 1e3 * t_ref / n, "port_ms_per_step": 1e3 * t_port / n,
       "reference_over_port": t_ref / t_port, "same_newton_counts": bool(same), "max_rel_dof": worst,
       "note": "reference = srsim with jax replaced by torch.func (tests/golden/_jaxshim); the "
               "port = oracle/ (numpy/scipy); the bench's CPU arms time the port"}
print(json.dumps(out, indent=1))
