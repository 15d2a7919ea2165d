"""Phase times of the full config-4 repair (robot.repair.repair_batch).

    python tools/repair_full_breakdown.py [E]
"""
import logging
import os
import sys
import time

logging.disable(logging.WARNING)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2311_05945_b200 import data_path  # noqa: E402
from paper_2311_05945_b200 import workloads as WL  # noqa: E402
from paper_2311_05945_b200.robot import batch as B  # noqa: E402
from paper_2311_05945_b200.robot import parse_urdf  # noqa: E402
from paper_2311_05945_b200.robot import repair as R  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = {}


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        out = fn(*a, **k)
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return out
    return w


R.max_penetration_batch = timed("penetration queries (incl. host sampling arg build)", R.max_penetration_batch)
R.retract_batch = timed("retraction", R.retract_batch)
B.BatchGrasp.__init__ = timed("BatchGrasp build (host scenes + GpuWorld upload)", B.BatchGrasp.__init__)
B.BatchGrasp.run = timed("AutoGrasp dynamics (BatchGrasp.run)", B.BatchGrasp.run)
B.BatchGrasp.sync_scenes = timed("state read-back", B.BatchGrasp.sync_scenes)
objs, poses, joints = WL.repair_batch(E, seed=0)
t0 = time.perf_counter()
res = R.repair_batch(parse_urdf(data_path("pj_gripper.urdf")), objs, poses, joints)
total = time.perf_counter() - t0
for k, v in T.items():
    print(f"{k:55s} {v:8.3f} s")
print(f"{'total':55s} {total:8.3f} s  ({sum(r.trial.steps for r in res)} env-steps)")
