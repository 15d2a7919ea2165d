import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2311_05945_b200 import workloads as WL
from paper_2311_05945_b200.robot.repair import repair_batch
n = int(sys.argv[1])
objs, poses, joints = WL.repair_batch_hand(n, seed=0)
t0 = time.time()
try:
    res = repair_batch(WL.hand_model(), objs, poses, joints)
    print("ok", time.time() - t0, sum(r.cleared for r in res), max(r.penetration_after_m for r in res), sum(r.trial.steps for r in res), flush=True)
except Exception as ex:
    print("ERR", ex, flush=True)
