"""Where the config-4 e2e time goes: host packing vs the C-ABI call
(allocation, H2D, kernel, D2H) vs the kernel alone.

    python tools/repair_e2e_breakdown.py [E]
"""
import logging
import os
import sys
import time

import numpy as np

logging.disable(logging.WARNING)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import _repair_inputs  # noqa: E402
from paper_2311_05945_b200 import _native as N  # noqa: E402
from paper_2311_05945_b200.robot import repair as R  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
model, objs, poses, joints, grippers, opened, meshes = _repair_inputs(E, 0)
lib = N.load()
real = lib.ipc_repair_retract
t_call = []


class Timed:
    def __getattr__(self, k):
        return getattr(lib, k)

    def ipc_repair_retract(self, d, idx):
        t0 = time.perf_counter()
        rc = real(d, idx)
        t_call.append(time.perf_counter() - t0)
        return rc


N.load = lambda *a, **k: Timed()
for _ in range(3):
    R.retract_batch(grippers, poses, opened, meshes)
t_call.clear()
tot, kms = [], []
ms = np.zeros(1)
for _ in range(10):
    t0 = time.perf_counter()
    R.retract_batch(grippers, poses, opened, meshes)
    tot.append(time.perf_counter() - t0)
    lib.ipc_repair_last_kernel_ms(N.ptr(ms, N._f64p))
    kms.append(ms[0])
print(f"E={E} total {1e3 * np.median(tot):.2f} ms | C-ABI call {1e3 * np.median(t_call):.2f} ms | "
      f"kernel {np.median(kms):.3f} ms | host packing {1e3 * (np.median(tot) - np.median(t_call)):.2f} ms")
