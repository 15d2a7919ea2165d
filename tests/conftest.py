import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))
        return cache[name]

    return load


# Every GPU test runs under the three step schedules of dense worlds: the
# fused per-environment kernel, the batched launch sequence, and the hybrid
# (batched, then per-env CTAs once few envs are still iterating). The native
# library reads IPC_FUSED / IPC_TAIL when a world is created.
SCHEDULES = {"fused": {"IPC_FUSED": "1"}, "batched": {"IPC_FUSED": "0", "IPC_TAIL": "0"},
             "hybrid": {"IPC_FUSED": "0", "IPC_TAIL": "1000000"}}


@pytest.fixture(autouse=True)
def ipc_schedule(request, monkeypatch):
    mode = getattr(request, "param", None)
    if mode is not None:
        for k, v in SCHEDULES[mode].items():
            monkeypatch.setenv(k, v)
    yield mode


def pytest_generate_tests(metafunc):
    if metafunc.definition.get_closest_marker("gpu") and "ipc_schedule" in metafunc.fixturenames:
        metafunc.parametrize("ipc_schedule", list(SCHEDULES), indirect=True)
