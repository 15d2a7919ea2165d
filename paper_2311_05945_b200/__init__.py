"""B200-native implicit time step for coupled soft (tet FEM) and affine rigid
bodies under intersection-free, frictional IPC contact.

Drop-in for the reference package's scene/step API (reference ``srsim``):
build scenes with ``bodies`` / ``scene`` / ``robot`` exactly as with the
reference, then ``solver.step(scene, config)`` advances them on the GPU
through the C-ABI library ``libipc_b200.so`` (``include/ipc_b200.h``).
"""

__version__ = "0.1.0"

import os as _os


def data_path(name: str) -> str:
    """Filesystem path of a bundled asset, e.g. data_path('pj_gripper.urdf')."""
    return _os.path.join(_os.path.dirname(__file__), "data", name)
