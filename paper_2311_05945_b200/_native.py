"""ctypes binding of libipc_b200.so (C-ABI: include/ipc_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2311_05945_b200.build``). There is no fallback: if the
library or a CUDA device is missing, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.environ.get("IPC_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libipc_b200.so")

_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class WorldDesc(C.Structure):
    _fields_ = (
        [(n, C.c_int32) for n in ("n_env", "n_dof", "n_vert", "n_aff", "n_tet", "n_slot", "n_tri",
                                  "n_edge", "n_cbody", "n_cons")]
        + [(n, _i32p) for n in ("env_dof", "env_vert", "env_aff", "env_tet", "env_slot", "env_tri",
                                "env_edge", "env_cbody", "env_cons")]
        + [("env_pairs", _u8p), ("env_has_ground", _u8p)]
        + [(n, _f64p) for n in ("env_ground_y", "env_gravity", "env_dhat", "env_kappa",
                                "env_kappa0", "env_mu", "env_eps_v")]
        + [("vert_dof", _i32p), ("vert_mass", _f64p), ("aff_dof", _i32p)]
        + [(n, _f64p) for n in ("aff_M", "aff_acc", "aff_ortho")]
        + [("tet_dof", _i32p)]
        + [(n, _f64p) for n in ("tet_Dminv", "tet_vol", "tet_mu", "tet_lam")]
        + [("tet_model", _u8p), ("slot_aff", _u8p), ("slot_dof", _i32p), ("slot_rest", _f64p),
           ("slot_cbody", _i32p), ("tri_v", _i32p), ("tri_cbody", _i32p), ("edge_v", _i32p),
           ("edge_cbody", _i32p), ("edge_len2", _f64p), ("cbody_rigid", _u8p), ("cbody_kin", _u8p),
           ("cbody_excl", _u64p), ("cons_aff", _i32p), ("cons_kappa0", _f64p),
           ("cons_mass", _f64p), ("x0", _f64p), ("v0", _f64p)]
    )


class StepConfig(C.Structure):
    _fields_ = [("h", C.c_double), ("newton_tol", C.c_double), ("max_newton_iters", C.c_int32),
                ("max_line_search_halvings", C.c_int32), ("ccd_conservative_factor", C.c_double),
                ("friction_fixed_point_iters", C.c_int32), ("al_max_outer", C.c_int32)]


class StepReportC(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("ccd_invocations", C.c_int32),
                ("converged", C.c_int32), ("line_search_failed", C.c_int32),
                ("al_outer", C.c_int32), ("error", C.c_int32), ("final_grad_norm", C.c_double),
                ("min_dist_before", C.c_double), ("min_dist_after", C.c_double),
                ("kappa", C.c_double)]


class RepairDesc(C.Structure):
    _fields_ = [("n_env", C.c_int32), ("env_link", _i32p), ("link_vert", _i32p),
                ("link_tri", _i32p), ("hand_v", _f64p), ("hand_t", _i32p),
                ("env_obj_vert", _i32p), ("env_obj_tri", _i32p), ("obj_v", _f64p),
                ("obj_t", _i32p), ("normal", _f64p), ("n_probe", C.c_int32),
                ("retraction", _f64p)]


# symbol -> (restype, argtypes); the authoritative list of C-ABI exports
SIGNATURES = {
    "ipc_last_error": (C.c_char_p, []),
    "ipc_device_count": (C.c_int, []),
    "ipc_world_create": (C.c_int, [C.POINTER(WorldDesc), C.POINTER(C.c_void_p)]),
    "ipc_world_destroy": (C.c_int, [C.c_void_p]),
    "ipc_world_step": (C.c_int, [C.c_void_p, C.POINTER(StepConfig), _f64p,
                                 C.POINTER(StepReportC)]),
    "ipc_world_step_ex": (C.c_int, [C.c_void_p, C.POINTER(StepConfig), _f64p, _u8p,
                                    C.POINTER(StepReportC)]),
    "ipc_world_upload_schedule": (C.c_int, [C.c_void_p, _f64p, C.c_int]),
    "ipc_world_step_scheduled": (C.c_int, [C.c_void_p, C.POINTER(StepConfig), C.c_int, _u8p,
                                           C.POINTER(StepReportC)]),
    "ipc_world_get_state": (C.c_int, [C.c_void_p, _f64p, _f64p]),
    "ipc_world_set_state": (C.c_int, [C.c_void_p, _f64p, _f64p]),
    "ipc_world_state_device": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_void_p)]),
    "ipc_world_get_kappa": (C.c_int, [C.c_void_p, _f64p]),
    "ipc_world_set_kappa": (C.c_int, [C.c_void_p, _f64p]),
    "ipc_world_get_constraints": (C.c_int, [C.c_void_p, _f64p, _f64p]),
    "ipc_world_slot_forces": (C.c_int, [C.c_void_p, C.c_double, _f64p]),
    "ipc_world_candidates": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _i32p, C.c_int64, _i64p]),
    "ipc_world_min_distance": (C.c_int, [C.c_void_p, _f64p]),
    "ipc_world_group_distance": (C.c_int, [C.c_void_p, _u64p, _u64p, _f64p]),
    "ipc_world_ground_distance": (C.c_int, [C.c_void_p, _u64p, _f64p]),
    "ipc_world_group_forces": (C.c_int, [C.c_void_p, C.c_double, _u64p, C.c_int, _f64p]),
    "ipc_set_device": (C.c_int, [C.c_int]),
    "ipc_world_profile": (C.c_int, [C.c_void_p, C.c_int, C.c_uint32]),
    "ipc_world_profile_read": (C.c_int, [C.c_void_p, _f64p, _i64p, _i64p]),
    "ipc_world_stats": (C.c_int, [C.c_void_p, _i64p]),
    "ipc_world_fused_timers": (C.c_int, [C.c_void_p, _i64p, C.c_int]),
    "ipc_world_set_fused": (C.c_int, [C.c_void_p, C.c_int]),
    "ipc_world_set_fused_timers": (C.c_int, [C.c_void_p, C.c_int]),
    "ipc_device_clock_khz": (C.c_int, [_i32p]),
    "ipc_world_run_scheduled": (C.c_int, [C.c_void_p, C.POINTER(StepConfig), C.c_int, C.c_int, C.c_void_p]),
    "ipc_world_flush_l2": (C.c_int, [C.c_void_p, C.c_int64]),
    "ipc_world_mark": (C.c_int, [C.c_void_p, C.c_int]),
    "ipc_world_elapsed": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _f64p]),
    "ipc_world_sync": (C.c_int, [C.c_void_p]),
    "ipc_dist2_derivs": (C.c_int, [C.c_int, C.c_int64, _f64p, _i32p, _f64p, _f64p, _f64p]),
    "ipc_ccd_pairs": (C.c_int, [C.c_int, C.c_int64, _f64p, _f64p, C.c_double, _f64p]),
    "ipc_psd_project": (C.c_int, [C.c_int, C.c_int64, _f64p]),
    "ipc_elastic_eval": (C.c_int, [C.c_int, C.c_int64, _f64p, C.c_double, C.c_double, _f64p,
                                   _f64p, _f64p]),
    "ipc_repair_retract": (C.c_int, [C.POINTER(RepairDesc), _i32p]),
    "ipc_repair_last_kernel_ms": (C.c_int, [_f64p]),
    "ipc_measure_fp64_peak": (C.c_int, [C.c_int, _f64p]),
    "ipc_max_penetration": (C.c_int, [C.c_int32, _i32p, _f64p, _i32p, _i32p, _f64p, _i32p,
                                      _f64p]),
    "ipc_winding_numbers": (C.c_int, [C.c_int64, _f64p, C.c_int32, _f64p, C.c_int32, _i32p,
                                      _f64p]),
    "ipc_count_mesh_intersections": (C.c_int, [C.c_int32, _f64p, C.c_int32, _i32p, C.c_int32,
                                               _f64p, C.c_int32, _i32p, _i64p]),
}

KERNEL_IDS = ("broad_dcd", "broad_ccd", "pairs_deriv", "pairs_value", "tet", "body", "ground",
              "friction", "energy_reduce", "dense_solve", "ccd", "lags", "world_pos", "sensing",
              "misc", "pcg", "assembly", "fused_step")

_lib = None


class NativeError(RuntimeError):
    pass


def load(require_device: bool = True):
    """Load the library (once). Raises when it is missing, or when
    require_device and no CUDA device is visible."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device and _lib.ipc_device_count() == 0:
        raise NativeError("no CUDA device visible: the IPC step has no CPU fallback")
    return _lib


def check(rc: int):
    if rc != 0:
        raise NativeError(_lib.ipc_last_error().decode())


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# kernel-level wrappers (parity tests)
# ---------------------------------------------------------------------------


def dist2_derivs(kind: str, stencils):
    lib = load()
    st = np.ascontiguousarray(stencils, dtype=np.float64).reshape(-1, 12)
    n = len(st)
    reg = np.zeros(n, np.int32)
    s = np.zeros(n)
    g = np.zeros((n, 12))
    h = np.zeros((n, 144))
    check(lib.ipc_dist2_derivs(0 if kind == "pt" else 1, n, ptr(st, _f64p), ptr(reg, _i32p),
                               ptr(s, _f64p), ptr(g, _f64p), ptr(h, _f64p)))
    return reg, s, g, h.reshape(n, 12, 12)


def ccd_pairs(kind: str, px, pdx, conservative=0.9):
    lib = load()
    a = np.ascontiguousarray(px, dtype=np.float64).reshape(-1, 12)
    b = np.ascontiguousarray(pdx, dtype=np.float64).reshape(-1, 12)
    out = np.zeros(len(a))
    check(lib.ipc_ccd_pairs(0 if kind == "pt" else 1, len(a), ptr(a, _f64p), ptr(b, _f64p),
                            conservative, ptr(out, _f64p)))
    return out


def psd_project(mats):
    lib = load()
    m = np.ascontiguousarray(mats, dtype=np.float64).copy()
    dim = m.shape[-1]
    n = m.size // (dim * dim)
    check(lib.ipc_psd_project(dim, n, ptr(m, _f64p)))
    return m


def elastic_eval(model: int, F, mu, lam):
    lib = load()
    f = np.ascontiguousarray(F, dtype=np.float64).reshape(-1, 9)
    n = len(f)
    psi, P, H = np.zeros(n), np.zeros((n, 9)), np.zeros((n, 81))
    check(lib.ipc_elastic_eval(model, n, ptr(f, _f64p), mu, lam, ptr(psi, _f64p), ptr(P, _f64p),
                               ptr(H, _f64p)))
    return psi, P.reshape(n, 3, 3), H.reshape(n, 9, 9)
