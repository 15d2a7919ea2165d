"""Pack scenes into the device world layout and drive the C-ABI engine.

``GpuWorld([scene_0, …, scene_{E-1}])`` uploads E independent scenes as one
batch (one environment each); ``step()`` advances all of them with one call
into ``libipc_b200.so``. The layout is documented in DESIGN.md and
csrc/world.cuh.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .bodies import MODEL_ID, affine_gravity_acceleration


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


class Packed:
    """Flat numpy arrays of a batch (host side of ipc_world_desc)."""

    def __init__(self, scenes):
        self.scenes = list(scenes)
        E = len(self.scenes)
        pre = {k: [0] for k in ("dof", "vert", "aff", "tet", "slot", "tri", "edge", "cbody", "cons")}
        A = {k: [] for k in ("vert_dof", "vert_mass", "aff_dof", "aff_M", "aff_acc", "aff_ortho",
                             "tet_dof", "tet_Dminv", "tet_vol", "tet_mu", "tet_lam", "tet_model",
                             "slot_aff", "slot_dof", "slot_rest", "slot_cbody", "tri_v",
                             "tri_cbody", "edge_v", "edge_cbody", "edge_len2", "cbody_rigid",
                             "cbody_kin", "cbody_excl", "cons_aff", "cons_kappa0", "cons_mass",
                             "x0", "v0")}
        env = {k: [] for k in ("pairs", "has_ground", "ground_y", "gravity", "dhat", "kappa",
                               "kappa0", "mu", "eps_v")}
        self.aff_index = []     # per env: {id(body): global affine index}
        self.cbody_index = []   # per env: {id(body): env-local collision body id}
        for sc in self.scenes:
            st = sc.state
            D = pre["dof"][-1]
            A0 = pre["aff"][-1]
            S0 = pre["slot"][-1]
            CB = pre["cbody"][-1]
            aff_idx, nv, na, nt = {}, 0, 0, 0
            for blk in st.blocks:
                b = blk.body
                if blk.is_affine:
                    aff_idx[id(b)] = A0 + na
                    A["aff_dof"].append([D + blk.offset])
                    A["aff_M"].append(b.M_b.ravel())
                    A["aff_acc"].append(affine_gravity_acceleration(b, sc.gravity))
                    A["aff_ortho"].append([b.stiffness * b.volume])
                    na += 1
                else:
                    if not hasattr(b, "rest_volumes"):
                        raise NotImplementedError("shell bodies are outside the GPU step's scope")
                    n = b.n_verts
                    A["vert_dof"].append(D + blk.offset + 3 * np.arange(n))
                    A["vert_mass"].append(b.mass)
                    nv += n
                    tets = b.mesh.tets.astype(np.int64)
                    A["tet_dof"].append((D + blk.offset + 3 * tets).ravel())
                    A["tet_Dminv"].append(b.dm_inv.reshape(-1))
                    A["tet_vol"].append(b.rest_volumes)
                    mu, lam = b.material.lame
                    A["tet_mu"].append(np.full(len(tets), mu))
                    A["tet_lam"].append(np.full(len(tets), lam))
                    A["tet_model"].append(np.full(len(tets), MODEL_ID[b.material.model]))
                    nt += len(tets)
            ci, tb = sc.cindex, sc.tables
            ns = len(ci.is_affine)
            A["slot_aff"].append(ci.is_affine.astype(np.uint8))
            A["slot_dof"].append(np.where(ci.is_affine, ci.body_offset, ci.soft_dof[:, 0]) + D)
            A["slot_rest"].append(ci.rest.ravel())
            A["slot_cbody"].append(tb.vert_body + CB)
            A["tri_v"].append((tb.tris + S0).ravel())
            A["tri_cbody"].append(tb.tri_body + CB)
            A["edge_v"].append((tb.edges + S0).ravel())
            A["edge_cbody"].append(tb.edge_body + CB)
            A["edge_len2"].append(ci.edge_rest_len2)
            ncb = len(tb.body_is_rigid)
            if ncb > 64:
                raise ValueError("at most 64 bodies per environment")
            A["cbody_rigid"].append(tb.body_is_rigid.astype(np.uint8))
            A["cbody_kin"].append(tb.body_is_kinematic.astype(np.uint8))
            excl = np.zeros(ncb, dtype=np.uint64)
            for a, b in np.asarray(tb.excluded_pairs, dtype=np.int64).reshape(-1, 2):
                excl[a] |= np.uint64(1) << np.uint64(b)
                excl[b] |= np.uint64(1) << np.uint64(a)
            A["cbody_excl"].append(excl)
            ncons = 0
            for c in sc.constraints:
                if not hasattr(c, "target") or not hasattr(c, "mass_scale"):
                    raise NotImplementedError(f"{type(c).__name__} is outside the GPU step's scope")
                A["cons_aff"].append([aff_idx[id(c.body)]])
                A["cons_kappa0"].append([c.kappa0])
                A["cons_mass"].append([c.mass_scale])
                ncons += 1
            A["x0"].append(st.gather())
            A["v0"].append(st.gather_velocity())
            env["pairs"].append(1 if tb.needs_pair_search() else 0)
            env["has_ground"].append(0 if sc.ground_y is None else 1)
            env["ground_y"].append(0.0 if sc.ground_y is None else float(sc.ground_y))
            env["gravity"].append(np.asarray(sc.gravity, dtype=np.float64))
            env["dhat"].append(sc.barrier.dhat)
            env["kappa"].append(sc.barrier.kappa)
            env["kappa0"].append(sc.kappa0)
            env["mu"].append(sc.mu)
            env["eps_v"].append(sc.eps_v)
            self.aff_index.append(aff_idx)
            self.cbody_index.append({id(blk.body): i for i, blk in enumerate(st.blocks)})
            for k, n in (("dof", st.n_dof), ("vert", nv), ("aff", na), ("tet", nt), ("slot", ns),
                         ("tri", len(tb.tris)), ("edge", len(tb.edges)), ("cbody", ncb),
                         ("cons", ncons)):
                pre[k].append(pre[k][-1] + n)

        def cat(parts, conv, width=1):
            if not parts:
                return conv(np.zeros(0))
            return conv(np.concatenate([np.asarray(p).ravel() for p in parts]))

        self.pre = {k: _i32(v) for k, v in pre.items()}
        self.E = E
        conv = {"vert_dof": _i32, "aff_dof": _i32, "tet_dof": _i32, "slot_dof": _i32,
                "slot_cbody": _i32, "tri_v": _i32, "tri_cbody": _i32, "edge_v": _i32,
                "edge_cbody": _i32, "cons_aff": _i32, "tet_model": _u8, "slot_aff": _u8,
                "cbody_rigid": _u8, "cbody_kin": _u8,
                "cbody_excl": lambda a: np.ascontiguousarray(a, dtype=np.uint64)}
        self.arr = {k: cat(v, conv.get(k, _f64)) for k, v in A.items()}
        self.env = {k: (_u8(v) if k in ("pairs", "has_ground") else _f64(np.ravel(v)))
                    for k, v in env.items()}

    def n(self, k):
        return int(self.pre[k][-1])

    def desc(self) -> N.WorldDesc:
        d = N.WorldDesc()
        d.n_env = self.E
        for k in ("dof", "vert", "aff", "tet", "slot", "tri", "edge", "cbody", "cons"):
            setattr(d, "n_" + k, self.n(k))
            setattr(d, "env_" + k, N.ptr(self.pre[k], N._i32p))
        d.env_pairs = N.ptr(self.env["pairs"], N._u8p)
        d.env_has_ground = N.ptr(self.env["has_ground"], N._u8p)
        for k in ("ground_y", "gravity", "dhat", "kappa", "kappa0", "mu", "eps_v"):
            setattr(d, "env_" + k, N.ptr(self.env[k], N._f64p))
        for k, a in self.arr.items():
            t = {np.int32: N._i32p, np.uint8: N._u8p, np.uint64: N._u64p}.get(a.dtype.type, N._f64p)
            setattr(d, k, N.ptr(a, t))
        return d


class GpuWorld:
    """A device-resident batch of scenes."""

    def __init__(self, scenes):
        self.lib = N.load()
        self.packed = Packed(scenes)
        self.scenes = self.packed.scenes
        h = C.c_void_p()
        N.check(self.lib.ipc_world_create(C.byref(self.packed.desc()), C.byref(h)))
        self.handle = h
        self.n_env = self.packed.E
        self.n_dof = self.packed.n("dof")
        self.n_cons = self.packed.n("cons")
        self.n_slot = self.packed.n("slot")
        self._targets = np.zeros(12 * max(self.n_cons, 1))

    def __del__(self):
        try:
            if getattr(self, "handle", None) and self.handle.value:
                self.lib.ipc_world_destroy(self.handle)
                self.handle = C.c_void_p()
        except Exception:
            pass

    # -- state -------------------------------------------------------------
    def get_state(self):
        x, v = np.empty(self.n_dof), np.empty(self.n_dof)
        N.check(self.lib.ipc_world_get_state(self.handle, N.ptr(x, N._f64p), N.ptr(v, N._f64p)))
        return x, v

    def set_state(self, x, v):
        x, v = _f64(x), _f64(v)
        N.check(self.lib.ipc_world_set_state(self.handle, N.ptr(x, N._f64p), N.ptr(v, N._f64p)))

    def get_kappa(self):
        k = np.empty(self.n_env)
        N.check(self.lib.ipc_world_get_kappa(self.handle, N.ptr(k, N._f64p)))
        return k

    def set_kappa(self, k):
        k = _f64(k)
        N.check(self.lib.ipc_world_set_kappa(self.handle, N.ptr(k, N._f64p)))

    def get_constraints(self):
        lam, kap = np.empty(12 * max(self.n_cons, 1)), np.empty(max(self.n_cons, 1))
        N.check(self.lib.ipc_world_get_constraints(self.handle, N.ptr(lam, N._f64p),
                                                    N.ptr(kap, N._f64p)))
        return lam[:12 * self.n_cons].reshape(-1, 12), kap[:self.n_cons]

    def constraint_targets(self):
        """Targets from the scenes' kinematic bodies (ref solver.py:399-400)."""
        out = []
        for sc in self.scenes:
            for c in sc.constraints:
                t = c.body.target_q if c.body.target_q is not None else c.target
                out.append(np.asarray(t, dtype=np.float64))
        return _f64(np.concatenate(out)) if out else self._targets

    # -- stepping ----------------------------------------------------------
    def step(self, cfg, targets=None, want_reports=True, enable=None):
        """Advance every (enabled) env one step. targets: 12 per kinematic
        constraint; None reads the scenes' bodies' target_q."""
        c = N.StepConfig(cfg.h, cfg.newton_tol, cfg.max_newton_iters, cfg.max_line_search_halvings,
                         cfg.ccd_conservative_factor, cfg.friction_fixed_point_iters,
                         cfg.al_max_outer)
        t = self.constraint_targets() if targets is None else _f64(targets)
        reps = (N.StepReportC * self.n_env)() if want_reports else None
        keep = None if enable is None else _u8(enable)
        en = None if keep is None else N.ptr(keep, N._u8p)
        N.check(self.lib.ipc_world_step_ex(self.handle, C.byref(c), N.ptr(t, N._f64p), en, reps))
        return reps

    def upload_schedule(self, targets):
        """Device-resident command stream: (n_steps, 12*n_cons) targets."""
        t = _f64(targets)
        N.check(self.lib.ipc_world_upload_schedule(self.handle, N.ptr(t, N._f64p), len(targets)))

    def step_scheduled(self, cfg, k, want_reports=True, enable=None):
        c = N.StepConfig(cfg.h, cfg.newton_tol, cfg.max_newton_iters, cfg.max_line_search_halvings,
                         cfg.ccd_conservative_factor, cfg.friction_fixed_point_iters,
                         cfg.al_max_outer)
        reps = (N.StepReportC * self.n_env)() if want_reports else None
        keep = None if enable is None else _u8(enable)
        en = None if keep is None else N.ptr(keep, N._u8p)
        N.check(self.lib.ipc_world_step_scheduled(self.handle, C.byref(c), int(k), en, reps))
        return reps

    def run_scheduled(self, cfg, k0, k1, want_reports=True):
        """Steps k0..k1-1 of the uploaded command stream, each env asynchronously
        in its own CTA (ipc_world_run_scheduled); reports of each env's last step."""
        c = N.StepConfig(cfg.h, cfg.newton_tol, cfg.max_newton_iters, cfg.max_line_search_halvings,
                         cfg.ccd_conservative_factor, cfg.friction_fixed_point_iters,
                         cfg.al_max_outer)
        reps = (N.StepReportC * self.n_env)() if want_reports else None
        N.check(self.lib.ipc_world_run_scheduled(self.handle, C.byref(c), int(k0), int(k1), reps))
        return reps

    # -- queries -----------------------------------------------------------
    def candidates(self, env=0, which=0):
        cap = 1 << 22
        buf = np.empty(cap * (1 if which == 2 else 2), dtype=np.int32)
        n = C.c_int64()
        N.check(self.lib.ipc_world_candidates(self.handle, env, which, N.ptr(buf, N._i32p), cap,
                                              C.byref(n)))
        n = n.value
        return buf[:n].astype(np.int64) if which == 2 else buf[:2 * n].reshape(-1, 2).astype(np.int64)

    def min_distance(self):
        out = np.empty(self.n_env)
        N.check(self.lib.ipc_world_min_distance(self.handle, N.ptr(out, N._f64p)))
        return out

    def slot_forces(self, h):
        out = np.empty(3 * self.n_slot)
        N.check(self.lib.ipc_world_slot_forces(self.handle, h, N.ptr(out, N._f64p)))
        return out.reshape(-1, 3)

    def mask(self, env, bodies):
        idx = self.packed.cbody_index[env]
        m = 0
        for b in bodies:
            m |= 1 << idx[id(b)]
        return m

    def group_forces(self, h, groups):
        """groups: (n_env, n_groups) uint64 masks → (n_env, n_groups, 3) N."""
        g = np.ascontiguousarray(groups, dtype=np.uint64)
        ng = g.shape[1]
        out = np.empty(self.n_env * ng * 3)
        N.check(self.lib.ipc_world_group_forces(self.handle, h, N.ptr(g, N._u64p), ng,
                                                N.ptr(out, N._f64p)))
        return out.reshape(self.n_env, ng, 3)

    def group_distance(self, ga, gb):
        a = np.ascontiguousarray(ga, dtype=np.uint64)
        b = np.ascontiguousarray(gb, dtype=np.uint64)
        out = np.empty(self.n_env)
        N.check(self.lib.ipc_world_group_distance(self.handle, N.ptr(a, N._u64p),
                                                  N.ptr(b, N._u64p), N.ptr(out, N._f64p)))
        return out

    def ground_distance(self, g):
        a = np.ascontiguousarray(g, dtype=np.uint64)
        out = np.empty(self.n_env)
        N.check(self.lib.ipc_world_ground_distance(self.handle, N.ptr(a, N._u64p),
                                                   N.ptr(out, N._f64p)))
        return out

    # -- instrumentation (bench.py) -----------------------------------------
    def profile(self, on=True, kernels=None):
        """Per-kernel CUDA-event timing on the world's stream; kernels: names
        from _native.KERNEL_IDS (None = all)."""
        mask = 0xFFFFFFFF if kernels is None else sum(1 << N.KERNEL_IDS.index(k) for k in kernels)
        N.check(self.lib.ipc_world_profile(self.handle, 1 if on else 0, mask))

    def profile_read(self):
        nk = len(N.KERNEL_IDS)
        ms, cnt, launches = np.zeros(nk), np.zeros(nk, np.int64), C.c_int64()
        N.check(self.lib.ipc_world_profile_read(self.handle, N.ptr(ms, N._f64p),
                                                N.ptr(cnt, N._i64p), C.byref(launches)))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(N.KERNEL_IDS)}, launches.value

    def stats(self):
        out = np.zeros(6, np.int64)
        N.check(self.lib.ipc_world_stats(self.handle, N.ptr(out, N._i64p)))
        return {"newton_iters": int(out[0]), "ls_rounds": int(out[1]), "syncs": int(out[2]),
                "pcg_iters": int(out[3]), "fused_env_iters": int(out[4]), "fused_ls_trials": int(out[5])}

    def set_fused(self, on: bool):
        """Fused per-environment step (True) or batched launch sequence with the
        per-env tail hand-off (False, default)."""
        N.check(self.lib.ipc_world_set_fused(self.handle, 1 if on else 0))

    def set_fused_timers(self, on: bool):
        """Per-phase SM-cycle timers of the fused per-env kernels (fused_timers)."""
        N.check(self.lib.ipc_world_set_fused_timers(self.handle, 1 if on else 0))

    def clock_khz(self) -> int:
        out = np.zeros(1, np.int32)
        N.check(self.lib.ipc_device_clock_khz(N.ptr(out, N._i32p)))
        return int(out[0])

    FUSED_PHASES = ("world", "broad_dcd", "terms", "energy", "dense", "ccd_prep", "broad_ccd", "ccd",
                    "line_search", "other",
                    # per-item latency of the terms phase: cycle sum, count, max
                    "pt_cycles", "pt_items", "pt_max", "ee_cycles", "ee_items", "ee_max",
                    "body_cycles", "body_items", "body_max", "fr_cycles", "fr_items", "fr_max",
                    # sub-phases of "dense"
                    "dense_setup", "dense_asm", "dense_gnorm", "dense_ldlt", "dense_subst", "dense_tail",
                    "dense_fwd_warp", "dense_bwd_warp", "dense_diverged")

    def fused_timers(self):
        """SM cycles per phase of the fused step (zeros unless the timers are on)."""
        out = np.zeros(len(self.FUSED_PHASES), np.int64)
        N.check(self.lib.ipc_world_fused_timers(self.handle, N.ptr(out, N._i64p), len(out)))
        return dict(zip(self.FUSED_PHASES, (int(v) for v in out)))

    def flush_l2(self, nbytes=256 << 20):
        N.check(self.lib.ipc_world_flush_l2(self.handle, int(nbytes)))

    def mark(self, slot):
        N.check(self.lib.ipc_world_mark(self.handle, slot))

    def elapsed_ms(self, a, b):
        out = C.c_double()
        N.check(self.lib.ipc_world_elapsed(self.handle, a, b, C.byref(out)))
        return out.value

    def sync(self):
        N.check(self.lib.ipc_world_sync(self.handle))
