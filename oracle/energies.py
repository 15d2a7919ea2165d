"""Oracle: energy terms of the incremental potential with gradients and
PSD-projected Hessians. TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every term returns a ``Term``: scalar value plus gradient entries and COO
Hessian triplets in global DoF coordinates (duplicates accumulate), which
is what ref pkg/src/srsim/energy/term.py:12 carries.
"""

from __future__ import annotations

import numpy as np

from . import distance as D

EE_MOLLIFIER_SCALE = 1e-6  # ref contact.py:279


class Term:
    __slots__ = ("value", "gi", "gv", "hr", "hc", "hv")

    def __init__(self, value=0.0, gi=None, gv=None, hr=None, hc=None, hv=None):
        z = np.empty(0, dtype=np.int64)
        self.value = float(value)
        self.gi = z if gi is None else gi
        self.gv = np.empty(0) if gv is None else gv
        self.hr = z if hr is None else hr
        self.hc = z if hc is None else hc
        self.hv = np.empty(0) if hv is None else hv

    @staticmethod
    def dense(value, idx, g, h):
        """Batch of dense local blocks: idx (n,k), g (n,k), h (n,k,k)."""
        n, k = idx.shape
        t = Term(value, idx.ravel(), g.ravel())
        if h is not None:
            t.hr = np.repeat(idx, k, axis=1).ravel()
            t.hc = np.tile(idx, (1, k)).ravel()
            t.hv = h.reshape(n, k * k).ravel()
        return t

    def scaled(self, c):
        return Term(c * self.value, self.gi, c * self.gv, self.hr, self.hc, c * self.hv)


def merge(value, terms):
    out = Term(value)
    if terms:
        out.gi = np.concatenate([t.gi for t in terms])
        out.gv = np.concatenate([t.gv for t in terms])
        out.hr = np.concatenate([t.hr for t in terms])
        out.hc = np.concatenate([t.hc for t in terms])
        out.hv = np.concatenate([t.hv for t in terms])
    return out


def psd(h):
    """Clamp negative eigenvalues of symmetric blocks (ref spd.py:6)."""
    h = 0.5 * (h + np.swapaxes(h, -1, -2))
    w, v = np.linalg.eigh(h)
    return (v * np.maximum(w, 0.0)[..., None, :]) @ np.swapaxes(v, -1, -2)


# ---------------------------------------------------------------------------
# barrier on squared distance (ref barrier.py:51)
# ---------------------------------------------------------------------------


def barrier_sq(s, shat, order=2):
    s = np.asarray(s, dtype=np.float64)
    if np.any(s <= 0):
        raise ValueError("barrier evaluated at non-positive squared distance")
    b, db, d2b = np.zeros_like(s), np.zeros_like(s), np.zeros_like(s)
    m = s < shat
    sm = s[m]
    g = sm - shat
    ln = np.log(sm / shat)
    b[m] = -g * g * ln
    db[m] = -2.0 * g * ln - g * g / sm
    d2b[m] = -2.0 * ln - 4.0 * g / sm + g * g / (sm * sm)
    return (b, db, d2b)[: order + 1] if order else b


# ---------------------------------------------------------------------------
# inertia, orthogonality, kinematic targets (ref terms.py, constraints.py)
# ---------------------------------------------------------------------------


def inertia(x, xhat, layout, derivatives=True):
    """½ (x − x̂)ᵀ M (x − x̂) (ref terms.py:12)."""
    d = x - xhat
    val = 0.0
    parts = []
    for off, dof, mass in layout.mass_blocks:
        seg = d[off:off + dof]
        if mass.ndim == 2:
            g = mass @ seg
            val += 0.5 * seg @ g
            if derivatives:
                parts.append(Term.dense(0.0, np.arange(off, off + 12)[None], g[None], mass[None]))
        else:
            m3 = np.repeat(mass, 3)
            g = m3 * seg
            val += 0.5 * seg @ g
            if derivatives:
                idx = np.arange(off, off + dof)
                parts.append(Term(0.0, idx, g, idx, idx, m3))
    return merge(val, parts) if derivatives else Term(val)


def orthogonality(x, layout, derivatives=True):
    """Σ λ V ‖A Aᵀ − I‖²_F with the 9x9 Hessian projected (ref terms.py:55)."""
    val = 0.0
    idx, gs, hs = [], [], []
    for off, coeff in layout.ortho:
        a = x[off + 3:off + 12].reshape(3, 3)
        m = a @ a.T - np.eye(3)
        val += coeff * np.sum(m * m)
        if not derivatives:
            continue
        ata = a.T @ a
        e = np.eye(3)
        h = 4.0 * coeff * (np.einsum("ik,lj->ijkl", e, ata) + np.einsum("il,kj->ijkl", a, a)
                           + np.einsum("ik,jl->ijkl", m, e))
        idx.append(np.arange(off + 3, off + 12))
        gs.append((4.0 * coeff * (m @ a)).ravel())
        hs.append(psd(h.reshape(9, 9)))
    if not derivatives or not idx:
        return Term(val)
    return Term.dense(val, np.stack(idx), np.stack(gs), np.stack(hs))


def kinematic(c, q, off):
    """(κ/2)‖q − q̃‖² − √m λ·(q − q̃) (ref constraints.py:55)."""
    d = q - c.target
    sm = np.sqrt(c.mass_scale)
    val = 0.5 * c.kappa * (d @ d) - sm * (c.lam @ d)
    g = c.kappa * d - sm * c.lam
    return Term.dense(val, (off + np.arange(12))[None], g[None], (c.kappa * np.eye(12))[None])


# ---------------------------------------------------------------------------
# hyperelastic tets (ref elastic.py)
# ---------------------------------------------------------------------------

_LC = np.zeros((3, 3, 3))
for _i, _j, _k in ((0, 1, 2), (1, 2, 0), (2, 0, 1)):
    _LC[_i, _j, _k], _LC[_i, _k, _j] = 1.0, -1.0


def deformation_gradients(xb, tets, dm_inv):
    ds = np.transpose(xb[tets[:, 1:]] - xb[tets[:, :1]], (0, 2, 1))
    return ds @ dm_inv


def _polar(f):
    u, sig, vt = np.linalg.svd(f)
    flip = np.linalg.det(u @ vt) < 0
    u, sig = u.copy(), sig.copy()
    u[flip, :, 2] *= -1.0
    sig[flip, 2] *= -1.0
    r = u @ vt
    s = np.einsum("nji,nj,njk->nik", vt, sig, vt)
    return r, s


def _cofactor(f):
    return np.stack([np.cross(f[:, :, 1], f[:, :, 2]), np.cross(f[:, :, 2], f[:, :, 0]),
                     np.cross(f[:, :, 0], f[:, :, 1])], axis=2)


def _drot(r, s):
    """∂R/∂F of the polar rotation (ref elastic.py:129), (n, 9, 9)."""
    n = len(r)
    m = np.trace(s, axis1=1, axis2=2)[:, None, None] * np.eye(3) - s
    out = np.empty((n, 3, 3, 3, 3))
    for k in range(3):
        for l in range(3):
            a = np.zeros((n, 3, 3))
            a[:, :, l] = r[:, k, :]
            rhs = np.stack([a[:, 2, 1] - a[:, 1, 2], a[:, 0, 2] - a[:, 2, 0],
                            a[:, 1, 0] - a[:, 0, 1]], axis=1)
            w = np.linalg.solve(m, rhs[..., None])[..., 0]
            out[:, :, :, k, l] = r @ D._skew(w)
    return out.reshape(n, 9, 9)


def elastic_psi(f, model, mu, lam):
    """Energy density; None when NeoHookean sees det F ≤ 0 (ref elastic.py:173)."""
    if model == "NeoHookean":
        j = np.linalg.det(f)
        if np.any(j <= 0):
            return None
        lj = np.log(j)
        return 0.5 * mu * (np.einsum("nij,nij->n", f, f) - 3.0) - mu * lj + 0.5 * lam * lj * lj
    if model == "StVK":
        e = 0.5 * (np.einsum("nji,njk->nik", f, f) - np.eye(3))
        tr = np.trace(e, axis1=1, axis2=2)
        return mu * np.einsum("nij,nij->n", e, e) + 0.5 * lam * tr * tr
    if model == "FixedCorotated":
        r, _ = _polar(f)
        j = np.linalg.det(f)
        d = f - r
        return mu * np.einsum("nij,nij->n", d, d) + 0.5 * lam * (j - 1.0) ** 2
    raise ValueError(f"unknown elastic model {model!r}")


def elastic_pk1_hess(f, model, mu, lam):
    """(ψ, P, 9x9 ∂²ψ/∂F²) per tet (ref elastic.py:79-167)."""
    e3 = np.eye(3)
    if model == "NeoHookean":
        j = np.linalg.det(f)
        if np.any(j <= 0):
            raise FloatingPointError("NeoHookean derivatives at inverted tet")
        psi = elastic_psi(f, model, mu, lam)
        lj = np.log(j)
        bt = np.transpose(np.linalg.inv(f), (0, 2, 1))
        p = mu * f + (lam * lj - mu)[:, None, None] * bt
        h = (mu * np.einsum("ik,jl->ijkl", e3, e3)[None]
             + (mu - lam * lj)[:, None, None, None, None] * np.einsum("nil,nkj->nijkl", bt, bt)
             + lam * np.einsum("nij,nkl->nijkl", bt, bt))
    elif model == "StVK":
        psi = elastic_psi(f, model, mu, lam)
        e = 0.5 * (np.einsum("nji,njk->nik", f, f) - e3)
        tr = np.trace(e, axis1=1, axis2=2)
        s2 = 2.0 * mu * e + lam * tr[:, None, None] * e3
        p = f @ s2
        fft = np.einsum("nij,nkj->nik", f, f)
        h = (np.einsum("ik,nlj->nijkl", e3, s2) + mu * np.einsum("nil,nkj->nijkl", f, f)
             + mu * np.einsum("jl,nik->nijkl", e3, fft) + lam * np.einsum("nij,nkl->nijkl", f, f))
    elif model == "FixedCorotated":
        r, s = _polar(f)
        j = np.linalg.det(f)
        psi = elastic_psi(f, model, mu, lam)
        g = _cofactor(f)
        p = 2.0 * mu * (f - r) + lam * (j - 1.0)[:, None, None] * g
        gv = g.reshape(-1, 9)
        dcof = np.einsum("ikm,jlq,bmq->bijkl", _LC, _LC, f).reshape(-1, 9, 9)
        h = (2.0 * mu * (np.eye(9)[None] - _drot(r, s)) + lam * gv[:, :, None] * gv[:, None, :]
             + lam * (j - 1.0)[:, None, None] * dcof)
    else:
        raise ValueError(f"unknown elastic model {model!r}")
    return psi, p, h.reshape(-1, 9, 9)


def _stencil(dm_inv):
    c = np.empty((len(dm_inv), 4, 3))
    c[:, 1:] = dm_inv
    c[:, 0] = -dm_inv.sum(axis=1)
    return c


def elastic(body, xb, off, derivatives=True):
    """Σ V ψ(F) over the body's tets; ∞ when NeoHookean inverts
    (ref elastic.py:185, :204)."""
    mu, lam = body.material.lame
    f = deformation_gradients(xb, body.mesh.tets, body.dm_inv)
    vol = body.rest_volumes
    if not derivatives:
        psi = elastic_psi(f, body.material.model, mu, lam)
        return Term(np.inf if psi is None else float(psi @ vol))
    psi, p, h9 = elastic_pk1_hess(f, body.material.model, mu, lam)
    c = _stencil(body.dm_inv)
    g = np.einsum("n,nij,nvj->nvi", vol, p, c).reshape(-1, 12)
    h4 = psd(h9).reshape(-1, 3, 3, 3, 3)
    h = np.einsum("n,nvj,nljmk,nwk->nvlwm", vol, c, h4, c).reshape(-1, 12, 12)
    idx = (off + 3 * body.mesh.tets[:, :, None].astype(np.int64) + np.arange(3)).reshape(-1, 12)
    return Term.dense(float(psi @ vol), idx, g, h)


# ---------------------------------------------------------------------------
# lifting slot-space stencils to DoF space (ref contact.py:346)
# ---------------------------------------------------------------------------


def lift(slots, g, h, cidx):
    """slots (m, ns), g (m, 3ns), h (m, 3ns, 3ns) → Terms in DoF space.

    Affine slots carry x = J(x0) q, so their rows/columns expand through
    J = [I | x0ᵀ⊗I]; soft slots keep their own three DoF. Grouped by the
    slot-kind signature so each group is a uniform dense batch.
    """
    m, ns = slots.shape
    if m == 0:
        return []
    kinds = cidx.is_affine[slots]
    sig = kinds.astype(np.int64) @ (1 << np.arange(ns))
    out = []
    for key in np.unique(sig):
        rows = np.nonzero(sig == key)[0]
        kin = kinds[rows[0]]
        width = np.where(kin, 12, 3)
        start = np.concatenate([[0], np.cumsum(width)])
        k = int(start[-1])
        r = len(rows)
        jac = np.zeros((r, 3 * ns, k))
        idx = np.empty((r, k), dtype=np.int64)
        for i in range(ns):
            sl = slots[rows, i]
            a = start[i]
            blk = slice(3 * i, 3 * i + 3)
            jac[:, blk, a:a + 3] = np.eye(3)
            if kin[i]:
                x0 = cidx.rest[sl]
                for c in range(3):
                    jac[:, 3 * i + c, a + 3 + 3 * c:a + 6 + 3 * c] = x0
                idx[:, a:a + 12] = cidx.body_offset[sl][:, None] + np.arange(12)
            else:
                idx[:, a:a + 3] = cidx.soft_dof[sl]
        gl = np.einsum("mak,ma->mk", jac, g[rows])
        hl = np.einsum("mak,mab,mbl->mkl", jac, h[rows], jac)
        out.append(Term.dense(0.0, idx, gl, hl))
    return out


# ---------------------------------------------------------------------------
# contact barrier (ref contact.py:216)
# ---------------------------------------------------------------------------

_EDGE_MAP = np.array([[-1.0, 1.0, 0.0, 0.0], [0.0, 0.0, -1.0, 1.0]])  # (u, v) from stencil


def _cross2(u, v, derivatives):
    uu, vv, uv = D._dot(u, u), D._dot(v, v), D._dot(u, v)
    c = uu * vv - uv * uv
    if not derivatives:
        return c
    e3 = np.eye(3)
    gu = 2.0 * (vv[:, None] * u - uv[:, None] * v)
    gv = 2.0 * (uu[:, None] * v - uv[:, None] * u)
    huu = 2.0 * vv[:, None, None] * e3 - 2.0 * D._outer(v, v)
    hvv = 2.0 * uu[:, None, None] * e3 - 2.0 * D._outer(u, u)
    huv = 4.0 * D._outer(u, v) - 2.0 * D._outer(v, u) - 2.0 * uv[:, None, None] * e3
    gw = [gu, gv]
    hw = [[huu, huv], [np.transpose(huv, (0, 2, 1)), hvv]]
    g, h = D._to_vertices(gw, hw, _EDGE_MAP)
    return c, g.reshape(-1, 12), h.reshape(-1, 12, 12)


def _mollifier(c, eps):
    t = c / eps
    lo = t < 1.0
    return (np.where(lo, t * (2.0 - t), 1.0), np.where(lo, (2.0 - 2.0 * t) / eps, 0.0),
            np.where(lo, -2.0 / (eps * eps), 0.0))


def pt_stencils(xw, cand, tables):
    tri = tables.tris[cand.pt[:, 1]]
    slots = np.stack([cand.pt[:, 0], tri[:, 0], tri[:, 1], tri[:, 2]], axis=1)
    return slots, xw[slots]


def ee_stencils(xw, cand, tables):
    ea, eb = tables.edges[cand.ee[:, 0]], tables.edges[cand.ee[:, 1]]
    slots = np.stack([ea[:, 0], ea[:, 1], eb[:, 0], eb[:, 1]], axis=1)
    return slots, xw[slots]


def contact(xw, cand, tables, cidx, dhat, kappa, ground_y, derivatives=True):
    """κ Σ b over candidates inside the barrier support; returns
    (Term, min_dist). Value pass returns ∞ at zero distance, derivative
    pass raises (ref contact.py:216-345)."""
    shat = dhat * dhat
    val = 0.0
    parts = []
    mins = np.inf

    if len(cand.pt):
        slots, st = pt_stencils(xw, cand, tables)
        reg = D.pt_regions(st[:, 0], st[:, 1], st[:, 2], st[:, 3])
        d2, _ = D.pt_dist2(st[:, 0], st[:, 1], st[:, 2], st[:, 3], reg)
        mins = min(mins, d2.min())
        act = d2 < shat
        if act.any():
            if np.any(d2[act] <= 0):
                if derivatives:
                    raise FloatingPointError("zero contact distance in derivative pass")
                return Term(np.inf), _md(mins)
            if derivatives:
                s, gs, hs = D.dist2_derivatives(st[act], reg[act], "pt")
                b, db, d2b = barrier_sq(s, shat)
                val += kappa * b.sum()
                g = kappa * db[:, None] * gs
                h = kappa * (d2b[:, None, None] * D._outer(gs, gs) + db[:, None, None] * hs)
                parts += lift(slots[act], g, psd(h), cidx)
            else:
                val += kappa * barrier_sq(d2[act], shat, 0).sum()

    if len(cand.ee):
        slots, st = ee_stencils(xw, cand, tables)
        reg, _ = D.ee_regions(st[:, 0], st[:, 1], st[:, 2], st[:, 3])
        d2, _ = D.ee_dist2(st[:, 0], st[:, 1], st[:, 2], st[:, 3], reg)
        mins = min(mins, d2.min())
        act = d2 < shat
        if act.any():
            if np.any(d2[act] <= 0):
                if derivatives:
                    raise FloatingPointError("zero contact distance in derivative pass")
                return Term(np.inf), _md(mins)
            eps = (EE_MOLLIFIER_SCALE * cidx.edge_rest_len2[cand.ee[act, 0]]
                   * cidx.edge_rest_len2[cand.ee[act, 1]])
            sa = st[act]
            u, v = sa[:, 1] - sa[:, 0], sa[:, 3] - sa[:, 2]
            if derivatives:
                s, gs, hs = D.dist2_derivatives(sa, reg[act], "ee")
                b, db, d2b = barrier_sq(s, shat)
                c, gc, hc = _cross2(u, v, True)
                e, de, d2e = _mollifier(c, eps)
                val += kappa * (e * b).sum()
                g = kappa * ((de * b)[:, None] * gc + (e * db)[:, None] * gs)
                x = D._outer(gc, gs)
                h = kappa * ((d2e * b)[:, None, None] * D._outer(gc, gc)
                             + (de * b)[:, None, None] * hc
                             + (de * db)[:, None, None] * (x + np.transpose(x, (0, 2, 1)))
                             + (e * d2b)[:, None, None] * D._outer(gs, gs)
                             + (e * db)[:, None, None] * hs)
                parts += lift(slots[act], g, psd(h), cidx)
            else:
                t = np.minimum(_cross2(u, v, False) / eps, 1.0)
                val += kappa * (t * (2.0 - t) * barrier_sq(d2[act], shat, 0)).sum()

    if ground_y is not None and len(cand.ground):
        d = xw[cand.ground, 1] - ground_y
        if np.any(d <= 0):
            if derivatives:
                raise FloatingPointError("vertex at or below ground in derivative pass")
            return Term(np.inf), _md(min(mins, 0.0))
        s = d * d
        mins = min(mins, s.min())
        act = s < shat
        if act.any():
            if derivatives:
                b, db, d2b = barrier_sq(s[act], shat)
                da = d[act]
                val += kappa * b.sum()
                g = np.zeros((len(da), 3))
                g[:, 1] = kappa * db * 2.0 * da
                h = np.zeros((len(da), 3, 3))
                h[:, 1, 1] = np.maximum(kappa * (d2b * 4.0 * da * da + db * 2.0), 0.0)
                parts += lift(cand.ground[act][:, None], g, h, cidx)
            else:
                val += kappa * barrier_sq(s[act], shat, 0).sum()

    return merge(val, parts), _md(mins)


def _md(min_s):
    return float(np.sqrt(min_s)) if np.isfinite(min_s) else np.inf


# ---------------------------------------------------------------------------
# lagged friction (ref friction.py)
# ---------------------------------------------------------------------------


class Lags:
    def __init__(self):
        self.slots = np.empty((0, 4), dtype=np.int64)
        self.gamma = np.empty((0, 4))
        self.tangent = np.empty((0, 3, 2))
        self.lam = np.empty(0)
        self.g_slots = np.empty(0, dtype=np.int64)
        self.g_lam = np.empty(0)

    @property
    def total(self):
        return len(self.lam) + len(self.g_lam)


def tangent_basis(n):
    """(m,3) normals → (m,3,2) frames (ref friction.py:50)."""
    ref = np.zeros_like(n)
    ux = np.abs(n[:, 0]) < 0.9
    ref[ux, 0] = 1.0
    ref[~ux, 1] = 1.0
    t1 = np.cross(n, ref)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    return np.stack([t1, np.cross(n, t1)], axis=2)


def friction_lags(xw, cand, tables, cidx, dhat, kappa, ground_y):
    """Freeze λ, tangent frames and mixing weights (ref friction.py:75)."""
    shat = dhat * dhat
    out = Lags()
    sl, ga, ta, la = [], [], [], []
    if len(cand.pt):
        slots, st = pt_stencils(xw, cand, tables)
        reg = D.pt_regions(st[:, 0], st[:, 1], st[:, 2], st[:, 3])
        d2, _ = D.pt_dist2(st[:, 0], st[:, 1], st[:, 2], st[:, 3], reg)
        act = d2 < shat
        if act.any():
            s, gs, _ = D.dist2_derivatives(st[act], reg[act], "pt")
            d = np.sqrt(s)
            _, db = barrier_sq(s, shat, 1)
            n = gs[:, :3] / (2.0 * d)[:, None]
            w = -np.einsum("nik,nk->ni", gs.reshape(-1, 4, 3)[:, 1:], n) / (2.0 * d)[:, None]
            sl.append(slots[act])
            ga.append(np.concatenate([np.ones((len(d), 1)), -w], axis=1))
            ta.append(tangent_basis(n))
            la.append(-kappa * db * 2.0 * d)
    if len(cand.ee):
        slots, st = ee_stencils(xw, cand, tables)
        reg, _ = D.ee_regions(st[:, 0], st[:, 1], st[:, 2], st[:, 3])
        d2, _ = D.ee_dist2(st[:, 0], st[:, 1], st[:, 2], st[:, 3], reg)
        act = d2 < shat
        if act.any():
            sa = st[act]
            s, gs, _ = D.dist2_derivatives(sa, reg[act], "ee")
            d = np.sqrt(s)
            _, db = barrier_sq(s, shat, 1)
            eps = (EE_MOLLIFIER_SCALE * cidx.edge_rest_len2[cand.ee[act, 0]]
                   * cidx.edge_rest_len2[cand.ee[act, 1]])
            t = np.minimum(_cross2(sa[:, 1] - sa[:, 0], sa[:, 3] - sa[:, 2], False) / eps, 1.0)
            g4 = gs.reshape(-1, 4, 3)
            n = (g4[:, 0] + g4[:, 1]) / (2.0 * d)[:, None]
            wa = np.einsum("nik,nk->ni", g4[:, :2], n) / (2.0 * d)[:, None]
            wb = -np.einsum("nik,nk->ni", g4[:, 2:], n) / (2.0 * d)[:, None]
            sl.append(slots[act])
            ga.append(np.concatenate([wa, -wb], axis=1))
            ta.append(tangent_basis(n))
            la.append(-kappa * t * (2.0 - t) * db * 2.0 * d)
    if sl:
        lam = np.concatenate(la)
        keep = lam > 0
        out.slots = np.concatenate(sl)[keep]
        out.gamma = np.concatenate(ga)[keep]
        out.tangent = np.concatenate(ta)[keep]
        out.lam = lam[keep]
    if ground_y is not None and len(cand.ground):
        d = xw[cand.ground, 1] - ground_y
        s = d * d
        act = s < shat
        if act.any():
            _, db = barrier_sq(s[act], shat, 1)
            lam = -kappa * db * 2.0 * d[act]
            keep = lam > 0
            out.g_slots = cand.ground[act][keep]
            out.g_lam = lam[keep]
    return out


def f0(y, eps_h):
    return np.where(y < eps_h, y * y / eps_h - y ** 3 / (3.0 * eps_h * eps_h) + eps_h / 3.0, y)


def f1(y, eps_h):
    return np.where(y < eps_h, 2.0 * y / eps_h - y * y / (eps_h * eps_h), 1.0)


_GROUND_T = np.array([[1.0, 0.0], [0.0, 0.0], [0.0, 1.0]])


def _smooth_norm(u3, tan, lam, mu, eps_h, derivatives):
    u = np.einsum("nkj,nk->nj", tan, u3)
    y = np.linalg.norm(u, axis=1)
    val = float((mu * lam * f0(y, eps_h)).sum())
    if not derivatives:
        return val, None, None
    fac = np.where(y > 0, f1(y, eps_h) / np.maximum(y, 1e-300), 2.0 / eps_h)
    gu = (mu * lam * fac)[:, None] * u
    df1 = np.where(y < eps_h, 2.0 / eps_h - 2.0 * y / (eps_h * eps_h), 0.0)
    coef = np.where(y > 1e-300, df1 - fac, 0.0)
    uh = u / np.maximum(y, 1e-300)[:, None]
    hu = (mu * lam)[:, None, None] * (fac[:, None, None] * np.eye(2)
                                      + coef[:, None, None] * D._outer(uh, uh))
    return val, gu, hu


def friction(xw, xw0, lags, mu, eps_v, h, cidx, derivatives=True):
    """μ λ f0(‖Tᵀ Σ γ_i Δx_i‖) over frozen contacts (ref friction.py:198)."""
    if np.any(lags.lam < 0) or np.any(lags.g_lam < 0):
        raise ValueError("negative lagged normal force")
    eps_h = eps_v * h
    dx = xw - xw0
    val = 0.0
    parts = []
    if len(lags.lam):
        u3 = np.einsum("ni,nik->nk", lags.gamma, dx[lags.slots])
        v, gu, hu = _smooth_norm(u3, lags.tangent, lags.lam, mu, eps_h, derivatives)
        val += v
        if derivatives:
            g3 = np.einsum("nkj,nj->nk", lags.tangent, gu)
            g = (lags.gamma[:, :, None] * g3[:, None, :]).reshape(-1, 12)
            h3 = np.einsum("naj,njl,nbl->nab", lags.tangent, hu, lags.tangent)
            hh = (D._outer(lags.gamma, lags.gamma)[:, :, None, :, None]
                  * h3[:, None, :, None, :]).reshape(-1, 12, 12)
            parts += lift(lags.slots, g, hh, cidx)
    if len(lags.g_lam):
        u3 = dx[lags.g_slots]
        tan = np.broadcast_to(_GROUND_T, (len(u3), 3, 2))
        v, gu, hu = _smooth_norm(u3, tan, lags.g_lam, mu, eps_h, derivatives)
        val += v
        if derivatives:
            g = np.einsum("nkj,nj->nk", tan, gu)
            hh = np.einsum("naj,njl,nbl->nab", tan, hu, tan)
            parts += lift(lags.g_slots[:, None], g, hh, cidx)
    return merge(val, parts) if derivatives else Term(val)
