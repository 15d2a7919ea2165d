"""Oracle: closest-feature classification, squared distances, and their
analytic derivatives. TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates reference pkg/src/srsim/geometry/distance.py (regions, distances)
and pkg/src/srsim/geometry/distgrad.py (derivatives). The reference obtains
derivatives by jax autodiff of four reduced formulas; here they are closed
forms of the same formulas (the same closed forms the CUDA kernels use), and
tests/test_oracle_golden.py checks them against the reference's autodiff
output.

Region codes (ref distance.py:1-9):
  point-triangle 0,1,2 vertex t0/t1/t2; 3,4,5 edge t0t1/t1t2/t2t0; 6 face
  edge-edge      3*ca + cb, ca/cb ∈ {0 endpoint0, 1 endpoint1, 2 interior}
"""

from __future__ import annotations

import numpy as np

PARALLEL_EPS = 1e-3   # ref distance.py:27
EE_DENOM_EPS = 1e-12  # ref distance.py:30


def _dot(a, b):
    return np.einsum("ij,ij->i", a, b)


# ---------------------------------------------------------------------------
# classification (ref distance.py:38, :125)
# ---------------------------------------------------------------------------


def pt_regions(p, t0, t1, t2):
    """Ericson's closest-point case analysis; first matching case wins
    (ref distance.py:38-68)."""
    ab, ac = t1 - t0, t2 - t0
    ap, bp, cp = p - t0, p - t1, p - t2
    d1, d2 = _dot(ab, ap), _dot(ac, ap)
    d3, d4 = _dot(ab, bp), _dot(ac, bp)
    d5, d6 = _dot(ab, cp), _dot(ac, cp)
    va = d3 * d6 - d5 * d4
    vb = d5 * d2 - d1 * d6
    vc = d1 * d4 - d3 * d2
    code = np.full(len(p), 6, dtype=np.int8)
    cases = [
        (d1 <= 0) & (d2 <= 0),
        (d3 >= 0) & (d4 <= d3),
        (d6 >= 0) & (d5 <= d6),
        (vc <= 0) & (d1 >= 0) & (d3 <= 0),
        (va <= 0) & (d4 - d3 >= 0) & (d5 - d6 >= 0),
        (vb <= 0) & (d2 >= 0) & (d6 <= 0),
    ]
    done = np.zeros(len(p), dtype=bool)
    for k, c in enumerate(cases):
        hit = c & ~done
        code[hit] = k
        done |= hit
    return code


def ee_regions(a0, a1, b0, b1):
    """Clamped segment-segment parameters → region code, plus the
    near-parallel flag (ref distance.py:125-162)."""
    da, db, r = a1 - a0, b1 - b0, a0 - b0
    a, e = _dot(da, da), _dot(db, db)
    f, c, b = _dot(db, r), _dot(da, r), _dot(da, db)
    den = a * e - b * b
    parallel = den < PARALLEL_EPS * a * e
    degen = den <= EE_DENOM_EPS * a * e
    safe = np.where(degen, 1.0, den)
    s = np.where(degen, 0.0, (b * f - c * e) / safe)
    s = np.clip(s, 0.0, 1.0)
    t = (b * s + f) / e
    redo = (t < 0.0) | (t > 1.0)
    t = np.clip(t, 0.0, 1.0)
    s = np.where(redo, np.clip((b * t - c) / a, 0.0, 1.0), s)
    ca = np.where(s <= 0.0, 0, np.where(s >= 1.0, 1, 2))
    cb = np.where(t <= 0.0, 0, np.where(t >= 1.0, 1, 2))
    return (3 * ca + cb).astype(np.int8), parallel


# ---------------------------------------------------------------------------
# squared distances (ref distance.py:71, :79, :165)
# ---------------------------------------------------------------------------


def point_line2(p, e0, e1):
    e = e1 - e0
    c = np.cross(e, p - e0)
    return _dot(c, c) / np.maximum(_dot(e, e), 1e-300)


def point_plane2(p, t0, t1, t2):
    n = np.cross(t1 - t0, t2 - t0)
    w = _dot(p - t0, n)
    return w * w / np.maximum(_dot(n, n), 1e-300)


def pt_dist2(p, t0, t1, t2, regions=None):
    if regions is None:
        regions = pt_regions(p, t0, t1, t2)
    out = np.empty(len(p))
    for k, t in enumerate((t0, t1, t2)):
        m = regions == k
        out[m] = _dot(p[m] - t[m], p[m] - t[m])
    for k, (a, b) in zip((3, 4, 5), ((t0, t1), (t1, t2), (t2, t0))):
        m = regions == k
        out[m] = point_line2(p[m], a[m], b[m])
    m = regions == 6
    out[m] = point_plane2(p[m], t0[m], t1[m], t2[m])
    return out, regions


def ee_dist2(a0, a1, b0, b1, regions=None):
    if regions is None:
        regions, _ = ee_regions(a0, a1, b0, b1)
    pts = (a0, a1, b0, b1)
    out = np.empty(len(a0))
    for code in range(9):
        m = regions == code
        if not m.any():
            continue
        ra, rb = divmod(code, 3)
        if ra < 2 and rb < 2:
            d = pts[ra][m] - pts[2 + rb][m]
            out[m] = _dot(d, d)
        elif ra < 2:
            out[m] = point_line2(pts[ra][m], b0[m], b1[m])
        elif rb < 2:
            out[m] = point_line2(pts[2 + rb][m], a0[m], a1[m])
        else:
            out[m] = _ll2(a0[m], a1[m], b0[m], b1[m])
    return out, regions


def _ll2(a0, a1, b0, b1):
    n = np.cross(a1 - a0, b1 - b0)
    w = _dot(b0 - a0, n)
    return w * w / np.maximum(_dot(n, n), 1e-300)


# ---------------------------------------------------------------------------
# reduced formulas with closed-form derivatives (restating ref distgrad.py)
# ---------------------------------------------------------------------------

_I3 = np.eye(3)


def _skew(a):
    z = np.zeros(a.shape[:-1] + (3, 3))
    z[..., 0, 1], z[..., 0, 2] = -a[..., 2], a[..., 1]
    z[..., 1, 0], z[..., 1, 2] = a[..., 2], -a[..., 0]
    z[..., 2, 0], z[..., 2, 1] = -a[..., 1], a[..., 0]
    return z


def _outer(a, b):
    return a[:, :, None] * b[:, None, :]


def _pp(x):
    """|x0 − x1|² over a (m, 2, 3) stencil."""
    d = x[:, 0] - x[:, 1]
    v = _dot(d, d)
    gv = [2.0 * d]
    hv = [[2.0 * np.broadcast_to(_I3, (len(x), 3, 3))]]
    return v, gv, hv, np.array([[1.0, -1.0]])


def _pl(x):
    """Point x0 to the line (x1, x2): vars (w, e) = (x0 − x1, x2 − x1)."""
    w, e = x[:, 0] - x[:, 1], x[:, 2] - x[:, 1]
    c = np.cross(e, w)
    n = _dot(e, e)
    v = _dot(c, c) / n
    t = _dot(e, w) / n
    r = w - t[:, None] * e
    g_w, g_e = 2.0 * r, -2.0 * t[:, None] * r
    k = r - t[:, None] * e
    h_ww = 2.0 * (_I3 - _outer(e, e) / n[:, None, None])
    h_we = -2.0 * t[:, None, None] * _I3 - (2.0 / n)[:, None, None] * _outer(e, k)
    h_ee = 2.0 * (t * t)[:, None, None] * _I3 - (2.0 / n)[:, None, None] * _outer(k, k)
    hv = [[h_ww, h_we], [np.transpose(h_we, (0, 2, 1)), h_ee]]
    return v, [g_w, g_e], hv, np.array([[1.0, -1.0, 0.0], [0.0, -1.0, 1.0]])


def _triple(w, u, v_):
    """f = (w·m)²/|m|², m = u × v, with gradient/Hessian in (w, u, v)."""
    m = np.cross(u, v_)
    nn = _dot(m, m)
    q = _dot(w, m)
    val = q * q / nn
    tau = q / nn
    a = 2.0 * tau[:, None] * (w - tau[:, None] * m)
    g_w = 2.0 * tau[:, None] * m
    g_u = np.cross(v_, a)
    g_v = np.cross(a, u)
    y = w - 2.0 * tau[:, None] * m
    s = (2.0 / nn)[:, None, None]
    h_ww = s * _outer(m, m)
    h_wm = s * _outer(m, y) + 2.0 * tau[:, None, None] * _I3
    h_mm = s * _outer(y, y) - 2.0 * (tau * tau)[:, None, None] * _I3
    ju, jv = -_skew(v_), _skew(u)
    tr = lambda z: np.transpose(z, (0, 2, 1))  # noqa: E731
    h_wu, h_wv = h_wm @ ju, h_wm @ jv
    h_uu = tr(ju) @ h_mm @ ju
    h_vv = tr(jv) @ h_mm @ jv
    h_uv = tr(ju) @ h_mm @ jv - _skew(a)
    hv = [[h_ww, h_wu, h_wv], [tr(h_wu), h_uu, h_uv], [tr(h_wv), tr(h_uv), h_vv]]
    return val, [g_w, g_u, g_v], hv


def _pf(x):
    """Point x0 to the plane of (x1, x2, x3): vars (x0−x1, x2−x1, x3−x1)."""
    v, g, h = _triple(x[:, 0] - x[:, 1], x[:, 2] - x[:, 1], x[:, 3] - x[:, 1])
    return v, g, h, np.array([[1.0, -1.0, 0, 0], [0, -1.0, 1.0, 0], [0, -1.0, 0, 1.0]])


def _ll(x):
    """Line (x0,x1) to line (x2,x3): vars (x2−x0, x1−x0, x3−x2)."""
    v, g, h = _triple(x[:, 2] - x[:, 0], x[:, 1] - x[:, 0], x[:, 3] - x[:, 2])
    return v, g, h, np.array([[-1.0, 0, 1.0, 0], [-1.0, 1.0, 0, 0], [0, 0, -1.0, 1.0]])


def _to_vertices(gv, hv, cmap):
    """Chain var-space derivatives to the k active vertices via the constant
    map var_i = Σ_a cmap[i, a] x_a."""
    nv, k = cmap.shape
    m = gv[0].shape[0]
    g = np.zeros((m, k, 3))
    h = np.zeros((m, k, 3, k, 3))
    for i in range(nv):
        for a in range(k):
            if cmap[i, a] != 0.0:
                g[:, a] += cmap[i, a] * gv[i]
    for i in range(nv):
        for j in range(nv):
            for a in range(k):
                for b in range(k):
                    c = cmap[i, a] * cmap[j, b]
                    if c != 0.0:
                        h[:, a, :, b, :] += c * hv[i][j]
    return g, h


_FORMS = {"pp": _pp, "pl": _pl, "pf": _pf, "ll": _ll}

# region → (formula, active stencil slots) (ref distgrad.py:68-89)
PT_TABLE = {0: ("pp", (0, 1)), 1: ("pp", (0, 2)), 2: ("pp", (0, 3)),
            3: ("pl", (0, 1, 2)), 4: ("pl", (0, 2, 3)), 5: ("pl", (0, 3, 1)),
            6: ("pf", (0, 1, 2, 3))}
EE_TABLE = {0: ("pp", (0, 2)), 1: ("pp", (0, 3)), 2: ("pl", (0, 2, 3)),
            3: ("pp", (1, 2)), 4: ("pp", (1, 3)), 5: ("pl", (1, 2, 3)),
            6: ("pl", (2, 0, 1)), 7: ("pl", (3, 0, 1)), 8: ("ll", (0, 1, 2, 3))}


def dist2_derivatives(stencils, regions, kind):
    """(m, 4, 3) stencils → s (m,), ∂s (m, 12), ∂²s (m, 12, 12)
    (restates ref distgrad.py:95)."""
    table = PT_TABLE if kind == "pt" else EE_TABLE
    m = len(stencils)
    s = np.zeros(m)
    g = np.zeros((m, 4, 3))
    h = np.zeros((m, 4, 3, 4, 3))
    for code in np.unique(regions):
        name, slots = table[int(code)]
        idx = np.nonzero(regions == code)[0]
        x = stencils[idx][:, list(slots)]
        val, gv, hv, cmap = _FORMS[name](x)
        gl, hl = _to_vertices(gv, hv, cmap)
        s[idx] = val
        for a, sa in enumerate(slots):
            g[idx, sa] = gl[:, a]
            for b, sb in enumerate(slots):
                h[idx, sa, :, sb, :] = hl[:, a, :, b, :]
    return s, g.reshape(m, 12), h.reshape(m, 12, 12)
