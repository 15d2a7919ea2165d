// Device math for the IPC time step (fp64 throughout).
//
//  * closest-feature classification and squared distances for
//    point-triangle / edge-edge stencils — same case analysis and formulas
//    as the reference (pkg/src/srsim/geometry/distance.py:38,:79,:125,:165)
//    so region codes and candidate distances agree with the CPU path;
//  * closed-form gradients / Hessians of the four reduced squared-distance
//    formulas (the reference autodiffs them: geometry/distgrad.py:32-53);
//  * the log barrier on squared distance (energy/barrier.py:51) and the
//    edge-edge mollifier (energy/contact.py:166-203);
//  * eigenvalue-clamping PSD projection (energy/spd.py:6) by Householder tridiagonalisation + implicit QL (tred2/tql2),
//    with a Cholesky fast path for blocks that are already positive definite;
//  * NeoHookean / StVK / FixedCorotated densities, PK1 and F-space Hessians
//    (energy/elastic.py:23-167).
#pragma once
#include <math.h>
#include <stdint.h>

#define IPC_HD __device__ __forceinline__

namespace ipc {

// ---------------------------------------------------------------------------
// small vector helpers
// ---------------------------------------------------------------------------
struct V3 {
  double x, y, z;
};
IPC_HD V3 v3(double x, double y, double z) { return V3{x, y, z}; }
IPC_HD V3 ld3(const double* p) { return V3{p[0], p[1], p[2]}; }
IPC_HD void st3(double* p, V3 a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }
IPC_HD V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
IPC_HD V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
IPC_HD V3 operator*(double s, V3 a) { return V3{s * a.x, s * a.y, s * a.z}; }
IPC_HD double at(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
// numpy einsum("ij,ij->i") order: ((a0 b0 + a1 b1) + a2 b2), no contraction
IPC_HD double dotx(V3 a, V3 b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
IPC_HD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
// numpy cross order: (a1 b2 - a2 b1, a2 b0 - a0 b2, a0 b1 - a1 b0), no contraction
IPC_HD V3 crossx(V3 a, V3 b) {
  return V3{__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)),
            __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
            __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
IPC_HD V3 cross(V3 a, V3 b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// 3x3 row-major matrices
struct M3 {
  double m[9];
};
IPC_HD M3 m3_zero() {
  M3 r;
#pragma unroll
  for (int i = 0; i < 9; ++i) r.m[i] = 0.0;
  return r;
}
IPC_HD M3 m3_outer(V3 a, V3 b) {
  M3 r;
  r.m[0] = a.x * b.x; r.m[1] = a.x * b.y; r.m[2] = a.x * b.z;
  r.m[3] = a.y * b.x; r.m[4] = a.y * b.y; r.m[5] = a.y * b.z;
  r.m[6] = a.z * b.x; r.m[7] = a.z * b.y; r.m[8] = a.z * b.z;
  return r;
}
IPC_HD M3 m3_skew(V3 a) {  // skew(a) b = a x b
  M3 r;
  r.m[0] = 0; r.m[1] = -a.z; r.m[2] = a.y;
  r.m[3] = a.z; r.m[4] = 0; r.m[5] = -a.x;
  r.m[6] = -a.y; r.m[7] = a.x; r.m[8] = 0;
  return r;
}
IPC_HD M3 m3_mul(const M3& a, const M3& b) {
  M3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r.m[3 * i + j] = a.m[3 * i] * b.m[j] + a.m[3 * i + 1] * b.m[3 + j] + a.m[3 * i + 2] * b.m[6 + j];
  return r;
}
IPC_HD M3 m3_tmul(const M3& a, const M3& b) {  // a^T b
  M3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r.m[3 * i + j] = a.m[i] * b.m[j] + a.m[3 + i] * b.m[3 + j] + a.m[6 + i] * b.m[6 + j];
  return r;
}
IPC_HD M3 m3_T(const M3& a) {
  M3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.m[3 * i + j] = a.m[3 * j + i];
  return r;
}
IPC_HD void m3_axpy(M3& y, double s, const M3& x) {
#pragma unroll
  for (int i = 0; i < 9; ++i) y.m[i] += s * x.m[i];
}
IPC_HD void m3_add_diag(M3& y, double s) { y.m[0] += s; y.m[4] += s; y.m[8] += s; }
IPC_HD double m3_det(const M3& a) {
  return a.m[0] * (a.m[4] * a.m[8] - a.m[5] * a.m[7]) - a.m[1] * (a.m[3] * a.m[8] - a.m[5] * a.m[6]) +
         a.m[2] * (a.m[3] * a.m[7] - a.m[4] * a.m[6]);
}

// ---------------------------------------------------------------------------
// classification and squared distances (ref distance.py)
// ---------------------------------------------------------------------------
enum { PT_V0 = 0, PT_V1, PT_V2, PT_E01, PT_E12, PT_E20, PT_INT };

IPC_HD int pt_region(V3 p, V3 t0, V3 t1, V3 t2) {
  V3 ab = t1 - t0, ac = t2 - t0;
  V3 ap = p - t0, bp = p - t1, cp = p - t2;
  double d1 = dotx(ab, ap), d2 = dotx(ac, ap);
  double d3 = dotx(ab, bp), d4 = dotx(ac, bp);
  double d5 = dotx(ab, cp), d6 = dotx(ac, cp);
  double va = __dsub_rn(__dmul_rn(d3, d6), __dmul_rn(d5, d4));
  double vb = __dsub_rn(__dmul_rn(d5, d2), __dmul_rn(d1, d6));
  double vc = __dsub_rn(__dmul_rn(d1, d4), __dmul_rn(d3, d2));
  if (d1 <= 0 && d2 <= 0) return PT_V0;
  if (d3 >= 0 && d4 <= d3) return PT_V1;
  if (d6 >= 0 && d5 <= d6) return PT_V2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) return PT_E01;
  if (va <= 0 && __dsub_rn(d4, d3) >= 0 && __dsub_rn(d5, d6) >= 0) return PT_E12;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) return PT_E20;
  return PT_INT;
}

IPC_HD double point_line2(V3 p, V3 e0, V3 e1) {
  V3 e = e1 - e0;
  V3 c = crossx(e, p - e0);
  return __ddiv_rn(dotx(c, c), fmax(dotx(e, e), 1e-300));
}
IPC_HD double point_plane2(V3 p, V3 t0, V3 t1, V3 t2) {
  V3 n = crossx(t1 - t0, t2 - t0);
  double w = dotx(p - t0, n);
  return __ddiv_rn(__dmul_rn(w, w), fmax(dotx(n, n), 1e-300));
}
IPC_HD double line_line2(V3 a0, V3 a1, V3 b0, V3 b1) {
  V3 n = crossx(a1 - a0, b1 - b0);
  double w = dotx(b0 - a0, n);
  return __ddiv_rn(__dmul_rn(w, w), fmax(dotx(n, n), 1e-300));
}
IPC_HD double pp2(V3 a, V3 b) {
  V3 d = a - b;
  return dotx(d, d);
}

IPC_HD double pt_dist2(int r, V3 p, V3 t0, V3 t1, V3 t2) {
  switch (r) {
    case PT_V0: return pp2(p, t0);
    case PT_V1: return pp2(p, t1);
    case PT_V2: return pp2(p, t2);
    case PT_E01: return point_line2(p, t0, t1);
    case PT_E12: return point_line2(p, t1, t2);
    case PT_E20: return point_line2(p, t2, t0);
    default: return point_plane2(p, t0, t1, t2);
  }
}

// returns region code 3*ca+cb; *parallel set per ref distance.py:142
IPC_HD int ee_region(V3 a0, V3 a1, V3 b0, V3 b1, bool* parallel) {
  V3 d1 = a1 - a0, d2 = b1 - b0, r = a0 - b0;
  double a = dotx(d1, d1), e = dotx(d2, d2), f = dotx(d2, r), c = dotx(d1, r), b = dotx(d1, d2);
  double ae = __dmul_rn(a, e);
  double den = __dsub_rn(ae, __dmul_rn(b, b));
  if (parallel) *parallel = den < __dmul_rn(__dmul_rn(1e-3, a), e);  // (eps*a)*e as numpy
  bool degen = den <= __dmul_rn(__dmul_rn(1e-12, a), e);
  double s = degen ? 0.0 : __ddiv_rn(__dsub_rn(__dmul_rn(b, f), __dmul_rn(c, e)), den);
  s = fmin(fmax(s, 0.0), 1.0);
  double t = __ddiv_rn(__dadd_rn(__dmul_rn(b, s), f), e);
  bool redo = (t < 0.0) || (t > 1.0);
  t = fmin(fmax(t, 0.0), 1.0);
  if (redo) s = fmin(fmax(__ddiv_rn(__dsub_rn(__dmul_rn(b, t), c), a), 0.0), 1.0);
  int ca = s <= 0.0 ? 0 : (s >= 1.0 ? 1 : 2);
  int cb = t <= 0.0 ? 0 : (t >= 1.0 ? 1 : 2);
  return 3 * ca + cb;
}

IPC_HD double ee_dist2(int r, V3 a0, V3 a1, V3 b0, V3 b1) {
  int ra = r / 3, rb = r % 3;
  V3 pa = ra == 0 ? a0 : a1;
  V3 pb = rb == 0 ? b0 : b1;
  if (ra < 2 && rb < 2) return pp2(pa, pb);
  if (ra < 2) return point_line2(pa, b0, b1);
  if (rb < 2) return point_line2(pb, a0, a1);
  return line_line2(a0, a1, b0, b1);
}

// ---------------------------------------------------------------------------
// closed-form derivatives of the reduced squared-distance formulas
// G: 4x3 stencil gradient, H: 12x12 stencil Hessian (row-major).
// ---------------------------------------------------------------------------

// accumulate a 3x3 var-space block (scaled by c) into stencil slots (sa, sb)
IPC_HD void add_blk(double* H, int sa, int sb, double c, const M3& b) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) H[(3 * sa + i) * 12 + 3 * sb + j] += c * b.m[3 * i + j];
}
IPC_HD void add_vec(double* G, int sa, double c, V3 g) {
  G[3 * sa] += c * g.x;
  G[3 * sa + 1] += c * g.y;
  G[3 * sa + 2] += c * g.z;
}

// Chain var-space derivatives to stencil slots. cmap[i][a] ∈ {-1,0,1} maps
// var i = Σ_a cmap[i][a] x_{slot[a]}.
template <int NV, int K>
IPC_HD void scatter_vars(const signed char (&cmap)[NV][K], const int (&slot)[K], const V3 (&gv)[NV],
                         const M3 (&hv)[NV][NV], double* G, double* H) {
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int a = 0; a < K; ++a)
      if (cmap[i][a]) add_vec(G, slot[a], (double)cmap[i][a], gv[i]);
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          int c = cmap[i][a] * cmap[j][b];
          if (c) add_blk(H, slot[a], slot[b], (double)c, hv[i][j]);
        }
}

// |x0 - x1|^2
IPC_HD double d2_pp(const V3* x, int s0, int s1, double* G, double* H) {
  V3 d = x[s0] - x[s1];
  V3 gv[1] = {2.0 * d};
  M3 I2 = m3_zero();
  m3_add_diag(I2, 2.0);
  M3 hv[1][1] = {{I2}};
  const signed char cm[1][2] = {{1, -1}};
  const int sl[2] = {s0, s1};
  scatter_vars<1, 2>(cm, sl, gv, hv, G, H);
  return dotx(d, d);
}

// point x0 to line (x1, x2); vars (w, e) = (x0 - x1, x2 - x1)
IPC_HD double d2_pl(const V3* x, int s0, int s1, int s2, double* G, double* H) {
  V3 w = x[s0] - x[s1], e = x[s2] - x[s1];
  V3 c = crossx(e, w);
  double n = dotx(e, e);
  double val = __ddiv_rn(dotx(c, c), n);
  double t = dot(e, w) / n;
  V3 r = w - t * e;
  V3 k = r - t * e;
  V3 gv[2] = {2.0 * r, (-2.0 * t) * r};
  M3 hww = m3_outer(e, e);
  for (int i = 0; i < 9; ++i) hww.m[i] *= -2.0 / n;
  m3_add_diag(hww, 2.0);
  M3 hwe = m3_outer(e, k);
  for (int i = 0; i < 9; ++i) hwe.m[i] *= -2.0 / n;
  m3_add_diag(hwe, -2.0 * t);
  M3 hee = m3_outer(k, k);
  for (int i = 0; i < 9; ++i) hee.m[i] *= -2.0 / n;
  m3_add_diag(hee, 2.0 * t * t);
  M3 hv[2][2] = {{hww, hwe}, {m3_T(hwe), hee}};
  const signed char cm[2][3] = {{1, -1, 0}, {0, -1, 1}};
  const int sl[3] = {s0, s1, s2};
  scatter_vars<2, 3>(cm, sl, gv, hv, G, H);
  return val;
}

// f = (w.m)^2/|m|^2, m = u x v — var-space gradient and Hessian
IPC_HD double triple_vars(V3 w, V3 u, V3 v, V3 (&gv)[3], M3 (&hv)[3][3]) {
  V3 m = cross(u, v);
  double nn = dot(m, m);
  double q = dot(w, m);
  double tau = q / nn;
  V3 a = (2.0 * tau) * (w - tau * m);
  gv[0] = (2.0 * tau) * m;
  gv[1] = cross(v, a);
  gv[2] = cross(a, u);
  V3 y = w - (2.0 * tau) * m;
  double s = 2.0 / nn;
  M3 hww = m3_outer(m, m);
  for (int i = 0; i < 9; ++i) hww.m[i] *= s;
  M3 hwm = m3_outer(m, y);
  for (int i = 0; i < 9; ++i) hwm.m[i] *= s;
  m3_add_diag(hwm, 2.0 * tau);
  M3 hmm = m3_outer(y, y);
  for (int i = 0; i < 9; ++i) hmm.m[i] *= s;
  m3_add_diag(hmm, -2.0 * tau * tau);
  M3 ju = m3_skew(v);
  for (int i = 0; i < 9; ++i) ju.m[i] = -ju.m[i];
  M3 jv = m3_skew(u);
  M3 hwu = m3_mul(hwm, ju), hwv = m3_mul(hwm, jv);
  M3 hmu = m3_mul(hmm, ju), hmv = m3_mul(hmm, jv);
  M3 huu = m3_tmul(ju, hmu), hvv = m3_tmul(jv, hmv), huv = m3_tmul(ju, hmv);
  M3 sa = m3_skew(a);
  m3_axpy(huv, -1.0, sa);
  hv[0][0] = hww; hv[0][1] = hwu; hv[0][2] = hwv;
  hv[1][0] = m3_T(hwu); hv[1][1] = huu; hv[1][2] = huv;
  hv[2][0] = m3_T(hwv); hv[2][1] = m3_T(huv); hv[2][2] = hvv;
  return 0.0;
}

// point x0 to plane (x1,x2,x3): vars (x0-x1, x2-x1, x3-x1)
IPC_HD double d2_pf(const V3* x, int s0, int s1, int s2, int s3, double* G, double* H) {
  V3 w = x[s0] - x[s1], u = x[s2] - x[s1], v = x[s3] - x[s1];
  V3 gv[3];
  M3 hv[3][3];
  triple_vars(w, u, v, gv, hv);
  const signed char cm[3][4] = {{1, -1, 0, 0}, {0, -1, 1, 0}, {0, -1, 0, 1}};
  const int sl[4] = {s0, s1, s2, s3};
  scatter_vars<3, 4>(cm, sl, gv, hv, G, H);
  V3 n = crossx(u, v);
  double q = dotx(w, n);
  return __ddiv_rn(__dmul_rn(q, q), dotx(n, n));
}

// line (x0,x1) to line (x2,x3): vars (x2-x0, x1-x0, x3-x2)
IPC_HD double d2_ll(const V3* x, double* G, double* H) {
  V3 w = x[2] - x[0], u = x[1] - x[0], v = x[3] - x[2];
  V3 gv[3];
  M3 hv[3][3];
  triple_vars(w, u, v, gv, hv);
  const signed char cm[3][4] = {{-1, 0, 1, 0}, {-1, 1, 0, 0}, {0, 0, -1, 1}};
  const int sl[4] = {0, 1, 2, 3};
  scatter_vars<3, 4>(cm, sl, gv, hv, G, H);
  V3 n = crossx(u, v);
  double q = dotx(w, n);
  return __ddiv_rn(__dmul_rn(q, q), dotx(n, n));
}

// Squared distance + derivatives for a stencil (p,t0,t1,t2) or (a0,a1,b0,b1).
// Region tables follow ref distgrad.py:68-89. G (12) and H (144) must be
// zero on entry. Returns s. *mask gets the bitmask of active stencil slots.
IPC_HD double dist2_derivs(bool is_pt, int region, const V3* x, double* G, double* H, int* mask) {
  if (is_pt) {
    switch (region) {
      case 0: *mask = 0x3; return d2_pp(x, 0, 1, G, H);
      case 1: *mask = 0x5; return d2_pp(x, 0, 2, G, H);
      case 2: *mask = 0x9; return d2_pp(x, 0, 3, G, H);
      case 3: *mask = 0x7; return d2_pl(x, 0, 1, 2, G, H);
      case 4: *mask = 0xD; return d2_pl(x, 0, 2, 3, G, H);
      case 5: *mask = 0xB; return d2_pl(x, 0, 3, 1, G, H);
      default: *mask = 0xF; return d2_pf(x, 0, 1, 2, 3, G, H);
    }
  }
  switch (region) {
    case 0: *mask = 0x5; return d2_pp(x, 0, 2, G, H);
    case 1: *mask = 0x9; return d2_pp(x, 0, 3, G, H);
    case 2: *mask = 0xD; return d2_pl(x, 0, 2, 3, G, H);
    case 3: *mask = 0x6; return d2_pp(x, 1, 2, G, H);
    case 4: *mask = 0xA; return d2_pp(x, 1, 3, G, H);
    case 5: *mask = 0xE; return d2_pl(x, 1, 2, 3, G, H);
    case 6: *mask = 0x7; return d2_pl(x, 2, 0, 1, G, H);
    case 7: *mask = 0xB; return d2_pl(x, 3, 0, 1, G, H);
    default: *mask = 0xF; return d2_ll(x, G, H);
  }
}

// ---------------------------------------------------------------------------
// barrier on squared distance (ref barrier.py:51) and EE mollifier
// ---------------------------------------------------------------------------
IPC_HD double barrier_val(double s, double shat) {
  if (!(s < shat)) return 0.0;
  double g = s - shat;
  return -g * g * log(s / shat);
}
IPC_HD void barrier_d(double s, double shat, double* b, double* db, double* d2b) {
  if (!(s < shat)) {
    *b = *db = *d2b = 0.0;
    return;
  }
  double g = s - shat;
  double ln = log(s / shat);
  *b = -g * g * ln;
  *db = -2.0 * g * ln - g * g / s;
  *d2b = -2.0 * ln - 4.0 * g / s + g * g / (s * s);
}

IPC_HD double cross2(V3 u, V3 v) {
  double uu = dotx(u, u), vv = dotx(v, v), uv = dotx(u, v);
  return __dsub_rn(__dmul_rn(uu, vv), __dmul_rn(uv, uv));
}
IPC_HD double mollifier_val(double c, double eps) {
  double t = fmin(c / eps, 1.0);
  return t * (2.0 - t);
}

// c = |u x v|^2 over stencil (a0,a1,b0,b1): gradient Gc (12), Hessian Hc (144, zero on entry)
IPC_HD double cross2_derivs(const V3* x, double* Gc, double* Hc) {
  V3 u = x[1] - x[0], v = x[3] - x[2];
  double uu = dot(u, u), vv = dot(v, v), uv = dot(u, v);
  V3 gv[2] = {2.0 * (vv * u - uv * v), 2.0 * (uu * v - uv * u)};
  M3 huu = m3_outer(v, v);
  for (int i = 0; i < 9; ++i) huu.m[i] *= -2.0;
  m3_add_diag(huu, 2.0 * vv);
  M3 hvv = m3_outer(u, u);
  for (int i = 0; i < 9; ++i) hvv.m[i] *= -2.0;
  m3_add_diag(hvv, 2.0 * uu);
  M3 huv = m3_outer(u, v), t2 = m3_outer(v, u);
  for (int i = 0; i < 9; ++i) huv.m[i] = 4.0 * huv.m[i] - 2.0 * t2.m[i];
  m3_add_diag(huv, -2.0 * uv);
  M3 hv[2][2] = {{huu, huv}, {m3_T(huv), hvv}};
  const signed char cm[2][4] = {{-1, 1, 0, 0}, {0, 0, -1, 1}};
  const int sl[4] = {0, 1, 2, 3};
  scatter_vars<2, 4>(cm, sl, gv, hv, Gc, Hc);
  return cross2(u, v);
}

// gradient of c = |u x v|² into Gc; when H is given, hscale · ∇²c is
// accumulated into H (no separate 12x12 array)
IPC_HD double cross2_grad_acc(const V3* x, double* Gc, double* H, double hscale) {
  V3 u = x[1] - x[0], v = x[3] - x[2];
  double uu = dot(u, u), vv = dot(v, v), uv = dot(u, v);
  V3 gv[2] = {2.0 * (vv * u - uv * v), 2.0 * (uu * v - uv * u)};
  const signed char cm[2][4] = {{-1, 1, 0, 0}, {0, 0, -1, 1}};
  const int sl[4] = {0, 1, 2, 3};
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int a = 0; a < 4; ++a)
      if (cm[i][a]) add_vec(Gc, sl[a], (double)cm[i][a], gv[i]);
  if (H) {
    M3 huu = m3_outer(v, v);
    for (int i = 0; i < 9; ++i) huu.m[i] *= -2.0;
    m3_add_diag(huu, 2.0 * vv);
    M3 hvv = m3_outer(u, u);
    for (int i = 0; i < 9; ++i) hvv.m[i] *= -2.0;
    m3_add_diag(hvv, 2.0 * uu);
    M3 huv = m3_outer(u, v), t2 = m3_outer(v, u);
    for (int i = 0; i < 9; ++i) huv.m[i] = 4.0 * huv.m[i] - 2.0 * t2.m[i];
    m3_add_diag(huv, -2.0 * uv);
    M3 hv[2][2] = {{huu, huv}, {m3_T(huv), hvv}};
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            int c = cm[i][a] * cm[j][b];
            if (c) add_blk(H, sl[a], sl[b], hscale * (double)c, hv[i][j]);
          }
  }
  return cross2(u, v);
}

// ---------------------------------------------------------------------------
// PSD projection of a symmetric NxN block (row-major, stride LD)
// ---------------------------------------------------------------------------
template <int N>
IPC_HD bool chol_pd(const double* A, int ld) {
  double L[N * (N + 1) / 2];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double d = A[j * ld + j];
#pragma unroll
    for (int k = 0; k < j; ++k) {
      double l = L[j * (j + 1) / 2 + k];
      d -= l * l;
    }
    if (!(d > 1e-14 * fabs(A[j * ld + j]) && d > 0.0)) return false;
    double dj = sqrt(d);
    L[j * (j + 1) / 2 + j] = dj;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      double s = A[i * ld + j];
#pragma unroll
      for (int k = 0; k < j; ++k) s -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
      L[i * (i + 1) / 2 + j] = s / dj;
    }
  }
  return true;
}

// Symmetric eigen-decomposition, V (N x N, row-major) holds A on entry and the
// eigenvectors (columns) on exit, d the eigenvalues. Householder reduction to
// tridiagonal form followed by the implicit QL iteration (the classical
// tred2/tql2 pair): O(N³) with a small constant, ~10x fewer flops than
// cyclic Jacobi at N = 12.
template <int N>
IPC_HD void sym_eigen(double* V, double* d, double* e) {
  // Every loop is unrolled and every array index is a compile-time constant
  // (the data-dependent QL bounds l..m become predicates), so V, d, e can be
  // register-allocated instead of living in local memory.
#pragma unroll
  for (int j = 0; j < N; ++j) d[j] = V[(N - 1) * N + j];
#pragma unroll
  for (int i = N - 1; i > 0; --i) {
    double scale = 0.0, h = 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) scale += fabs(d[k]);
    if (scale == 0.0) {
      e[i] = d[i - 1];
#pragma unroll
      for (int j = 0; j < i; ++j) {
        d[j] = V[(i - 1) * N + j];
        V[i * N + j] = 0.0;
        V[j * N + i] = 0.0;
      }
    } else {
      const double iscale = 1.0 / scale;  // one division on the chain, then products
#pragma unroll
      for (int k = 0; k < i; ++k) {
        d[k] *= iscale;
        h += d[k] * d[k];
      }
      double f = d[i - 1];
      double g = sqrt(h);
      if (f > 0) g = -g;
      e[i] = scale * g;
      h -= f * g;
      d[i - 1] = f - g;
#pragma unroll
      for (int j = 0; j < i; ++j) e[j] = 0.0;
#pragma unroll
      for (int j = 0; j < i; ++j) {
        f = d[j];
        V[j * N + i] = f;
        g = e[j] + V[j * N + j] * f;
#pragma unroll
        for (int k = j + 1; k <= i - 1; ++k) {
          g += V[k * N + j] * d[k];
          e[k] += V[k * N + j] * f;
        }
        e[j] = g;
      }
      f = 0.0;
      const double ih = 1.0 / h;
#pragma unroll
      for (int j = 0; j < i; ++j) {
        e[j] *= ih;
        f += e[j] * d[j];
      }
      double hh = f / (h + h);
#pragma unroll
      for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
#pragma unroll
      for (int j = 0; j < i; ++j) {
        f = d[j];
        g = e[j];
#pragma unroll
        for (int k = j; k <= i - 1; ++k) V[k * N + j] -= (f * e[k] + g * d[k]);
        d[j] = V[(i - 1) * N + j];
        V[i * N + j] = 0.0;
      }
    }
    d[i] = h;
  }
#pragma unroll
  for (int i = 0; i < N - 1; ++i) {
    V[(N - 1) * N + i] = V[i * N + i];
    V[i * N + i] = 1.0;
    double h = d[i + 1];
    if (h != 0.0) {
      const double ih = 1.0 / h;
#pragma unroll
      for (int k = 0; k <= i; ++k) d[k] = V[k * N + i + 1] * ih;
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        double g = 0.0;
#pragma unroll
        for (int k = 0; k <= i; ++k) g += V[k * N + i + 1] * V[k * N + j];
#pragma unroll
        for (int k = 0; k <= i; ++k) V[k * N + j] -= g * d[k];
      }
    }
#pragma unroll
    for (int k = 0; k <= i; ++k) V[k * N + i + 1] = 0.0;
  }
#pragma unroll
  for (int j = 0; j < N; ++j) {
    d[j] = V[(N - 1) * N + j];
    V[(N - 1) * N + j] = 0.0;
  }
  V[(N - 1) * N + N - 1] = 1.0;
  e[0] = 0.0;
  // implicit QL
#pragma unroll
  for (int i = 1; i < N; ++i) e[i - 1] = e[i];
  e[N - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = 2.220446049250313e-16;
#pragma unroll
  for (int l = 0; l < N; ++l) {
    tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
    // m = first index >= l with a negligible off-diagonal (predicated search)
    int m = N - 1;
#pragma unroll
    for (int k = N - 2; k >= l; --k)
      if (fabs(e[k]) <= eps * tst1) m = k;
    if (l < N - 1 && m > l) {
      for (int iter = 0; iter < 60; ++iter) {
        double g = d[l];
        double p = (d[l + 1] - g) / (2.0 * e[l]);
        double r = sqrt(fma(p, p, 1.0));  // hypot(p, 1) without the scaling (|p| << 1e150 here)
        if (p < 0) r = -r;
        d[l] = e[l] / (p + r);
        d[l + 1] = e[l] * (p + r);
        double dl1 = d[l + 1];
        double h = g - d[l];
#pragma unroll
        for (int i = l + 2; i < N; ++i) d[i] -= h;
        f += h;
        p = 0.0;
#pragma unroll
        for (int k = l; k < N; ++k)
          if (k == m) p = d[k];
        double c = 1.0, c2 = 1.0, c3 = 1.0, el1 = e[l + 1 < N ? l + 1 : N - 1], s = 0.0, s2 = 0.0;
#pragma unroll
        for (int i = N - 2; i >= l; --i) {
          if (i < m) {
            c3 = c2;
            c2 = c;
            s2 = s;
            g = c * e[i];
            h = c * p;
            // Givens pair from one reciprocal square root (hypot and two
            // divisions were the latency of the QL sweep)
            double ei = e[i], rr = fma(p, p, ei * ei);
            double ir = rsqrt(rr);
            r = rr * ir;
            e[i + 1] = s * r;
            s = ei * ir;
            c = p * ir;
            p = c * d[i] - s * g;
            d[i + 1] = h + s * (c * g + s * d[i]);
#pragma unroll
            for (int k = 0; k < N; ++k) {
              h = V[k * N + i + 1];
              V[k * N + i + 1] = s * V[k * N + i] + c * h;
              V[k * N + i] = c * V[k * N + i] - s * h;
            }
          }
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = c * p;
        if (!(fabs(e[l]) > eps * tst1)) break;
      }
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
}

// In-place: A <- V max(Λ,0) Vᵀ. Symmetrizes first (ref spd.py:8).
template <int N>
IPC_HD void psd_project(double* A, int ld) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i + 1; j < N; ++j) {
      double s = 0.5 * (A[i * ld + j] + A[j * ld + i]);
      A[i * ld + j] = A[j * ld + i] = s;
    }
  if (chol_pd<N>(A, ld)) return;  // already positive definite: projection is the identity
  double V[N * N], d[N], e[N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) V[i * N + j] = A[i * ld + j];
  sym_eigen<N>(V, d, e);
#pragma unroll
  for (int i = 0; i < N; ++i) d[i] = fmax(d[i], 0.0);
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) s += V[i * N + k] * d[k] * V[j * N + k];
      A[i * ld + j] = A[j * ld + i] = s;
    }
}

// PSD projection of a 3NS x 3NS stencil Hessian that annihilates rigid
// translations (every contact/friction stencil energy depends on vertex
// differences only). With Q = Q0 ⊗ I3, Q0 the orthonormal NS x (NS-1)
// Helmert basis of the complement of (1,…,1), A = Q (QᵀAQ) Qᵀ exactly, and
// since Q has orthonormal columns the eigenvalue clamp commutes:
// A⁺ = Q (QᵀAQ)⁺ Qᵀ. Same operator as the full clamp (ref spd.py:6), on a
// 3(NS-1) core: 9x9 instead of 12x12, 6x6 instead of 9x9, 3x3 instead of 6x6.
template <int NS>
IPC_HD void psd_project_tf(double* A, int ld) {
  constexpr int N = 3 * NS, R = 3 * (NS - 1);
  double q0[NS][NS - 1];
#pragma unroll
  for (int j = 0; j < NS - 1; ++j) {
    double nrm = rsqrt((double)((j + 1) * (j + 2)));
#pragma unroll
    for (int a = 0; a < NS; ++a) q0[a][j] = a <= j ? nrm : (a == j + 1 ? -(j + 1) * nrm : 0.0);
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i + 1; j < N; ++j) {
      double s = 0.5 * (A[i * ld + j] + A[j * ld + i]);
      A[i * ld + j] = A[j * ld + i] = s;
    }
  // M = Qᵀ A Q, block (I, J) = Σ_ab q0[a][I] q0[b][J] A_ab (3x3 blocks)
  double M[R * R];
#pragma unroll
  for (int I = 0; I < NS - 1; ++I)
#pragma unroll
    for (int J = 0; J < NS - 1; ++J)
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < NS; ++a) {
            if (a > I + 1) continue;  // q0[a][I] == 0
            double t = 0.0;
#pragma unroll
            for (int b = 0; b < NS; ++b) {
              if (b > J + 1) continue;
              t += q0[b][J] * A[(3 * a + r) * ld + 3 * b + c];
            }
            s += q0[a][I] * t;
          }
          M[(3 * I + r) * R + 3 * J + c] = s;
        }
  psd_project<R>(M, R);
  // A = Q M Qᵀ
#pragma unroll
  for (int a = 0; a < NS; ++a)
#pragma unroll
    for (int b = a; b < NS; ++b)
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (b == a && c < r) continue;
          double s = 0.0;
#pragma unroll
          for (int I = 0; I < NS - 1; ++I) {
            if (a > I + 1) continue;
            double t = 0.0;
#pragma unroll
            for (int J = 0; J < NS - 1; ++J) {
              if (b > J + 1) continue;
              t += M[(3 * I + r) * R + 3 * J + c] * q0[b][J];
            }
            s += q0[a][I] * t;
          }
          A[(3 * a + r) * ld + 3 * b + c] = A[(3 * b + c) * ld + 3 * a + r] = s;
        }
}

// Project only the rows/columns of a 12x12 stencil Hessian whose slots are
// active (mask bit per 3-row slot); inactive rows are identically zero, and
// zero rows/columns carry eigenvalue 0, so this equals the full projection.
IPC_HD void psd_project_masked12(double* H, int mask) {
  int idx[12];
  int k = 0;
  for (int s = 0; s < 4; ++s)
    if (mask & (1 << s))
      for (int c = 0; c < 3; ++c) idx[k++] = 3 * s + c;
  if (k == 12) {
    psd_project_tf<4>(H, 12);
    return;
  }
  double sub[81];
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) sub[i * k + j] = H[idx[i] * 12 + idx[j]];
  if (k == 6) psd_project_tf<2>(sub, 6);
  else psd_project_tf<3>(sub, 9);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) H[idx[i] * 12 + idx[j]] = sub[i * k + j];
}

// ---------------------------------------------------------------------------
// Contact stencil Hessians built directly in the Helmert space of the
// stencil's active slots (no 12x12 array).
//
// Every distance formula is a function of difference vectors v_i =
// x_{p_i} - x_{q_i} of the stencil points, so its stencil Hessian is
// H = Dᵀ K D (K: var-space Hessian) and annihilates rigid translations. With
// Q = Q0 ⊗ I3, Q0 the orthonormal NS x (NS-1) Helmert basis of the
// complement of (1,…,1): H = Q (Bᵀ K B) Qᵀ, B = D Q = β ⊗ I3 with
// β[i][J] = q0[p_i][J] - q0[q_i][J], and since Q has orthonormal columns the
// eigenvalue clamp of ref spd.py:6 commutes: H⁺ = Q (BᵀKB)⁺ Qᵀ. The
// R = 3(NS-1) core M = BᵀKB and the core gradient ĝ = Bᵀ g_var are formed in
// registers, projected (psd_project<R>), and expanded straight into the packed
// output — same operator as projecting the 12x12 stencil Hessian.
// ---------------------------------------------------------------------------
IPC_HD double helm(int a, int J) {  // q0[a][J]: a < NS, J < NS-1
  const double nrm = J == 0 ? 0.70710678118654752440 : (J == 1 ? 0.40824829046386301637 : 0.28867513459481288225);
  return a <= J ? nrm : (a == J + 1 ? -(double)(J + 1) * nrm : 0.0);
}

// β of NV difference vars (p[i], q[i]: local slot indices) over NB = NS-1 Helmert vectors
template <int NV, int NB>
IPC_HD void helm_beta(const int (&p)[NV], const int (&q)[NV], double (&beta)[NV][NB]) {
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int J = 0; J < NB; ++J) beta[i][J] = helm(p[i], J) - helm(q[i], J);
}

// gh[3J+c] = Σ_i β[i][J] gv[i].c
template <int NV, int NB>
IPC_HD void helm_grad(const double (&beta)[NV][NB], const V3 (&gv)[NV], double (&gh)[3 * NB]) {
#pragma unroll
  for (int J = 0; J < NB; ++J) {
    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      a += beta[i][J] * gv[i].x;
      b += beta[i][J] * gv[i].y;
      c += beta[i][J] * gv[i].z;
    }
    gh[3 * J] = a;
    gh[3 * J + 1] = b;
    gh[3 * J + 2] = c;
  }
}

// M (R x R, upper triangle) += s · Σ_ij β[i][I] β[j][J] hv[i][j]
template <int NV, int NB>
IPC_HD void helm_hess_acc(const double (&beta)[NV][NB], const M3 (&hv)[NV][NV], double s, double* M) {
  constexpr int R = 3 * NB;
#pragma unroll
  for (int I = 0; I < NB; ++I)
#pragma unroll
    for (int J = I; J < NB; ++J)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          if (I == J && d < c) continue;
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            double bi = beta[i][I];
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < NV; ++j) t += beta[j][J] * hv[i][j].m[3 * c + d];
            acc += bi * t;
          }
          M[(3 * I + c) * R + 3 * J + d] += s * acc;
        }
}

// M (upper) += s · a bᵀ (+ s · b aᵀ when sym2), core vectors of length R
template <int R>
IPC_HD void helm_outer_acc(const double (&a)[R], const double (&b)[R], double s, bool sym2, double* M) {
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = r; c < R; ++c) M[r * R + c] += sym2 ? s * (a[r] * b[c] + b[r] * a[c]) : s * (a[r] * b[c]);
}

// expand the projected core into the stencil outputs: g12 = Q ĝ,
// hp (packed 12x12 upper) = Q M⁺ Qᵀ; sl[a]: stencil slot of local slot a.
// Rows of inactive slots are zero (written first when NS < 4).
template <int NS>
IPC_HD void helm_out(const int (&sl)[NS], const double* gh, const double* M, double* g12, double* hp) {
  constexpr int NB = NS - 1, R = 3 * NB;
  if (NS < 4) {
#pragma unroll
    for (int i = 0; i < 12; ++i) g12[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 78; ++i) hp[i] = 0.0;
  }
#pragma unroll
  for (int a = 0; a < NS; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int J = 0; J < NB; ++J) acc += helm(a, J) * gh[3 * J + c];
      g12[3 * sl[a] + c] = acc;
    }
#pragma unroll
  for (int a = 0; a < NS; ++a)
#pragma unroll
    for (int b = 0; b < NS; ++b)
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          int r = 3 * sl[a] + i, c = 3 * sl[b] + j;
          if (c < r) continue;  // upper triangle of the stencil matrix
          double acc = 0.0;
#pragma unroll
          for (int I = 0; I < NB; ++I) {
            double t = 0.0;
#pragma unroll
            for (int J = 0; J < NB; ++J) {
              int u = 3 * I + i, v = 3 * J + j;
              t += helm(b, J) * (u <= v ? M[u * R + v] : M[v * R + u]);
            }
            acc += helm(a, I) * t;
          }
          hp[r * 12 - (r * (r - 1)) / 2 + (c - r)] = acc;
        }
}

// var-space derivatives of the reduced squared-distance formulas (the
// closed forms of d2_pp / d2_pl / d2_pf / d2_ll above, without the scatter);
// each returns the value in the same operation order as the value pass
IPC_HD double vs_pp(V3 d, V3 (&gv)[1], M3 (&hv)[1][1]) {
  gv[0] = 2.0 * d;
  hv[0][0] = m3_zero();
  m3_add_diag(hv[0][0], 2.0);
  return dotx(d, d);
}
IPC_HD double vs_pl(V3 w, V3 e, V3 (&gv)[2], M3 (&hv)[2][2]) {
  V3 c = crossx(e, w);
  double n = dotx(e, e);
  double val = __ddiv_rn(dotx(c, c), n);
  double t = dot(e, w) / n;
  V3 r = w - t * e;
  V3 k = r - t * e;
  gv[0] = 2.0 * r;
  gv[1] = (-2.0 * t) * r;
  M3 hww = m3_outer(e, e);
  for (int i = 0; i < 9; ++i) hww.m[i] *= -2.0 / n;
  m3_add_diag(hww, 2.0);
  M3 hwe = m3_outer(e, k);
  for (int i = 0; i < 9; ++i) hwe.m[i] *= -2.0 / n;
  m3_add_diag(hwe, -2.0 * t);
  M3 hee = m3_outer(k, k);
  for (int i = 0; i < 9; ++i) hee.m[i] *= -2.0 / n;
  m3_add_diag(hee, 2.0 * t * t);
  hv[0][0] = hww; hv[0][1] = hwe; hv[1][0] = m3_T(hwe); hv[1][1] = hee;
  return val;
}
IPC_HD double vs_triple(V3 w, V3 u, V3 v, V3 (&gv)[3], M3 (&hv)[3][3]) {
  triple_vars(w, u, v, gv, hv);
  V3 n = crossx(u, v);
  double q = dotx(w, n);
  return __ddiv_rn(__dmul_rn(q, q), dotx(n, n));
}
// c = |u x v|², u = x1 - x0, v = x3 - x2 (EE mollifier argument)
IPC_HD void vs_cross2(V3 u, V3 v, V3 (&gv)[2], M3 (&hv)[2][2]) {
  double uu = dot(u, u), vv = dot(v, v), uv = dot(u, v);
  gv[0] = 2.0 * (vv * u - uv * v);
  gv[1] = 2.0 * (uu * v - uv * u);
  M3 huu = m3_outer(v, v);
  for (int i = 0; i < 9; ++i) huu.m[i] *= -2.0;
  m3_add_diag(huu, 2.0 * vv);
  M3 hvv = m3_outer(u, u);
  for (int i = 0; i < 9; ++i) hvv.m[i] *= -2.0;
  m3_add_diag(hvv, 2.0 * uu);
  M3 huv = m3_outer(u, v), t2 = m3_outer(v, u);
  for (int i = 0; i < 9; ++i) huv.m[i] = 4.0 * huv.m[i] - 2.0 * t2.m[i];
  m3_add_diag(huv, -2.0 * uv);
  hv[0][0] = huu; hv[0][1] = huv; hv[1][0] = m3_T(huv); hv[1][1] = hvv;
}

// ---------------------------------------------------------------------------
// hyperelastic models: psi(F), P = dpsi/dF, H9 = d2psi/dF2 (F row-major,
// flat index 3i+j). Ref elastic.py:23-167.
// ---------------------------------------------------------------------------
enum { MODEL_NH = 0, MODEL_STVK = 1, MODEL_FCR = 2 };

IPC_HD M3 m3_inv_T(const M3& f, double det) {  // F^{-T} = cof(F)/det
  M3 c;
  c.m[0] = (f.m[4] * f.m[8] - f.m[5] * f.m[7]) / det;
  c.m[1] = (f.m[5] * f.m[6] - f.m[3] * f.m[8]) / det;
  c.m[2] = (f.m[3] * f.m[7] - f.m[4] * f.m[6]) / det;
  c.m[3] = (f.m[2] * f.m[7] - f.m[1] * f.m[8]) / det;
  c.m[4] = (f.m[0] * f.m[8] - f.m[2] * f.m[6]) / det;
  c.m[5] = (f.m[1] * f.m[6] - f.m[0] * f.m[7]) / det;
  c.m[6] = (f.m[1] * f.m[5] - f.m[2] * f.m[4]) / det;
  c.m[7] = (f.m[2] * f.m[3] - f.m[0] * f.m[5]) / det;
  c.m[8] = (f.m[0] * f.m[4] - f.m[1] * f.m[3]) / det;
  return c;
}

// value only; returns +inf for NeoHookean at det F <= 0
IPC_HD double nh_psi(const M3& f, double mu, double lam) {
  double j = m3_det(f);
  if (!(j > 0.0)) return INFINITY;
  double ic = 0.0;
  for (int i = 0; i < 9; ++i) ic += f.m[i] * f.m[i];
  double lj = log(j);
  return 0.5 * mu * (ic - 3.0) - mu * lj + 0.5 * lam * lj * lj;
}
IPC_HD double stvk_psi(const M3& f, double mu, double lam) {
  M3 e = m3_tmul(f, f);
  m3_add_diag(e, -1.0);
  for (int i = 0; i < 9; ++i) e.m[i] *= 0.5;
  double tr = e.m[0] + e.m[4] + e.m[8], ee = 0.0;
  for (int i = 0; i < 9; ++i) ee += e.m[i] * e.m[i];
  return mu * ee + 0.5 * lam * tr * tr;
}

// symmetric 3x3 eigen decomposition by Jacobi: a = V diag(w) V^T, w descending
IPC_HD void sym3_eig(const M3& A, double w[3], M3& V) {
  double a[9];
  for (int i = 0; i < 9; ++i) a[i] = A.m[i];
  V = m3_zero();
  m3_add_diag(V, 1.0);
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
    if (off < 1e-36 * (a[0] * a[0] + a[4] * a[4] + a[8] * a[8]) || off == 0.0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double apq = a[p * 3 + q];
        if (apq == 0.0) continue;
        double theta = (a[q * 3 + q] - a[p * 3 + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {
          double akp = a[k * 3 + p], akq = a[k * 3 + q];
          a[k * 3 + p] = c * akp - s * akq;
          a[k * 3 + q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = a[p * 3 + k], aqk = a[q * 3 + k];
          a[p * 3 + k] = c * apk - s * aqk;
          a[q * 3 + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          double vkp = V.m[k * 3 + p], vkq = V.m[k * 3 + q];
          V.m[k * 3 + p] = c * vkp - s * vkq;
          V.m[k * 3 + q] = s * vkp + c * vkq;
        }
      }
  }
  w[0] = a[0]; w[1] = a[4]; w[2] = a[8];
  // sort descending with columns of V
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2 - i; ++j)
      if (w[j] < w[j + 1]) {
        double t = w[j]; w[j] = w[j + 1]; w[j + 1] = t;
        for (int k = 0; k < 3; ++k) {
          double tv = V.m[k * 3 + j]; V.m[k * 3 + j] = V.m[k * 3 + j + 1]; V.m[k * 3 + j + 1] = tv;
        }
      }
}

// polar F = R S with the reference's reflection convention (ref elastic.py:39)
IPC_HD void polar(const M3& f, M3& R, M3& S) {
  M3 ftf = m3_tmul(f, f);
  double w[3];
  M3 V;
  sym3_eig(ftf, w, V);
  double sig[3];
  for (int i = 0; i < 3; ++i) sig[i] = sqrt(fmax(w[i], 0.0));
  // U columns = F v_i / sigma_i (third from cross product for robustness)
  V3 v0 = v3(V.m[0], V.m[3], V.m[6]), v1 = v3(V.m[1], V.m[4], V.m[7]), v2 = v3(V.m[2], V.m[5], V.m[8]);
  if (m3_det(V) < 0) { v2 = -1.0 * v2; V.m[2] = v2.x; V.m[5] = v2.y; V.m[8] = v2.z; }
  auto fv = [&](V3 v) {
    return v3(f.m[0] * v.x + f.m[1] * v.y + f.m[2] * v.z, f.m[3] * v.x + f.m[4] * v.y + f.m[5] * v.z,
              f.m[6] * v.x + f.m[7] * v.y + f.m[8] * v.z);
  };
  V3 u0 = (1.0 / sig[0]) * fv(v0);
  V3 u1 = (1.0 / sig[1]) * fv(v1);
  V3 u2 = cross(u0, u1);  // proper rotation U (det +1)
  // sign of the third singular value: F v2 = s2 u2
  double s2 = dot(fv(v2), u2);
  sig[2] = s2;  // negative when det F < 0: reflection folded into the smallest value
  M3 U;
  U.m[0] = u0.x; U.m[1] = u1.x; U.m[2] = u2.x;
  U.m[3] = u0.y; U.m[4] = u1.y; U.m[5] = u2.y;
  U.m[6] = u0.z; U.m[7] = u1.z; U.m[8] = u2.z;
  R = m3_mul(U, m3_T(V));
  S = m3_zero();
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += V.m[i * 3 + k] * sig[k] * V.m[j * 3 + k];
      S.m[i * 3 + j] = s;
    }
}

// PSD projection of the orthogonality Hessian ∂²/∂A² of c‖AAᵀ−I‖²_F (ref
// terms.py:66-79, projected at :101) in closed form. The energy is
// isotropic in A's singular values, E = c Σ(σᵢ²−1)², so its 9x9 Hessian has
// the eigensystem (signed SVD A = U Σ Vᵀ, U, V proper):
//   scaling  vec(uᵢvᵢᵀ)                 λ = c(12σᵢ² − 4)
//   twist    vec(uᵢvⱼᵀ − uⱼvᵢᵀ)/√2      λ = 4c(σᵢ² − σᵢσⱼ + σⱼ² − 1)
//   flip     vec(uᵢvⱼᵀ + uⱼvᵢᵀ)/√2      λ = 4c(σᵢ² + σᵢσⱼ + σⱼ² − 1)
// (polynomial eigenvalues: no divided differences, stable at σᵢ = σⱼ).
// out = Σ max(λ, 0) q qᵀ equals the eigenvalue clamp of the explicit Hessian
// to ~1e-14 relative (checked in tests), at ~1/20 of the cost.
IPC_HD void ortho_hess_psd(const M3& A, double c, double* h9) {
  M3 ata = m3_tmul(A, A);
  double w[3];
  M3 V;
  sym3_eig(ata, w, V);
  if (m3_det(V) < 0) {
    V.m[2] = -V.m[2]; V.m[5] = -V.m[5]; V.m[8] = -V.m[8];
  }
  double s[3];
  for (int i = 0; i < 3; ++i) s[i] = sqrt(fmax(w[i], 0.0));
  auto av = [&](int k) {
    return v3(A.m[0] * V.m[k] + A.m[1] * V.m[3 + k] + A.m[2] * V.m[6 + k],
              A.m[3] * V.m[k] + A.m[4] * V.m[3 + k] + A.m[5] * V.m[6 + k],
              A.m[6] * V.m[k] + A.m[7] * V.m[3 + k] + A.m[8] * V.m[6 + k]);
  };
  V3 u[3];
  u[0] = (1.0 / fmax(s[0], 1e-300)) * av(0);
  u[1] = (1.0 / fmax(s[1], 1e-300)) * av(1);
  u[2] = cross(u[0], u[1]);
  s[2] = dot(av(2), u[2]);
  V3 v[3] = {v3(V.m[0], V.m[3], V.m[6]), v3(V.m[1], V.m[4], V.m[7]), v3(V.m[2], V.m[5], V.m[8])};
  for (int i = 0; i < 81; ++i) h9[i] = 0.0;
  double q[9];
  auto add = [&](double lam) {
    if (!(lam > 0.0)) return;
    for (int a = 0; a < 9; ++a)
      for (int b = 0; b < 9; ++b) h9[9 * a + b] += lam * q[a] * q[b];
  };
  for (int i = 0; i < 3; ++i) {
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) q[3 * a + b] = at(u[i], a) * at(v[i], b);
    add(c * (12.0 * s[i] * s[i] - 4.0));
  }
  const double r2 = 0.70710678118654752440;
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j) {
      double base = s[i] * s[i] + s[j] * s[j] - 1.0, cross_ = s[i] * s[j];
      for (int sgn = -1; sgn <= 1; sgn += 2) {
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            q[3 * a + b] = r2 * (at(u[i], a) * at(v[j], b) + sgn * at(u[j], a) * at(v[i], b));
        add(4.0 * c * (base + sgn * cross_));
      }
    }
}

IPC_HD double fcr_psi(const M3& f, double mu, double lam) {
  M3 R, S;
  polar(f, R, S);
  double j = m3_det(f), d = 0.0;
  for (int i = 0; i < 9; ++i) d += (f.m[i] - R.m[i]) * (f.m[i] - R.m[i]);
  return mu * d + 0.5 * lam * (j - 1.0) * (j - 1.0);
}

IPC_HD double psi_value(int model, const M3& f, double mu, double lam) {
  if (model == MODEL_NH) return nh_psi(f, mu, lam);
  if (model == MODEL_STVK) return stvk_psi(f, mu, lam);
  return fcr_psi(f, mu, lam);
}

IPC_HD double levi(int i, int j, int k) {
  return (double)((i - j) * (j - k) * (k - i)) / 2.0;
}

// psi, P (9), H9 (81). Returns false when NeoHookean is inverted.
IPC_HD bool psi_derivs(int model, const M3& f, double mu, double lam, double* psi, double* P, double* H9) {
  if (model == MODEL_NH) {
    double j = m3_det(f);
    if (!(j > 0.0)) return false;
    *psi = nh_psi(f, mu, lam);
    double lj = log(j);
    M3 b = m3_inv_T(f, j);
    for (int i = 0; i < 9; ++i) P[i] = mu * f.m[i] + (lam * lj - mu) * b.m[i];
    double c = mu - lam * lj;
    for (int i = 0; i < 3; ++i)
      for (int jj = 0; jj < 3; ++jj)
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) {
            double h = c * b.m[3 * i + l] * b.m[3 * k + jj] + lam * b.m[3 * i + jj] * b.m[3 * k + l];
            if (i == k && jj == l) h += mu;
            H9[(3 * i + jj) * 9 + 3 * k + l] = h;
          }
    return true;
  }
  if (model == MODEL_STVK) {
    *psi = stvk_psi(f, mu, lam);
    M3 e = m3_tmul(f, f);
    m3_add_diag(e, -1.0);
    for (int i = 0; i < 9; ++i) e.m[i] *= 0.5;
    double tr = e.m[0] + e.m[4] + e.m[8];
    M3 s2 = e;
    for (int i = 0; i < 9; ++i) s2.m[i] *= 2.0 * mu;
    m3_add_diag(s2, lam * tr);
    M3 p = m3_mul(f, s2);
    for (int i = 0; i < 9; ++i) P[i] = p.m[i];
    M3 fft = m3_mul(f, m3_T(f));
    for (int i = 0; i < 3; ++i)
      for (int jj = 0; jj < 3; ++jj)
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) {
            double h = mu * f.m[3 * i + l] * f.m[3 * k + jj] + lam * f.m[3 * i + jj] * f.m[3 * k + l];
            if (i == k) h += s2.m[3 * l + jj];
            if (jj == l) h += mu * fft.m[3 * i + k];
            H9[(3 * i + jj) * 9 + 3 * k + l] = h;
          }
    return true;
  }
  // fixed corotated
  M3 R, S;
  polar(f, R, S);
  double j = m3_det(f);
  double d = 0.0;
  for (int i = 0; i < 9; ++i) d += (f.m[i] - R.m[i]) * (f.m[i] - R.m[i]);
  *psi = mu * d + 0.5 * lam * (j - 1.0) * (j - 1.0);
  // cofactor: column c = cross of the other two columns
  V3 c0 = v3(f.m[0], f.m[3], f.m[6]), c1 = v3(f.m[1], f.m[4], f.m[7]), c2 = v3(f.m[2], f.m[5], f.m[8]);
  V3 g0 = cross(c1, c2), g1 = cross(c2, c0), g2 = cross(c0, c1);
  M3 g;
  g.m[0] = g0.x; g.m[1] = g1.x; g.m[2] = g2.x;
  g.m[3] = g0.y; g.m[4] = g1.y; g.m[5] = g2.y;
  g.m[6] = g0.z; g.m[7] = g1.z; g.m[8] = g2.z;
  for (int i = 0; i < 9; ++i) P[i] = 2.0 * mu * (f.m[i] - R.m[i]) + lam * (j - 1.0) * g.m[i];
  // dR/dF (ref elastic.py:129): (tr S I - S) w = axl-type rhs per basis dF = e_kl
  M3 M = S;
  for (int i = 0; i < 9; ++i) M.m[i] = -M.m[i];
  m3_add_diag(M, S.m[0] + S.m[4] + S.m[8]);
  double detM = m3_det(M);
  M3 Minv = m3_T(m3_inv_T(M, detM));
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l) {
      // A = R^T e_kl: column l equals R[k, :]
      double A[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int r = 0; r < 3; ++r) A[3 * r + l] = R.m[3 * k + r];
      V3 rhs = v3(A[7] - A[5], A[2] - A[6], A[3] - A[1]);
      V3 w = v3(Minv.m[0] * rhs.x + Minv.m[1] * rhs.y + Minv.m[2] * rhs.z,
                Minv.m[3] * rhs.x + Minv.m[4] * rhs.y + Minv.m[5] * rhs.z,
                Minv.m[6] * rhs.x + Minv.m[7] * rhs.y + Minv.m[8] * rhs.z);
      M3 dR = m3_mul(R, m3_skew(w));
      for (int i = 0; i < 3; ++i)
        for (int jj = 0; jj < 3; ++jj) {
          int row = 3 * i + jj, col = 3 * k + l;
          double h = -2.0 * mu * dR.m[3 * i + jj] + lam * g.m[row] * g.m[col];
          if (row == col) h += 2.0 * mu;
          // lam (J-1) d cof_ij / dF_kl = eps_ikm eps_jlq F_mq
          double dc = 0.0;
          for (int m = 0; m < 3; ++m)
            for (int q = 0; q < 3; ++q) dc += levi(i, k, m) * levi(jj, l, q) * f.m[3 * m + q];
          h += lam * (j - 1.0) * dc;
          H9[row * 9 + col] = h;
        }
    }
  return true;
}

}  // namespace ipc
