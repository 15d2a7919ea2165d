// Penetrated-grasp repair geometry on the GPU (ref pkg/src/srsim/robot/
// repair.py:98-113 and robot/proximity.py): generalized winding numbers,
// crossing-triangle counts, maximum penetration depth, and the batched
// retraction probe search.
//
// Layout: a batch of E independent repair problems, flattened with per-env
// prefix arrays (include/ipc_b200.h ipc_repair_desc). Each env is owned by one
// CTA: the retraction search evaluates a window of probe distances at once
// (every crossing-pair / containment test of every probe in the window is an
// independent item spread over the CTA's threads), stops at the first window
// that holds a clear probe and reports the first clear probe in it — the
// reference's sequential probe loop returns the same index because probes are
// independent.
//
// Exactness: the segment/triangle test, box filter, point-triangle distance
// and the solid-angle terms use round-to-nearest intrinsics in numpy's
// operation order (no FMA contraction), so decisions on identical inputs
// match the CPU path; atan2 and the per-point sum order are the only
// deviations (≤ a few ulp on a winding number that is thresholded at 0.5).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ipc_b200.h"
#include "ipc_math.cuh"

using namespace ipc;

extern "C" int ipc__set_error(const char* msg);  // engine.cu

#define RCK(call)                                                                    \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw std::runtime_error(std::string(#call) + ": " + cudaGetErrorString(e_));  \
  } while (0)

#define RGUARD(...)                                   \
  try {                                               \
    __VA_ARGS__;                                      \
    return 0;                                         \
  } catch (const std::exception& ex) {                \
    return ipc__set_error(ex.what());                 \
  }

namespace ipc_repair {

constexpr double kSegEps = 1e-14;     // ref proximity.py:112
constexpr double kTwoPi = 6.283185307179586;
constexpr int kThreads = 256;
#ifndef RETRACT_WINDOW
#define RETRACT_WINDOW 1
#endif
constexpr int kMaxWindow = RETRACT_WINDOW;  // probes evaluated together after probe 0

// RAII device copy of a host array
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t n_) : n(n_) {
    if (n) RCK(cudaMalloc(&p, n * sizeof(T)));
  }
  DBuf(const T* h, size_t n_) : DBuf(n_) {
    if (n) RCK(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void get(T* h) const {
    if (n) RCK(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost));
  }
};

__device__ __forceinline__ V3 ldv(const double* __restrict__ v, int i) {
  return V3{__ldg(v + 3 * i), __ldg(v + 3 * i + 1), __ldg(v + 3 * i + 2)};
}

// ref proximity.py:110-125, numpy operation order
__device__ __forceinline__ bool seg_tri_hit(V3 o, V3 vec, V3 t0, V3 t1, V3 t2) {
  V3 e1 = t1 - t0, e2 = t2 - t0;
  V3 p = crossx(vec, e2);
  double det = dotx(e1, p);
  if (!(fabs(det) > kSegEps)) return false;
  double inv = __ddiv_rn(1.0, det);
  V3 s = o - t0;
  double u = __dmul_rn(dotx(s, p), inv);
  V3 q = crossx(s, e1);
  double v = __dmul_rn(dotx(vec, q), inv);
  double t = __dmul_rn(dotx(e2, q), inv);
  return u >= 0 && v >= 0 && __dadd_rn(u, v) <= 1 && t >= 0 && t <= 1;
}

// ref proximity.py:146-160: any edge of one triangle through the other
__device__ __forceinline__ bool tri_tri_hit(const V3 (&a)[3], const V3 (&b)[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    int i = k, j = (k + 1) % 3;
    if (seg_tri_hit(a[i], a[j] - a[i], b[0], b[1], b[2])) return true;
    if (seg_tri_hit(b[i], b[j] - b[i], a[0], a[1], a[2])) return true;
  }
  return false;
}

__device__ __forceinline__ void tri_box(const V3 (&t)[3], V3& lo, V3& hi) {
  lo = V3{fmin(fmin(t[0].x, t[1].x), t[2].x), fmin(fmin(t[0].y, t[1].y), t[2].y),
          fmin(fmin(t[0].z, t[1].z), t[2].z)};
  hi = V3{fmax(fmax(t[0].x, t[1].x), t[2].x), fmax(fmax(t[0].y, t[1].y), t[2].y),
          fmax(fmax(t[0].z, t[1].z), t[2].z)};
}

// closed-box overlap, margin 0 (ref bvh.py:118,128)
__device__ __forceinline__ bool boxes_overlap(V3 alo, V3 ahi, V3 blo, V3 bhi) {
  return alo.x <= bhi.x && ahi.x >= blo.x && alo.y <= bhi.y && ahi.y >= blo.y &&
         alo.z <= bhi.z && ahi.z >= blo.z;
}

// one solid-angle term of ref proximity.py:196-206 (van Oosterom–Strackee)
__device__ __forceinline__ double solid_angle(V3 p, V3 A, V3 B, V3 C) {
  V3 a = A - p, b = B - p, c = C - p;
  double la = __dsqrt_rn(dotx(a, a)), lb = __dsqrt_rn(dotx(b, b)), lc = __dsqrt_rn(dotx(c, c));
  double num = dotx(a, crossx(b, c));
  double den = __dmul_rn(__dmul_rn(la, lb), lc);
  den = __dadd_rn(den, __dmul_rn(dotx(a, b), lc));
  den = __dadd_rn(den, __dmul_rn(dotx(b, c), la));
  den = __dadd_rn(den, __dmul_rn(dotx(c, a), lb));
  return atan2(num, den);
}

// winding number of p w.r.t. triangles [t0, t1) of (v, t); vertices shifted by -d
__device__ double winding(V3 p, const double* __restrict__ v, const int32_t* __restrict__ t,
                          int t0, int t1, int vbase, V3 d, bool shift) {
  double w = 0.0;
  for (int j = t0; j < t1; ++j) {
    V3 A = ldv(v, vbase + __ldg(t + 3 * j)), B = ldv(v, vbase + __ldg(t + 3 * j + 1)),
       C = ldv(v, vbase + __ldg(t + 3 * j + 2));
    if (shift) {
      A = A - d;
      B = B - d;
      C = C - d;
    }
    w += solid_angle(p, A, B, C);
  }
  return w / kTwoPi;
}

__device__ __forceinline__ V3 shifted(V3 a, double r, V3 n) {
  // probe translation t - r*n (ref repair.py:105), applied to world vertices
  return V3{__dsub_rn(a.x, __dmul_rn(r, n.x)), __dsub_rn(a.y, __dmul_rn(r, n.y)),
            __dsub_rn(a.z, __dmul_rn(r, n.z))};
}

struct RepairDev {
  int n_env, n_probe;
  const int32_t *env_link, *link_vert, *link_tri, *hand_t, *env_ov, *env_ot, *obj_t;
  const double *hand_v, *obj_v, *normal, *retr;
};

// Containment shortcut: the winding number of a closed surface is 0 at every
// point outside the surface's bounding box (it is 0 outside the solid), so a
// point outside the box (with a 1e-9 m guard against rounding) is decided
// "not inside" without evaluating it; the reference's thresholded decision
// (> 0.5) is unchanged.
constexpr double kBoxGuard = 1e-9;

__device__ __forceinline__ bool outside_box(V3 x, V3 lo, V3 hi) {
  return x.x < lo.x - kBoxGuard || x.x > hi.x + kBoxGuard || x.y < lo.y - kBoxGuard ||
         x.y > hi.y + kBoxGuard || x.z < lo.z - kBoxGuard || x.z > hi.z + kBoxGuard;
}

// block-wide bounding box of vertices [v0, v1) of v (all threads call)
__device__ void block_box(const double* __restrict__ v, int v0, int v1, V3& lo, V3& hi) {
  __shared__ double red[6][kThreads / 32];
  double a[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
    V3 x = ldv(v, i);
    a[0] = fmin(a[0], x.x), a[1] = fmin(a[1], x.y), a[2] = fmin(a[2], x.z);
    a[3] = fmax(a[3], x.x), a[4] = fmax(a[4], x.y), a[5] = fmax(a[5], x.z);
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    for (int o = 16; o; o >>= 1) {
      double b = __shfl_xor_sync(0xffffffffu, a[c], o);
      a[c] = c < 3 ? fmin(a[c], b) : fmax(a[c], b);
    }
    if ((threadIdx.x & 31) == 0) red[c][threadIdx.x >> 5] = a[c];
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int c = threadIdx.x;
    double m = red[c][0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = c < 3 ? fmin(m, red[c][w]) : fmax(m, red[c][w]);
    red[c][0] = m;
  }
  __syncthreads();
  lo = V3{red[0][0], red[1][0], red[2][0]};
  hi = V3{red[3][0], red[4][0], red[5][0]};
  __syncthreads();
}

constexpr int kMaxLinks = 32;
// triangle boxes staged in shared memory when an env fits (hand at probe 0,
// object); larger envs test boxes from the vertices in global memory
constexpr int kStageHT = 128, kStageOT = 448;  // 128: the three-finger hand has 84 triangles

// ref repair.py:103-113 for one env per CTA; out[e] = first clear probe or n_probe.
// Items of one probe, crossing pairs first (cheap, box-filtered, and the
// usual reason a probe is rejected — a hit flags the probe and its remaining
// items, including the winding numbers, are skipped), then hand-vertex
// containment, then link-swallows-object containment.
#ifndef RETRACT_MIN_BLOCKS
#define RETRACT_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kThreads, RETRACT_MIN_BLOCKS) k_repair_retract(RepairDev D, int32_t* out) {
  const int e = blockIdx.x;
  __shared__ int flag[kMaxWindow];
  __shared__ int s_found;
  __shared__ double s_d[kMaxWindow][3];  // rn(r_k * n) of the window's probes
  __shared__ double s_lbox[kMaxLinks][6];
  __shared__ double s_hbox[kStageHT][6];
  __shared__ double s_obox[kStageOT][6];
  // one-probe rounds: hand triangles whose translated box meets the object's
  // box (no other hand triangle can overlap any object triangle box)
  __shared__ int s_act[kStageHT];
  __shared__ int s_nact;
  const int l0 = D.env_link[e], l1 = D.env_link[e + 1];
  const int hv0 = D.link_vert[l0], hv1 = D.link_vert[l1];
  const int ht0 = D.link_tri[l0], ht1 = D.link_tri[l1];
  const int ov0 = D.env_ov[e], ov1 = D.env_ov[e + 1], ot0 = D.env_ot[e], ot1 = D.env_ot[e + 1];
  const int HT = ht1 - ht0, HV = hv1 - hv0, NL = l1 - l0, NOT = ot1 - ot0;
  const V3 n = V3{D.normal[3 * e], D.normal[3 * e + 1], D.normal[3 * e + 2]};
  const int n_cross = HT * NOT;
  const bool staged = HT <= kStageHT && NOT <= kStageOT;
  V3 olo, ohi;
  block_box(D.obj_v, ov0, ov1, olo, ohi);
  // probe-0 link boxes (NL <= kMaxLinks: links beyond it are never boxed)
  for (int l = 0; l < min(NL, kMaxLinks); ++l) {
    V3 lo, hi;
    block_box(D.hand_v, D.link_vert[l0 + l], D.link_vert[l0 + l + 1], lo, hi);
    if (threadIdx.x == 0) {
      s_lbox[l][0] = lo.x, s_lbox[l][1] = lo.y, s_lbox[l][2] = lo.z;
      s_lbox[l][3] = hi.x, s_lbox[l][4] = hi.y, s_lbox[l][5] = hi.z;
    }
  }
  if (staged) {
    // box of a translated triangle == translated box: x -> rn(x - d) is monotone
    for (int i = threadIdx.x; i < HT + NOT; i += blockDim.x) {
      V3 t[3];
      const bool hand = i < HT;
      const int j = hand ? ht0 + i : ot0 + i - HT;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        t[c] = hand ? ldv(D.hand_v, __ldg(D.hand_t + 3 * j + c))
                    : ldv(D.obj_v, ov0 + __ldg(D.obj_t + 3 * j + c));
      V3 lo, hi;
      tri_box(t, lo, hi);
      double* b = hand ? s_hbox[i] : s_obox[i - HT];
      b[0] = lo.x, b[1] = lo.y, b[2] = lo.z, b[3] = hi.x, b[4] = hi.y, b[5] = hi.z;
    }
  }
  int k0 = 0, win = 1;
  if (threadIdx.x == 0) s_found = D.n_probe;
  while (k0 < D.n_probe) {
    const int W = min(win, D.n_probe - k0);
    if (threadIdx.x == 0) s_nact = 0;
    if (threadIdx.x < kMaxWindow) {
      flag[threadIdx.x] = 0;
      if ((int)threadIdx.x < W) {
        const double rk = D.retr[k0 + threadIdx.x];
        s_d[threadIdx.x][0] = __dmul_rn(rk, n.x);
        s_d[threadIdx.x][1] = __dmul_rn(rk, n.y);
        s_d[threadIdx.x][2] = __dmul_rn(rk, n.z);
      }
    }
    __syncthreads();
    constexpr bool kOne = kMaxWindow == 1;
    const bool compact = kOne && staged;
    if (compact) {
      if ((int)threadIdx.x < HT) {
        const double* hb = s_hbox[threadIdx.x];
        const double dx = s_d[0][0], dy = s_d[0][1], dz = s_d[0][2];
        if (__dsub_rn(hb[0], dx) <= ohi.x && __dsub_rn(hb[3], dx) >= olo.x &&
            __dsub_rn(hb[1], dy) <= ohi.y && __dsub_rn(hb[4], dy) >= olo.y &&
            __dsub_rn(hb[2], dz) <= ohi.z && __dsub_rn(hb[5], dz) >= olo.z)
          s_act[atomicAdd(&s_nact, 1)] = threadIdx.x;
      }
      __syncthreads();
    }
    const int n_cross_k = compact ? s_nact * NOT : n_cross;
    const int per_probe_k = n_cross_k + HV + NL;
    const int total = per_probe_k * W;
    for (int it = threadIdx.x; it < total; it += blockDim.x) {
      const int p = it / per_probe_k;
      if (*(volatile int*)&flag[p]) continue;
      const int r = it - p * per_probe_k;
      const double rr = D.retr[k0 + p];
      bool hit = false;
      if (r < n_cross_k) {
        // crossing triangle pair (ref repair.py:53, proximity.py:163)
        const int ic = r / NOT, jl = r - ic * NOT;
        const int il = compact ? s_act[ic] : ic;
        const int i = ht0 + il, j = ot0 + jl;
        if (staged) {
          const double* hb = s_hbox[il];
          const double* ob = s_obox[jl];
          const double dx = s_d[p][0], dy = s_d[p][1], dz = s_d[p][2];
          const bool ov = __dsub_rn(hb[0], dx) <= ob[3] && __dsub_rn(hb[3], dx) >= ob[0] &&
                          __dsub_rn(hb[1], dy) <= ob[4] && __dsub_rn(hb[4], dy) >= ob[1] &&
                          __dsub_rn(hb[2], dz) <= ob[5] && __dsub_rn(hb[5], dz) >= ob[2];
          if (!ov) continue;
        }
        V3 a[3], b[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          a[c] = shifted(ldv(D.hand_v, __ldg(D.hand_t + 3 * i + c)), rr, n);
          b[c] = ldv(D.obj_v, ov0 + __ldg(D.obj_t + 3 * j + c));
        }
        V3 alo, ahi, blo, bhi;
        tri_box(a, alo, ahi);
        tri_box(b, blo, bhi);
        hit = boxes_overlap(alo, ahi, blo, bhi) && tri_tri_hit(a, b);
      } else if (r < n_cross_k + HV) {
        // hand vertex contained in the object (ref repair.py:56)
        V3 x = shifted(ldv(D.hand_v, hv0 + (r - n_cross_k)), rr, n);
        hit = !outside_box(x, olo, ohi) &&
              winding(x, D.obj_v, D.obj_t, ot0, ot1, ov0, V3{0, 0, 0}, false) > 0.5;
      } else {
        // object's first vertex swallowed by a link (ref repair.py:59)
        const int li = r - n_cross_k - HV, l = l0 + li;
        V3 d = V3{__dmul_rn(rr, n.x), __dmul_rn(rr, n.y), __dmul_rn(rr, n.z)};
        V3 x = ldv(D.obj_v, ov0);
        bool skip = false;
        if (li < kMaxLinks) {
          V3 xs = x + d;  // the point in the link's probe-0 frame
          skip = outside_box(xs, V3{s_lbox[li][0], s_lbox[li][1], s_lbox[li][2]},
                             V3{s_lbox[li][3], s_lbox[li][4], s_lbox[li][5]});
        }
        if (!skip) {
          double w = 0.0;
          for (int j = D.link_tri[l]; j < D.link_tri[l + 1]; ++j) {
            V3 A = ldv(D.hand_v, __ldg(D.hand_t + 3 * j)),
               B = ldv(D.hand_v, __ldg(D.hand_t + 3 * j + 1)),
               C = ldv(D.hand_v, __ldg(D.hand_t + 3 * j + 2));
            A = V3{__dsub_rn(A.x, d.x), __dsub_rn(A.y, d.y), __dsub_rn(A.z, d.z)};
            B = V3{__dsub_rn(B.x, d.x), __dsub_rn(B.y, d.y), __dsub_rn(B.z, d.z)};
            C = V3{__dsub_rn(C.x, d.x), __dsub_rn(C.y, d.y), __dsub_rn(C.z, d.z)};
            w += solid_angle(x, A, B, C);
          }
          hit = w / kTwoPi > 0.5;
        }
      }
      if (hit) flag[p] = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int p = 0; p < W; ++p)
        if (!flag[p]) {
          s_found = k0 + p;
          break;
        }
    }
    __syncthreads();
    if (s_found < D.n_probe) break;
    k0 += W;
    win = kMaxWindow;
  }
  if (threadIdx.x == 0) out[e] = s_found;
}

// ref proximity.py:235-246 per env: max over contained points of the
// unsigned surface distance (ref :214), 0 if none is contained
__global__ void __launch_bounds__(kThreads) k_max_penetration(
    const int32_t* __restrict__ env_pt, const double* __restrict__ pts,
    const int32_t* __restrict__ env_ov, const int32_t* __restrict__ env_ot,
    const double* __restrict__ ov, const int32_t* __restrict__ ot, double* out) {
  const int e = blockIdx.x;
  const int p0 = env_pt[e], p1 = env_pt[e + 1], vb = env_ov[e], t0 = env_ot[e], t1 = env_ot[e + 1];
  V3 olo, ohi;
  block_box(ov, vb, env_ov[e + 1], olo, ohi);
  double best = 0.0;
  for (int i = p0 + threadIdx.x; i < p1; i += blockDim.x) {
    V3 x = ldv(pts, i);
    if (outside_box(x, olo, ohi)) continue;
    if (!(winding(x, ov, ot, t0, t1, vb, V3{0, 0, 0}, false) > 0.5)) continue;
    double d2 = INFINITY;
    for (int j = t0; j < t1; ++j) {
      V3 A = ldv(ov, vb + __ldg(ot + 3 * j)), B = ldv(ov, vb + __ldg(ot + 3 * j + 1)),
         C = ldv(ov, vb + __ldg(ot + 3 * j + 2));
      d2 = fmin(d2, pt_dist2(pt_region(x, A, B, C), x, A, B, C));
    }
    best = fmax(best, __dsqrt_rn(d2));
  }
  __shared__ double red[kThreads / 32];
  for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    out[e] = m;
  }
}

__global__ void k_winding(int64_t n, const double* __restrict__ pts, const double* __restrict__ v,
                          const int32_t* __restrict__ t, int nt, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = winding(ldv(pts, (int)i), v, t, 0, nt, 0, V3{0, 0, 0}, false);
}

// ref proximity.py:163: boxes of every (a, b) triangle pair, then the hit test
__global__ void k_count_crossings(const double* __restrict__ va, const int32_t* __restrict__ ta,
                                  int nta, const double* __restrict__ vb,
                                  const int32_t* __restrict__ tb, int ntb,
                                  unsigned long long* count) {
  unsigned long long c = 0;
  const int64_t total = (int64_t)nta * ntb;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(it / ntb), j = (int)(it % ntb);
    V3 a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      a[k] = ldv(va, __ldg(ta + 3 * i + k));
      b[k] = ldv(vb, __ldg(tb + 3 * j + k));
    }
    V3 alo, ahi, blo, bhi;
    tri_box(a, alo, ahi);
    tri_box(b, blo, bhi);
    c += boxes_overlap(alo, ahi, blo, bhi) && tri_tri_hit(a, b);
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// device time of the last retraction-search launch (CUDA events around the
// kernel on the launching stream; read by bench.py for the roofline)
double g_retract_ms = 0.0;

// grow-only device arena of the retraction entry point (calls are serialised)
struct Arena {
  std::mutex mu;
  char* p = nullptr;
  size_t cap = 0;
  char* reserve(size_t bytes) {
    if (bytes > cap) {
      if (p) RCK(cudaFree(p));
      p = nullptr;
      cap = 0;
      size_t want = bytes + bytes / 2;
      RCK(cudaMalloc(&p, want));
      cap = want;
    }
    return p;
  }
};
Arena g_arena;

int grid_for(int64_t n, int t) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, (int64_t)sms * 8));
}

}  // namespace ipc_repair

using namespace ipc_repair;

extern "C" {

int ipc_repair_retract(const ipc_repair_desc* d, int32_t* probe_index) {
  RGUARD({
    if (!d || d->n_env < 0 || d->n_probe < 0) throw std::runtime_error("bad repair descriptor");
    const int E = d->n_env;
    if (E == 0) return 0;
    const int L = d->env_link[E];
    const int HV = d->link_vert[L], HT = d->link_tri[L];
    const int OV = d->env_obj_vert[E], OT = d->env_obj_tri[E];
    // per-probe work items are 32-bit: (hand tris x object tris + points) of one env
    for (int e = 0; e < E; ++e) {
      const long long ht = d->link_tri[d->env_link[e + 1]] - d->link_tri[d->env_link[e]];
      const long long hv = d->link_vert[d->env_link[e + 1]] - d->link_vert[d->env_link[e]];
      const long long ot = d->env_obj_tri[e + 1] - d->env_obj_tri[e];
      if (ht * ot + hv + (d->env_link[e + 1] - d->env_link[e]) > (1LL << 30))
        throw std::runtime_error("repair env too large for one CTA's 32-bit probe item space");
    }
    // one grow-only device arena for every input (no per-call cudaMalloc/cudaFree)
    std::lock_guard<std::mutex> lock(g_arena.mu);
    size_t off = 0;
    auto slot = [&](size_t bytes) {
      size_t o = off;
      off += (bytes + 255) & ~size_t(255);
      return o;
    };
    const size_t o_el = slot(4 * (E + 1)), o_lv = slot(4 * (L + 1)), o_lt = slot(4 * (L + 1)),
                 o_ht = slot(12 * (size_t)HT), o_eov = slot(4 * (E + 1)), o_eot = slot(4 * (E + 1)),
                 o_ot = slot(12 * (size_t)OT), o_hv = slot(24 * (size_t)HV),
                 o_ov = slot(24 * (size_t)OV), o_n = slot(24 * (size_t)E),
                 o_r = slot(8 * (size_t)d->n_probe), o_out = slot(4 * (size_t)E);
    char* base = g_arena.reserve(off);
    auto up = [&](size_t o, const void* h, size_t bytes) {
      if (bytes) RCK(cudaMemcpyAsync(base + o, h, bytes, cudaMemcpyHostToDevice, 0));
    };
    up(o_el, d->env_link, 4 * (E + 1));
    up(o_lv, d->link_vert, 4 * (L + 1));
    up(o_lt, d->link_tri, 4 * (L + 1));
    up(o_ht, d->hand_t, 12 * (size_t)HT);
    up(o_eov, d->env_obj_vert, 4 * (E + 1));
    up(o_eot, d->env_obj_tri, 4 * (E + 1));
    up(o_ot, d->obj_t, 12 * (size_t)OT);
    up(o_hv, d->hand_v, 24 * (size_t)HV);
    up(o_ov, d->obj_v, 24 * (size_t)OV);
    up(o_n, d->normal, 24 * (size_t)E);
    up(o_r, d->retraction, 8 * (size_t)d->n_probe);
    auto I = [&](size_t o) { return reinterpret_cast<const int32_t*>(base + o); };
    auto F = [&](size_t o) { return reinterpret_cast<const double*>(base + o); };
    RepairDev D{E, d->n_probe, I(o_el), I(o_lv), I(o_lt), I(o_ht), I(o_eov), I(o_eot), I(o_ot),
                F(o_hv), F(o_ov), F(o_n), F(o_r)};
    int32_t* out_p = reinterpret_cast<int32_t*>(base + o_out);
    cudaEvent_t ev[2];
    RCK(cudaEventCreate(&ev[0]));
    RCK(cudaEventCreate(&ev[1]));
    RCK(cudaEventRecord(ev[0], 0));
    k_repair_retract<<<E, kThreads>>>(D, out_p);
    RCK(cudaGetLastError());
    RCK(cudaEventRecord(ev[1], 0));
    RCK(cudaMemcpy(probe_index, out_p, 4 * (size_t)E, cudaMemcpyDeviceToHost));
    float ms = 0.f;
    RCK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    g_retract_ms = ms;
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
  })
}

int ipc_repair_last_kernel_ms(double* ms) {
  if (!ms) return ipc__set_error("null output");
  *ms = g_retract_ms;
  return 0;
}

int ipc_max_penetration(int32_t n_env, const int32_t* env_pt, const double* pts,
                        const int32_t* env_obj_vert, const int32_t* env_obj_tri,
                        const double* obj_v, const int32_t* obj_t, double* out) {
  RGUARD({
    if (n_env <= 0) return 0;
    const int NP = env_pt[n_env], OV = env_obj_vert[n_env], OT = env_obj_tri[n_env];
    DBuf<int32_t> ept(env_pt, n_env + 1), eov(env_obj_vert, n_env + 1), eot(env_obj_tri, n_env + 1),
        t(obj_t, 3 * (size_t)OT);
    DBuf<double> p(pts, 3 * (size_t)NP), v(obj_v, 3 * (size_t)OV), o(n_env);
    k_max_penetration<<<n_env, kThreads>>>(ept.p, p.p, eov.p, eot.p, v.p, t.p, o.p);
    RCK(cudaGetLastError());
    o.get(out);
  })
}

int ipc_winding_numbers(int64_t n_pts, const double* pts, int32_t n_verts, const double* verts,
                        int32_t n_tris, const int32_t* tris, double* out) {
  RGUARD({
    if (n_pts <= 0) return 0;
    DBuf<double> p(pts, 3 * (size_t)n_pts), v(verts, 3 * (size_t)n_verts), o(n_pts);
    DBuf<int32_t> t(tris, 3 * (size_t)n_tris);
    k_winding<<<grid_for(n_pts, 128), 128>>>(n_pts, p.p, v.p, t.p, n_tris, o.p);
    RCK(cudaGetLastError());
    o.get(out);
  })
}

int ipc_count_mesh_intersections(int32_t nva, const double* va, int32_t nta, const int32_t* ta,
                                 int32_t nvb, const double* vb, int32_t ntb, const int32_t* tb,
                                 int64_t* count) {
  RGUARD({
    *count = 0;
    if (nta <= 0 || ntb <= 0) return 0;
    DBuf<double> a(va, 3 * (size_t)nva), b(vb, 3 * (size_t)nvb);
    DBuf<int32_t> at(ta, 3 * (size_t)nta), bt(tb, 3 * (size_t)ntb);
    DBuf<unsigned long long> c(1);
    RCK(cudaMemset(c.p, 0, sizeof(unsigned long long)));
    k_count_crossings<<<grid_for((int64_t)nta * ntb, 256), 256>>>(a.p, at.p, nta, b.p, bt.p, ntb, c.p);
    RCK(cudaGetLastError());
    unsigned long long h = 0;
    c.get(&h);
    *count = (int64_t)h;
  })
}

}  // extern "C"
