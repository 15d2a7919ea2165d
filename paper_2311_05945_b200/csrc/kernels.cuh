// Kernels of the batched IPC time step. See DESIGN.md for the data flow.
#pragma once
#include <climits>
#include "ipc_math.cuh"
#include "lbvh.cuh"
#include "world.cuh"

namespace ipc {

constexpr int PK = 78;  // packed upper triangle of a 12x12 block

IPC_HD int pk(int i, int j) {  // i <= j
  return i * 12 - (i * (i - 1)) / 2 + (j - i);
}
IPC_HD double pk_get(const double* h, int i, int j) { return i <= j ? h[pk(i, j)] : h[pk(j, i)]; }

IPC_HD void atomic_min_pos(double* addr, double v) {
  // non-negative doubles order like their int64 bit patterns
  atomicMin(reinterpret_cast<long long*>(addr), __double_as_longlong(v));
}

// ---------------------------------------------------------------------------
// world-space slot positions: soft slots copy their DoF, affine slots
// p + A x0 with numpy's operation order (ref contact.py:296)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void world_slot(const World& W, const double* __restrict__ x, double* __restrict__ xw,
                                           int s) {
  int d = W.slot_dof[s];
  if (!W.slot_aff[s]) {
    xw[3 * s] = x[d];
    xw[3 * s + 1] = x[d + 1];
    xw[3 * s + 2] = x[d + 2];
    return;
  }
  const double* r = W.slot_rest + 3 * s;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double* a = x + d + 3 + 3 * i;
    double m = __dadd_rn(__dadd_rn(__dmul_rn(a[0], r[0]), __dmul_rn(a[1], r[1])), __dmul_rn(a[2], r[2]));
    xw[3 * s + i] = __dadd_rn(x[d + i], m);
  }
}

IPC_GLOBAL void k_world(World W, const double* __restrict__ x, double* __restrict__ xw) {
  ipc_pdl_wait();
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < W.n_slot) world_slot(W, x, xw, s);
}


// out = a + (scale * alpha_e) * b over DoFs of flagged envs (others copy a);
// scale is a power of two, so scale * alpha equals repeated halving exactly
IPC_GLOBAL void k_axpy_env(World W, const double* a, const double* b, const double* alpha, double scale,
                           const int* flag, double* out) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W.n_dof) return;
  int e = W.dof_env[i];
  out[i] = (flag == nullptr || flag[e]) ? __dadd_rn(a[i], __dmul_rn(alpha ? alpha[e] * scale : 1.0, b[i])) : a[i];
}

IPC_GLOBAL void k_sub(int n, const double* a, const double* b, double* out) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __dsub_rn(a[i], b[i]);
}

// ---------------------------------------------------------------------------
// broad phase: exhaustive box tests, one CTA per environment, ordered
// compaction (lexicographic output, ref broadphase.py:162-166). Boxes:
// query box [lo, hi] vs primitive box inflated by `margin` (ref bvh.py:87-88, :129-130).
// ---------------------------------------------------------------------------
template <int NT>
static __device__ int block_ordered_offset(bool hit, int* warp_tot, int* total) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned m = __ballot_sync(0xffffffffu, hit);
  int pre = __popc(m & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[wid] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < NT / 32; ++w) {
      int t = warp_tot[w];
      warp_tot[w] = acc;
      acc += t;
    }
    *total = acc;
  }
  __syncthreads();
  return warp_tot[wid] + pre;
}

__device__ __forceinline__ bool box_hit(const double* qlo, const double* qhi, const double* plo,
                                        const double* phi, double margin) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double pmin = __dsub_rn(plo[c], margin), pmax = __dadd_rn(phi[c], margin);
    if (!(qlo[c] <= pmax && qhi[c] >= pmin)) return false;
  }
  return true;
}


__device__ __forceinline__ bool excluded(const World& W, int cb0, int b1, int b2) {
  unsigned long long m = W.cbody_excl[b1];
  return (m >> (b2 - cb0)) & 1ull;
}

constexpr int BP_THREADS = 256;
constexpr int BP_WIN = 1024;  // broad-phase items per window (multiple of BP_THREADS)

// kind 0: PT, 1: EE, 2: ground. One CTA per environment. Work items are
// (row primitive, collision body) pairs in lexicographic order; an item is
// skipped when the pair is excluded (same rigid body, excluded bodies) or
// when the row's box misses the body's box inflated by `margin` — exact,
// because every primitive's inflated box lies inside its body's inflated
// box. Surviving items test the body's primitives in index order, so the
// output stays in the reference's lexicographic order.
constexpr int MAX_BODIES = 64;

__device__ __forceinline__ bool cull_item(const World& W, int cb0, int rb, int B, const double* qlo,
                                          const double* qhi, const double* blo, const double* bhi,
                                          double margin) {
  int gb = cb0 + B;
  if (gb == rb && W.cbody_rigid[rb]) return true;
  if (excluded(W, cb0, rb, gb)) return true;
  return !box_hit(qlo, qhi, blo + 3 * B, bhi + 3 * B, margin);
}

// primitive test of one (row, primitive) pair: inflated box overlap and the
// topological filter (shared vertex); the body-level filters ran already
__device__ __forceinline__ bool prim_hit(const World& W, int kind, int row, int2 er, int t, const double* qlo,
                                         const double* qhi, const double* __restrict__ lo,
                                         const double* __restrict__ hi, double margin) {
  double plo[3], phi[3];
  if (kind == 0) {
    int3 tv = W.tri_v[t];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      plo[c] = fmin(fmin(lo[3 * tv.x + c], lo[3 * tv.y + c]), lo[3 * tv.z + c]);
      phi[c] = fmax(fmax(hi[3 * tv.x + c], hi[3 * tv.y + c]), hi[3 * tv.z + c]);
    }
    return box_hit(qlo, qhi, plo, phi, margin) && !(tv.x == row || tv.y == row || tv.z == row);
  }
  int2 ej = W.edge_v[t];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    plo[c] = fmin(lo[3 * ej.x + c], lo[3 * ej.y + c]);
    phi[c] = fmax(hi[3 * ej.x + c], hi[3 * ej.y + c]);
  }
  return box_hit(qlo, qhi, plo, phi, margin) && !(er.x == ej.x || er.x == ej.y || er.y == ej.x || er.y == ej.y);
}

// visit, in increasing index order, the primitives of body gb in [c0, c1)
// that hit the row's query box; 32-primitive chunks whose inflated AABB
// misses the query box are skipped whole (exact: each primitive's inflated
// box lies inside its chunk's)
// (bvh: the body's LBVH, when it has one, was built from this call's [lo, hi]
// by k_lbvh_build — the global broad phase; the chunk walk otherwise)
template <typename F>
__device__ __forceinline__ void for_item_prims(const World& W, int kind, int row, int2 er, const double* qlo,
                                               const double* qhi, const double* __restrict__ lo,
                                               const double* __restrict__ hi, double margin, int gb, int c0,
                                               int c1, F f, bool bvh = false) {
  if (bvh) {
    int tr = kind == 0 ? W.cbody_tbvh[gb] : W.cbody_ebvh[gb];
    if (tr >= 0 &&
        lbvh_visit(W, tr, qlo, qhi, margin, c0, c1,
                   [&](int t) { return prim_hit(W, kind, row, er, t, qlo, qhi, lo, hi, margin); }, f))
      return;
  }
  const int* cp0 = kind == 0 ? W.tchunk_p0 : W.echunk_p0;
  const double* cbox = kind == 0 ? W.tchunk_box : W.echunk_box;
  int ch0 = kind == 0 ? W.cbody_tchunk[gb] : W.cbody_echunk[gb];
  int ch1 = kind == 0 ? W.cbody_tchunk[gb + 1] : W.cbody_echunk[gb + 1];
  for (int ch = ch0; ch < ch1; ++ch) {
    int p0 = max(cp0[ch], c0), p1 = min(cp0[ch + 1], c1);
    if (p0 >= p1) continue;
    if (!box_hit(qlo, qhi, cbox + 6 * ch, cbox + 6 * ch + 3, margin)) continue;
    for (int t = p0; t < p1; ++t)
      if (prim_hit(W, kind, row, er, t, qlo, qhi, lo, hi, margin)) f(t);
  }
}

// AABBs of the 32-primitive chunks (triangles then edges) at [lo, hi]
// c indexes triangle chunks then edge chunks
__device__ __forceinline__ void chunk_box(const World& W, const double* __restrict__ lo,
                                          const double* __restrict__ hi, int c) {
  int nt = W.n_tchunk;
  bool tri = c < nt;
  int ch = tri ? c : c - nt;
  const int* cp0 = tri ? W.tchunk_p0 : W.echunk_p0;
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int t = cp0[ch]; t < cp0[ch + 1]; ++t) {
    int vs[3];
    int nv = 2;
    if (tri) {
      int3 tv = W.tri_v[t];
      vs[0] = tv.x; vs[1] = tv.y; vs[2] = tv.z;
      nv = 3;
    } else {
      int2 ev = W.edge_v[t];
      vs[0] = ev.x; vs[1] = ev.y;
    }
    for (int k = 0; k < nv; ++k)
      for (int d = 0; d < 3; ++d) {
        mn[d] = fmin(mn[d], lo[3 * vs[k] + d]);
        mx[d] = fmax(mx[d], hi[3 * vs[k] + d]);
      }
  }
  double* box = (tri ? W.tchunk_box : W.echunk_box) + 6 * ch;
  for (int d = 0; d < 3; ++d) {
    box[d] = mn[d];
    box[3 + d] = mx[d];
  }
}

IPC_GLOBAL void k_chunk_boxes(World W, const double* __restrict__ lo, const double* __restrict__ hi) {
  ipc_pdl_wait();
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < W.n_tchunk + W.n_echunk) chunk_box(W, lo, hi, c);
}

// Multi-CTA split (gridDim.z = Z > 1, large envs): the env's item list is cut
// into Z contiguous ranges; pass 0 counts each range's hits into blk_cnt,
// pass 1 writes at the range's exclusive offset, so the output order is the
// same as with one CTA. pass -1: single CTA per env, count + write.
// block function (blockDim.x == BP_THREADS): range z of Z of env e's items
static __device__ void broad_env(const World& W, const double* __restrict__ lo, const double* __restrict__ hi,
                          const Cands& C, int kind, int e, int z, int Z, int pass, int* blk_cnt,
                          bool bvh = false) {
  __shared__ int warp_tot[BP_THREADS / 32];
  __shared__ int total;
  __shared__ double blo[3 * MAX_BODIES], bhi[3 * MAX_BODIES];
  double margin = W.env_dhat[e];
  int s0 = W.env_slot[e], s1 = W.env_slot[e + 1];
  int cb0 = W.env_cbody[e], nb = W.env_cbody[e + 1] - cb0;
  if (kind == 2) {
    if (z != 0 || pass == 1) return;
    int base = 0;
    if (!W.env_has_ground[e]) {
      if (threadIdx.x == 0) C.n_gnd[e] = 0;
      return;
    }
    double lim = __dadd_rn(W.env_ground_y[e], margin);
    int off = C.gnd_off[e];
    for (int s = s0; s < s1; s += BP_THREADS) {
      int v = s + threadIdx.x;
      bool hit = v < s1 && lo[3 * v + 1] < lim && !W.cbody_kin[W.slot_cbody[v]];
      int o = block_ordered_offset<BP_THREADS>(hit, warp_tot, &total);
      if (hit) C.gnd[off + base + o] = v;
      base += total;
      __syncthreads();
    }
    if (threadIdx.x == 0) C.n_gnd[e] = base;
    return;
  }
  if (!W.env_pairs[e]) {
    if (threadIdx.x == 0 && z == 0 && pass != 1) {
      if (kind == 0) C.n_pt[e] = 0; else C.n_ee[e] = 0;
    }
    return;
  }
  int* bc = blk_cnt ? blk_cnt + ((long long)e * 2 + kind) * Z : nullptr;
  // body boxes: one warp per body
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int B = wid; B < nb; B += BP_THREADS / 32) {
    int a0 = W.cbody_slot[cb0 + B], a1 = W.cbody_slot[cb0 + B + 1];
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int v = a0 + lane; v < a1; v += 32)
      for (int c = 0; c < 3; ++c) {
        mn[c] = fmin(mn[c], lo[3 * v + c]);
        mx[c] = fmax(mx[c], hi[3 * v + c]);
      }
    for (int o = 16; o > 0; o >>= 1)
      for (int c = 0; c < 3; ++c) {
        mn[c] = fmin(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
        mx[c] = fmax(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
      }
    if (lane == 0)
      for (int c = 0; c < 3; ++c) {
        blo[3 * B + c] = mn[c];
        bhi[3 * B + c] = mx[c];
      }
  }
  __syncthreads();
  long long cap, off;
  int r0, nrow;
  if (kind == 0) {
    r0 = s0;
    nrow = s1 - s0;
    off = C.pt_off[e];
    cap = C.pt_off[e + 1] - off;
  } else {
    r0 = W.env_edge[e];
    nrow = W.env_edge[e + 1] - r0;
    off = C.ee_off[e];
    cap = C.ee_off[e + 1] - off;
  }
  long long n_items = (long long)nrow * nb;
  long long per = ((n_items + Z - 1) / Z + BP_THREADS - 1) / BP_THREADS * BP_THREADS;
  long long i_begin = min(n_items, z * per), i_end = min(n_items, i_begin + per);
  long long base = 0, grand = 0;
  if (pass == 1) {
    for (int k = 0; k < Z; ++k) {
      if (k < z) base += bc[k];
      grand += bc[k];
    }
  }
  // Windows of BP_WIN items; warp w owns the contiguous segment
  // [win + w·SEG, win + (w+1)·SEG). Stage A: body-level culling, ordered
  // warp-local compaction of the surviving items (ballots, no block barrier).
  // Stage B: each survivor's hit count (chunk-culled primitive loop) and a
  // warp-local exclusive scan. One block barrier publishes the warp totals;
  // the write pass re-traverses the survivors. Output order = item order.
  __shared__ int surv[BP_WIN], soff[BP_WIN];
  __shared__ int wtot[BP_THREADS / 32];
  constexpr int SEG = BP_WIN / (BP_THREADS / 32);
  auto item = [&](long long it, int& row, int& B, int& c0, int& c1, int& rb, int2& er, double* qlo,
                  double* qhi) {
    row = r0 + (int)(it / nb);
    B = (int)(it % nb);
    if (kind == 0) {
      rb = W.slot_cbody[row];
      for (int c = 0; c < 3; ++c) {
        qlo[c] = lo[3 * row + c];
        qhi[c] = hi[3 * row + c];
      }
      c0 = W.cbody_tri[cb0 + B];
      c1 = W.cbody_tri[cb0 + B + 1];
    } else {
      rb = W.edge_cbody[row];
      er = W.edge_v[row];
      for (int c = 0; c < 3; ++c) {
        qlo[c] = fmin(lo[3 * er.x + c], lo[3 * er.y + c]);
        qhi[c] = fmax(hi[3 * er.x + c], hi[3 * er.y + c]);
      }
      c0 = max(W.cbody_edge[cb0 + B], row + 1);
      c1 = W.cbody_edge[cb0 + B + 1];
    }
  };
  for (long long win = i_begin; win < i_end; win += BP_WIN) {
    // stage A
    int ns = 0;
    long long seg0 = win + (long long)wid * SEG;
    for (int j = 0; j < SEG; j += 32) {
      long long it = seg0 + j + lane;
      bool live = false;
      if (it < i_end) {
        int row, B, c0, c1, rb;
        int2 er = make_int2(0, 0);
        double qlo[3], qhi[3];
        item(it, row, B, c0, c1, rb, er, qlo, qhi);
        live = c0 < c1 && !cull_item(W, cb0, rb, B, qlo, qhi, blo, bhi, margin);
      }
      unsigned m = __ballot_sync(0xffffffffu, live);
      if (live) surv[wid * SEG + ns + __popc(m & ((1u << lane) - 1u))] = (int)(it - win);
      ns += __popc(m);
    }
    __syncwarp();
    // stage B: counts + warp-local exclusive scan (survivor order)
    int run = 0;
    for (int j0 = 0; j0 < ns; j0 += 32) {
      int j = j0 + lane, n_hit = 0;
      if (j < ns) {
        int row, B, c0, c1, rb;
        int2 er = make_int2(0, 0);
        double qlo[3], qhi[3];
        item(win + surv[wid * SEG + j], row, B, c0, c1, rb, er, qlo, qhi);
        for_item_prims(W, kind, row, er, qlo, qhi, lo, hi, margin, B + cb0, c0, c1, [&](int) { ++n_hit; }, bvh);
      }
      int incl = n_hit;
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (j < ns) soff[wid * SEG + j] = run + incl - n_hit;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) wtot[wid] = run;
    __syncthreads();
    long long wbase = base, wsum = 0;
    for (int w = 0; w < BP_THREADS / 32; ++w) {
      if (w < wid) wbase += wtot[w];
      wsum += wtot[w];
    }
    if (pass != 0) {
      for (int j = lane; j < ns; j += 32) {
        int row, B, c0, c1, rb;
        int2 er = make_int2(0, 0);
        double qlo[3], qhi[3];
        item(win + surv[wid * SEG + j], row, B, c0, c1, rb, er, qlo, qhi);
        long long dst = wbase + soff[wid * SEG + j];
        for_item_prims(W, kind, row, er, qlo, qhi, lo, hi, margin, B + cb0, c0, c1, [&](int t) {
          if (dst < cap) {
            if (kind == 0) C.pt[off + dst] = make_int2(row, t);
            else C.ee[off + dst] = make_int2(row, t);
          }
          ++dst;
        }, bvh);
      }
    }
    base += wsum;
    __syncthreads();
  }
  if (pass == 0) {  // count only: this range's total
    if (threadIdx.x == 0) bc[z] = (int)base;
    return;
  }
  if (pass == 1) {
    if (z != 0) return;
    base = grand;
  }
  if (threadIdx.x == 0) {
    int need = (int)min(base, (long long)INT_MAX);
    if (kind == 0) C.need_pt[e] = need; else C.need_ee[e] = need;
    if (base > cap) {
      atomicExch(C.overflow, 1);
      base = cap;
    }
    if (kind == 0) C.n_pt[e] = (int)base; else C.n_ee[e] = (int)base;
  }
}

IPC_GLOBAL void __launch_bounds__(BP_THREADS) k_broad(World W, const double* __restrict__ lo,
                                                       const double* __restrict__ hi, Cands C,
                                                       int kind, const int* env_mask, int pass,
                                                       int* blk_cnt) {
  ipc_pdl_wait();
  if (kind < 0) kind = blockIdx.y;  // all three kinds in one launch
  int e = blockIdx.x;
  if (env_mask && !env_mask[e]) return;
  broad_env(W, lo, hi, C, kind, e, blockIdx.z, gridDim.z, pass, blk_cnt, W.n_tree > 0);
}

// Exact candidates of the query boxes [lo, hi] of env e from its cached
// superset S into C (fused.cuh env_candidates explains the superset): the
// prim-level box test of the broad phase, same arithmetic, in S's order.
static __device__ bool ss_filter_env(const World& W, const Cands& S, const double* lo, const double* hi,
                                     const Cands& C, int e) {
  __shared__ int wtot[BP_THREADS / 32];
  __shared__ int s_total, s_ov;
  int tid = threadIdx.x;
  double margin = W.env_dhat[e];
  if (!W.env_has_ground[e]) {
    if (tid == 0) C.n_gnd[e] = 0;
  } else {
    double lim = __dadd_rn(W.env_ground_y[e], margin);
    int off = C.gnd_off[e], n = S.n_gnd[e], base = 0;
    for (int k0 = 0; k0 < n; k0 += BP_THREADS) {
      int k = k0 + tid, sl = k < n ? S.gnd[off + k] : 0;
      bool hit = k < n && lo[3 * sl + 1] < lim;
      int o = block_ordered_offset<BP_THREADS>(hit, wtot, &s_total);
      if (hit) C.gnd[off + base + o] = sl;
      base += s_total;
      __syncthreads();
    }
    if (tid == 0) C.n_gnd[e] = base;
  }
  for (int kind = 0; kind < 2; ++kind) {
    int n = W.env_pairs[e] ? (kind == 0 ? S.n_pt[e] : S.n_ee[e]) : 0;
    long long soff = kind == 0 ? S.pt_off[e] : S.ee_off[e];
    long long coff = kind == 0 ? C.pt_off[e] : C.ee_off[e];
    long long cap = (kind == 0 ? C.pt_off[e + 1] : C.ee_off[e + 1]) - coff;
    long long base = 0;
    for (int k0 = 0; k0 < n; k0 += BP_THREADS) {
      int k = k0 + tid;
      bool hit = false;
      int2 pr = make_int2(0, 0);
      if (k < n) {
        pr = kind == 0 ? S.pt[soff + k] : S.ee[soff + k];
        double q[6], p[6];
        if (kind == 0) {  // slot box vs triangle box (env_broad_sm: sb, tb)
          int3 v = W.tri_v[pr.y];
          for (int c = 0; c < 3; ++c) {
            q[c] = lo[3 * pr.x + c];
            q[3 + c] = hi[3 * pr.x + c];
            p[c] = fmin(fmin(lo[3 * v.x + c], lo[3 * v.y + c]), lo[3 * v.z + c]);
            p[3 + c] = fmax(fmax(hi[3 * v.x + c], hi[3 * v.y + c]), hi[3 * v.z + c]);
          }
        } else {  // edge box vs edge box (eb)
          int2 a = W.edge_v[pr.x], b = W.edge_v[pr.y];
          for (int c = 0; c < 3; ++c) {
            q[c] = fmin(lo[3 * a.x + c], lo[3 * a.y + c]);
            q[3 + c] = fmax(hi[3 * a.x + c], hi[3 * a.y + c]);
            p[c] = fmin(lo[3 * b.x + c], lo[3 * b.y + c]);
            p[3 + c] = fmax(hi[3 * b.x + c], hi[3 * b.y + c]);
          }
        }
        hit = box_hit(q, q + 3, p, p + 3, margin);
      }
      int o = block_ordered_offset<BP_THREADS>(hit, wtot, &s_total);
      if (hit && base + o < cap) {
        if (kind == 0) C.pt[coff + base + o] = pr;
        else C.ee[coff + base + o] = pr;
      }
      base += s_total;
      __syncthreads();
    }
    if (tid == 0) {
      int need = (int)min(base, (long long)INT_MAX);
      if (kind == 0) C.need_pt[e] = need; else C.need_ee[e] = need;
      if (base > cap) {
        atomicExch(C.overflow, 1);
        base = cap;
      }
      if (kind == 0) C.n_pt[e] = (int)base; else C.n_ee[e] = (int)base;
    }
  }
  __syncthreads();
  if (tid == 0) s_ov = *(volatile int*)C.overflow;
  __syncthreads();
  return !s_ov;
}

// Batched superset check (one CTA per env): does every slot's query box lie
// inside its build box? If not, write fresh build boxes (query box ± pad·d̂)
// and flag the env for a superset rebuild.
// With wx given, the CTA first writes its env's world positions xw(wx) into
// xw_out (k_world folded in, every env; lo / hi may alias xw_out, hence no
// __restrict__ / read-only loads on them).
IPC_GLOBAL void k_ss_check(World W, const double* lo, const double* hi, double* bb_lo, double* bb_hi, double pad,
                           const int* env_mask, int* valid, int* rebuild, const double* __restrict__ wx,
                           double* xw_out) {
  ipc_pdl_wait();
  int e = blockIdx.x;
  if (wx) {
    for (int s = W.env_slot[e] + threadIdx.x; s < W.env_slot[e + 1]; s += blockDim.x) world_slot(W, wx, xw_out, s);
    __syncthreads();
  }
  if (env_mask && !env_mask[e]) {
    if (threadIdx.x == 0) rebuild[e] = 0;
    return;
  }
  int i0 = 3 * W.env_slot[e], i1 = 3 * W.env_slot[e + 1];
  int ok = valid[e];
  if (ok)
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) ok &= (lo[i] >= bb_lo[i]) & (hi[i] <= bb_hi[i]);
  ok = __syncthreads_and(ok);
  if (!ok) {
    double p = pad * W.env_dhat[e];
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      bb_lo[i] = __dsub_rn(lo[i], p);
      bb_hi[i] = __dadd_rn(hi[i], p);
    }
  }
  if (threadIdx.x == 0) {
    rebuild[e] = !ok;
    valid[e] = 1;
  }
}

IPC_GLOBAL void __launch_bounds__(BP_THREADS) k_ss_filter(World W, const double* __restrict__ lo,
                                                          const double* __restrict__ hi, Cands S, Cands C,
                                                          const int* env_mask, const int* order) {
  ipc_pdl_wait();
  int e = order ? order[blockIdx.x] : blockIdx.x;
  if (env_mask && !env_mask[e]) return;
  ss_filter_env(W, S, lo, hi, C, e);
}

// per-env exclusive prefix of counts over flagged envs, one CTA: each thread
// sums a contiguous run of envs, the run totals are scanned with warp
// shuffles (two barriers), then each thread writes its run. pre has n_env + 1
// entries, pre[n_env] = total.
__device__ __forceinline__ void block_prefix_envs(int n_env, const int* __restrict__ cnt, const int* flag,
                                                  int* pre) {
  __shared__ int wsum[32];
  int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  int per = (n_env + nt - 1) / nt;
  int a = tid * per, b = min(n_env, a + per);
  int s = 0;
  for (int e = a; e < b; ++e) s += (flag == nullptr || flag[e]) ? cnt[e] : 0;
  int inc = s;  // inclusive scan within the warp
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int nw = (nt + 31) >> 5;
    int w = lane < nw ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    wsum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int run = inc - s + (wid ? wsum[wid - 1] : 0);
  for (int e = a; e < b; ++e) {
    pre[e] = run;
    run += (flag == nullptr || flag[e]) ? cnt[e] : 0;
  }
  if (tid == nt - 1) pre[n_env] = run;
}

IPC_GLOBAL void k_prefix(int n_env, const int* cnt, const int* flag, int* pre) {
  ipc_pdl_wait();
  block_prefix_envs(n_env, cnt, flag, pre);
}

// the three candidate-count prefixes (PT, EE, ground) in one launch; a
// fourth CTA (when fill is given) sets fill[e] = v on the flagged envs (the
// per-iteration reset of min_s / alpha_max that follows every broad phase)
IPC_GLOBAL void k_prefix3(int n_env, Cands C, const int* flag, double* fill, double v) {
  ipc_pdl_wait();
  if (blockIdx.x == 3) {
    for (int e = threadIdx.x; e < n_env; e += blockDim.x)
      if (flag[e]) fill[e] = v;
    return;
  }
  const int* cnt = blockIdx.x == 0 ? C.n_pt : (blockIdx.x == 1 ? C.n_ee : C.n_gnd);
  int* pre = blockIdx.x == 0 ? C.pre_pt : (blockIdx.x == 1 ? C.pre_ee : C.pre_gnd);
  block_prefix_envs(n_env, cnt, flag, pre);
}

// env owning flattened item g: pre[e] <= g < pre[e+1] (last such e)
__device__ __forceinline__ int find_env(const int* __restrict__ pre, int n_env, int g) {
  int lo = 0, hi = n_env;  // invariant: pre[lo] <= g < pre[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pre[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// element terms. Outputs per element: value, gradient, packed Hessian.
// ---------------------------------------------------------------------------

// per affine body: inertia + h² orthogonality (projected) + kinematic target
__device__ __forceinline__ void body_item(const World& W, const double* __restrict__ x,
                                          const double* __restrict__ xhat, double h2, int deriv, int b,
                                          double* val, double* g12, double* h144) {
  int e = W.aff_env[b];
  int o = W.aff_dof[b];
  const double* M = W.aff_M + 144 * b;
  double d[12];
  for (int i = 0; i < 12; ++i) d[i] = x[o + i] - xhat[o + i];
  double g[12];
  double v = 0.0;
  for (int i = 0; i < 12; ++i) {
    double s = 0.0;
    for (int j = 0; j < 12; ++j) s += M[12 * i + j] * d[j];
    g[i] = s;
    v += d[i] * s;
  }
  v *= 0.5;
  // orthogonality coeff ||A A^T - I||^2 (ref terms.py:66)
  double c = W.aff_ortho[b];
  M3 A;
  for (int i = 0; i < 9; ++i) A.m[i] = x[o + 3 + i];
  M3 Mm = m3_mul(A, m3_T(A));
  m3_add_diag(Mm, -1.0);
  double ov = 0.0;
  for (int i = 0; i < 9; ++i) ov += Mm.m[i] * Mm.m[i];
  v += h2 * c * ov;
  // Hessian = M_b + h² (projected orthogonality block) + Σ κ_A I, written
  // straight to the output (no 12x12 local array)
  double h9[81];
  if (deriv) {
    M3 MA = m3_mul(Mm, A);
    for (int i = 0; i < 9; ++i) g[3 + i] += h2 * 4.0 * c * MA.m[i];
    ortho_hess_psd(A, c, h9);
  }
  // kinematic constraints on this body (ref constraints.py:55)
  double kap_diag = 0.0;
  for (int k = W.env_cons[e]; k < W.env_cons[e + 1]; ++k) {
    if (W.cons_aff[k] != b) continue;
    double kap = W.cons_kappa[k], sm = sqrt(W.cons_mass[k]);
    const double* tg = W.cons_target + 12 * k;
    const double* lam = W.cons_lam + 12 * k;
    double dd = 0.0, ld = 0.0;
    for (int i = 0; i < 12; ++i) {
      double di = x[o + i] - tg[i];
      dd += di * di;
      ld += lam[i] * di;
      if (deriv) g[i] += kap * di - sm * lam[i];
    }
    kap_diag += kap;
    v += 0.5 * kap * dd - sm * ld;
  }
  val[b] = v;
  if (deriv) {
    for (int i = 0; i < 12; ++i) g12[12 * b + i] = g[i];
    double* ho = h144 + 144 * b;
#pragma unroll
    for (int i = 0; i < 12; ++i)
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        double hv = M[12 * i + j];
        if (i >= 3 && j >= 3) hv += h2 * h9[9 * (i - 3) + j - 3];
        if (i == j) hv += kap_diag;
        ho[12 * i + j] = hv;
      }
  }
}

IPC_GLOBAL void k_body(World W, const double* __restrict__ x, const double* __restrict__ xhat,
                       double h2, int deriv, const int* env_flag, double* val, double* g12,
                       double* h144) {
  ipc_pdl_wait();
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= W.n_aff) return;
  if (env_flag && !env_flag[W.aff_env[b]]) return;
  body_item(W, x, xhat, h2, deriv, b, val, g12, h144);
}

// per tet: h² V ψ(F), gradient, PSD-projected stencil Hessian (ref elastic.py:204)
__device__ __forceinline__ void tet_item(const World& W, const double* __restrict__ x, double h2, int deriv,
                                         int t, double* val, double* g12, double* hp) {
  int4 d = W.tet_dof[t];
  V3 x0 = ld3(x + d.x), x1 = ld3(x + d.y), x2 = ld3(x + d.z), x3 = ld3(x + d.w);
  V3 e1 = x1 - x0, e2 = x2 - x0, e3 = x3 - x0;
  const double* Dm = W.tet_Dminv + 9 * t;
  M3 Ds;  // columns e1 e2 e3
  Ds.m[0] = e1.x; Ds.m[1] = e2.x; Ds.m[2] = e3.x;
  Ds.m[3] = e1.y; Ds.m[4] = e2.y; Ds.m[5] = e3.y;
  Ds.m[6] = e1.z; Ds.m[7] = e2.z; Ds.m[8] = e3.z;
  M3 Dmi;
  for (int i = 0; i < 9; ++i) Dmi.m[i] = Dm[i];
  M3 F = m3_mul(Ds, Dmi);
  double vol = W.tet_vol[t], mu = W.tet_mu[t], lam = W.tet_lam[t];
  int model = W.tet_model[t];
  double s = h2 * vol;
  if (!deriv) {
    double psi = psi_value(model, F, mu, lam);
    val[t] = isinf(psi) ? INFINITY : s * psi;
    return;
  }
  double psi, P[9], H9[81];
  if (!psi_derivs(model, F, mu, lam, &psi, P, H9)) {
    val[t] = INFINITY;
    return;
  }
  val[t] = s * psi;
  psd_project<9>(H9, 9);
  // stencil coefficients: dF_ij = Σ_v C[v][j] dx_{v,i}
  double Cc[4][3];
  for (int j = 0; j < 3; ++j) {
    Cc[1][j] = Dm[j];
    Cc[2][j] = Dm[3 + j];
    Cc[3][j] = Dm[6 + j];
    Cc[0][j] = -(Dm[j] + Dm[3 + j] + Dm[6 + j]);
  }
  for (int v = 0; v < 4; ++v)
    for (int i = 0; i < 3; ++i) {
      double acc = 0.0;
      for (int j = 0; j < 3; ++j) acc += P[3 * i + j] * Cc[v][j];
      g12[12 * t + 3 * v + i] = s * acc;
    }
  // H[(v,l),(w,m)] = s Σ_jk C[v][j] C[w][k] H9[(l,j),(m,k)]
  for (int r = 0; r < 12; ++r) {
    int v = r / 3, l = r % 3;
    for (int c = r; c < 12; ++c) {
      int w = c / 3, m = c % 3;
      double acc = 0.0;
      for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) acc += Cc[v][j] * Cc[w][k] * H9[(3 * l + j) * 9 + 3 * m + k];
      hp[PK * t + pk(r, c)] = s * acc;
    }
  }
}

IPC_GLOBAL void k_tet(World W, const double* __restrict__ x, double h2, int deriv,
                      const int* env_flag, double* val, double* g12, double* hp) {
  ipc_pdl_wait();
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= W.n_tet) return;
  if (env_flag && !env_flag[W.tet_env[t]]) return;
  tet_item(W, x, h2, deriv, t, val, g12, hp);
}

// Contact pairs, pass 1 (light, every candidate of every flagged env):
// region + squared distance, value κ b (× mollifier) for active pairs, 0
// otherwise, INF when an active pair has non-positive distance
// (ref contact.py:239-268); min distance stats. In the derivative pass the
// active pairs are appended to a work list for pass 2. Persistent
// grid-stride over the flattened candidate index (prefix C.pre_*).
__device__ __forceinline__ void pair_slots(const World& W, int kind, int2 pr, int* sl) {
  if (kind == 0) {
    int3 tv = W.tri_v[pr.y];
    sl[0] = pr.x; sl[1] = tv.x; sl[2] = tv.y; sl[3] = tv.z;
  } else {
    int2 a = W.edge_v[pr.x], b = W.edge_v[pr.y];
    sl[0] = a.x; sl[1] = a.y; sl[2] = b.x; sl[3] = b.y;
  }
}

struct PairIO {  // per-kind (0 PT, 1 EE) buffers; kind = blockIdx.y
  double* val[2];
  unsigned char* act[2];
  double* g[2];
  double* h[2];
  long long* work[2];
  int* work_env[2];
  int* work_n;
};

// value of candidate q of env e; returns true when the pair is active
// (0 < d² < ŝ: its derivatives are needed)
__device__ __forceinline__ bool pair_value_item(const World& W, const double* __restrict__ xw, const Cands& C,
                                                int kind, long long q, int e, double* val,
                                                unsigned char* active, double* env_min_s) {
    int2 pr = kind == 0 ? C.pt[q] : C.ee[q];
    int sl[4];
    pair_slots(W, kind, pr, sl);
    V3 X[4];
    for (int i = 0; i < 4; ++i) X[i] = ld3(xw + 3 * sl[i]);
    double d2;
    if (kind == 0) {
      int r = pt_region(X[0], X[1], X[2], X[3]);
      d2 = pt_dist2(r, X[0], X[1], X[2], X[3]);
    } else {
      int r = ee_region(X[0], X[1], X[2], X[3], nullptr);
      d2 = ee_dist2(r, X[0], X[1], X[2], X[3]);
    }
    if (env_min_s) atomic_min_pos(env_min_s, d2);
    double dhat = W.env_dhat[e], shat = dhat * dhat;
    if (active) active[q] = 0;
    if (!(d2 < shat)) {
      val[q] = 0.0;
      return false;
    }
    if (d2 <= 0.0) {
      val[q] = INFINITY;
      return false;
    }
    double kappa = W.env_kappa[e];
    double b = barrier_val(d2, shat);
    double m = 1.0;
    if (kind == 1) m = mollifier_val(cross2(X[1] - X[0], X[3] - X[2]), 1e-6 * W.edge_len2[pr.x] * W.edge_len2[pr.y]);
    val[q] = kind == 1 ? kappa * (m * b) : kappa * b;
    return true;
}

IPC_GLOBAL void k_pair_dist(World W, const double* __restrict__ xw, Cands C, int deriv, PairIO io,
                            double* env_min_s) {
  ipc_pdl_wait();
  const int kind = blockIdx.y;
  const int* pre = kind == 0 ? C.pre_pt : C.pre_ee;
  int total = pre[W.n_env];
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    int e = find_env(pre, W.n_env, g);
    long long q = (kind == 0 ? C.pt_off[e] : C.ee_off[e]) + (g - pre[e]);
    bool act = pair_value_item(W, xw, C, kind, q, e, io.val[kind], io.act[kind],
                               env_min_s ? env_min_s + e : nullptr);
    if (act && deriv) {
      int slot = atomicAdd(io.work_n + kind, 1);
      io.work[kind][slot] = q;
      io.work_env[kind][slot] = e;
    }
  }
}

// Contact pairs, pass 2 (heavy, active pairs only): closed-form distance
// derivatives in var space, barrier chain rule, mollifier product rule, and
// the PSD projection in the Helmert space of the region's active slots
// (ipc_math.cuh helm_*; ref contact.py:255-266, spd.py:6). Everything stays in
// registers: no 12x12 stencil array is formed.

// var-space derivatives of a region: NV difference vars v_i = x_{p_i} - x_{q_i}
// (p, q: local slot indices of the region's NS active slots)
template <int NV>
struct VarSet {
  V3 gv[NV];
  M3 hv[NV][NV];
  int p[NV], q[NV];
  double s;
};

template <int NS>
__device__ __forceinline__ void pair_core_out(const int (&sl)[NS], double* gh, double* M, double* g12,
                                              double* hp) {
  constexpr int R = 3 * (NS - 1);
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < r; ++c) M[r * R + c] = M[c * R + r];
#ifndef IPC_NO_PSD
  psd_project<R>(M, R);
#endif
  helm_out<NS>(sl, gh, M, g12, hp);
}

// Every region of every pair kind reduces to one core: up to three difference
// vars over the stencil's four slots (p, q: stencil slot indices; unused vars
// have zero derivatives), projected in the 9-dim Helmert space of all four
// slots. A region's stencil Hessian annihilates translations of the whole
// stencil (inactive slots have zero rows), so Q4 (Q4ᵀHQ4)⁺ Q4ᵀ is the same
// projection (ref spd.py:6) as in the region's own smaller Helmert space —
// and one psd_project<9> per kernel keeps the code small (instruction-cache
// bound otherwise).
template <int NV>
__device__ __forceinline__ void var_pad(const VarSet<NV>& A, const int* sl, VarSet<3>& V) {
  V.s = A.s;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    V.p[i] = i < NV ? sl[A.p[i < NV ? i : 0]] : 0;
    V.q[i] = i < NV ? sl[A.q[i < NV ? i : 0]] : 0;
    V.gv[i] = i < NV ? A.gv[i < NV ? i : 0] : V3{0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 3; ++j) V.hv[i][j] = (i < NV && j < NV) ? A.hv[i < NV ? i : 0][j < NV ? j : 0] : m3_zero();
  }
}

// H = κ(b'' ∇s∇sᵀ + b' ∇²s), g = κ b' ∇s (core, upper triangle of M)
__device__ __forceinline__ void pair_plain_core(const VarSet<3>& V, double kappa, double shat, double (&gh)[9],
                                                double (&M)[81]) {
  double b, db, d2b;
  barrier_d(V.s, shat, &b, &db, &d2b);
  double beta[3][3];
  helm_beta<3, 3>(V.p, V.q, beta);
  helm_grad<3, 3>(beta, V.gv, gh);
#pragma unroll
  for (int i = 0; i < 81; ++i) M[i] = 0.0;
  helm_hess_acc<3, 3>(beta, V.hv, kappa * db, M);
  helm_outer_acc<9>(gh, gh, kappa * d2b, false, M);
#pragma unroll
  for (int i = 0; i < 9; ++i) gh[i] *= kappa * db;
}

// mollified EE (ref contact.py:166-203, :286-312), all 4 slots: the s part in its
// region vars (stencil slot indices) and the mollifier c = |u x v|²
__device__ __forceinline__ void ee_mollified_core(const VarSet<3>& V, const V3* X, double t, double eps, double kappa,
                                                  double shat, double (&gh)[9], double (&M)[81]) {
  double b, db, d2b;
  barrier_d(V.s, shat, &b, &db, &d2b);
  double em = t * (2.0 - t), de = (2.0 - 2.0 * t) / eps, d2e = -2.0 / (eps * eps);
  double bs[3][3], bc[2][3];
  helm_beta<3, 3>(V.p, V.q, bs);
  VarSet<2> Cv;
  vs_cross2(X[1] - X[0], X[3] - X[2], Cv.gv, Cv.hv);
  Cv.p[0] = 1; Cv.q[0] = 0; Cv.p[1] = 3; Cv.q[1] = 2;
  helm_beta<2, 3>(Cv.p, Cv.q, bc);
  double gs[9], gc[9];
  helm_grad<3, 3>(bs, V.gv, gs);
  helm_grad<2, 3>(bc, Cv.gv, gc);
#pragma unroll
  for (int i = 0; i < 81; ++i) M[i] = 0.0;
  helm_hess_acc<3, 3>(bs, V.hv, kappa * (em * db), M);
  helm_hess_acc<2, 3>(bc, Cv.hv, kappa * (de * b), M);
  helm_outer_acc<9>(gs, gs, kappa * (em * d2b), false, M);
  helm_outer_acc<9>(gc, gc, kappa * (d2e * b), false, M);
  helm_outer_acc<9>(gc, gs, kappa * (de * db), true, M);
#pragma unroll
  for (int i = 0; i < 9; ++i) gh[i] = kappa * ((de * b) * gc[i] + (em * db) * gs[i]);
}

__device__ __forceinline__ VarSet<1> region_pp(const V3* X, int i, int j) {
  VarSet<1> V;
  V.s = vs_pp(X[i] - X[j], V.gv, V.hv);
  V.p[0] = i; V.q[0] = j;
  return V;
}
// point a to line (b, c): w = x_a - x_b, e = x_c - x_b
__device__ __forceinline__ VarSet<2> region_pl(const V3* X, int a, int b, int c) {
  VarSet<2> V;
  V.s = vs_pl(X[a] - X[b], X[c] - X[b], V.gv, V.hv);
  V.p[0] = a; V.q[0] = b; V.p[1] = c; V.q[1] = b;
  return V;
}

// squared distance and its stencil gradient only (G: 12, zero on entry), for
// the friction lags (ref friction.py:75) — no Hessian is formed
template <int NV>
__device__ __forceinline__ double scatter_grad(const VarSet<NV>& V, const int* sl, double* G) {
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    int a = sl[V.p[i]], b = sl[V.q[i]];
    G[3 * a] += V.gv[i].x; G[3 * a + 1] += V.gv[i].y; G[3 * a + 2] += V.gv[i].z;
    G[3 * b] -= V.gv[i].x; G[3 * b + 1] -= V.gv[i].y; G[3 * b + 2] -= V.gv[i].z;
  }
  return V.s;
}
__device__ __forceinline__ double dist2_grad(bool is_pt, int region, const V3* X, double* G) {
  const int id[4] = {0, 1, 2, 3};
  if (is_pt) {
    if (region < 3) return scatter_grad<1>(region_pp(X, 0, region + 1), id, G);
    if (region == 3) return scatter_grad<2>(region_pl(X, 0, 1, 2), id, G);
    if (region == 4) return scatter_grad<2>(region_pl(X, 0, 2, 3), id, G);
    if (region == 5) return scatter_grad<2>(region_pl(X, 0, 3, 1), id, G);
    VarSet<3> V;
    V.s = vs_triple(X[0] - X[1], X[2] - X[1], X[3] - X[1], V.gv, V.hv);
    V.p[0] = 0; V.q[0] = 1; V.p[1] = 2; V.q[1] = 1; V.p[2] = 3; V.q[2] = 1;
    return scatter_grad<3>(V, id, G);
  }
  int ra = region / 3, rb = region % 3;
  if (ra < 2 && rb < 2) return scatter_grad<1>(region_pp(X, ra, 2 + rb), id, G);
  if (ra < 2) return scatter_grad<2>(region_pl(X, ra, 2, 3), id, G);
  if (rb < 2) return scatter_grad<2>(region_pl(X, 2 + rb, 0, 1), id, G);
  VarSet<3> V;
  V.s = vs_triple(X[2] - X[0], X[1] - X[0], X[3] - X[2], V.gv, V.hv);
  V.p[0] = 2; V.q[0] = 0; V.p[1] = 1; V.q[1] = 0; V.p[2] = 3; V.q[2] = 2;
  return scatter_grad<3>(V, id, G);
}

template <int kind>
__device__ __forceinline__ void pair_hess_item(const World& W, const double* __restrict__ xw, const Cands& C,
                                               long long k, int e, double* g12, double* hp,
                                               unsigned char* active) {
    int2 pr = kind == 0 ? C.pt[k] : C.ee[k];
    int sl4[4];
    pair_slots(W, kind, pr, sl4);
    V3 X[4];
    for (int i = 0; i < 4; ++i) X[i] = ld3(xw + 3 * sl4[i]);
    double dhat = W.env_dhat[e], shat = dhat * dhat, kappa = W.env_kappa[e];
    double* g = g12 + 12 * k;
    double* h = hp + PK * k;
    // the region's vars over stencil slots
    VarSet<3> V;
    bool moll = false;
    double t = 0.0, eps = 0.0;
    if (kind == 0) {
      int region = pt_region(X[0], X[1], X[2], X[3]);
      if (region < 3) {  // point-point: var x0 - xt
        int tt = region + 1;
        VarSet<1> A;
        A.s = vs_pp(X[0] - X[tt], A.gv, A.hv);
        A.p[0] = 0; A.q[0] = 1;
        const int sl[2] = {0, tt};
        var_pad<1>(A, sl, V);
      } else if (region < 6) {  // point-edge (a, bb)
        int a = region == 3 ? 1 : (region == 4 ? 2 : 3);
        int bb = region == 3 ? 2 : (region == 4 ? 3 : 1);
        VarSet<2> A;
        A.s = vs_pl(X[0] - X[a], X[bb] - X[a], A.gv, A.hv);
        A.p[0] = 0; A.q[0] = 1; A.p[1] = 2; A.q[1] = 1;
        const int sl[3] = {0, a, bb};
        var_pad<2>(A, sl, V);
      } else {  // point-face: w = x0 - x1, u = x2 - x1, v = x3 - x1
        V.s = vs_triple(X[0] - X[1], X[2] - X[1], X[3] - X[1], V.gv, V.hv);
        V.p[0] = 0; V.q[0] = 1; V.p[1] = 2; V.q[1] = 1; V.p[2] = 3; V.q[2] = 1;
      }
    } else {
      int region = ee_region(X[0], X[1], X[2], X[3], nullptr);
      eps = 1e-6 * W.edge_len2[pr.x] * W.edge_len2[pr.y];
      t = cross2(X[1] - X[0], X[3] - X[2]) / eps;
      moll = t < 1.0;
      // region slots: PP (i, j) / point i to line (j, k) / line-line
      int ra = region / 3, rb = region % 3;
      const int id[4] = {0, 1, 2, 3};
      if (ra < 2 && rb < 2) {
        var_pad<1>(region_pp(X, ra, 2 + rb), id, V);
      } else if (ra < 2) {
        var_pad<2>(region_pl(X, ra, 2, 3), id, V);
      } else if (rb < 2) {
        var_pad<2>(region_pl(X, 2 + rb, 0, 1), id, V);
      } else {
        V.s = vs_triple(X[2] - X[0], X[1] - X[0], X[3] - X[2], V.gv, V.hv);
        V.p[0] = 2; V.q[0] = 0; V.p[1] = 1; V.q[1] = 0; V.p[2] = 3; V.q[2] = 2;
      }
    }
    double gh[9], M[81];
    if (kind == 1 && moll) ee_mollified_core(V, X, t, eps, kappa, shat, gh, M);
    else pair_plain_core(V, kappa, shat, gh, M);
    const int sl[4] = {0, 1, 2, 3};
    pair_core_out<4>(sl, gh, M, g, h);
    active[k] = (unsigned char)0xF;
}

template <int kind>
__global__ void __launch_bounds__(64) k_pair_hess(World W, const double* __restrict__ xw, Cands C, PairIO io) {
  ipc_pdl_wait();
  int total = io.work_n[kind];
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < total; w += gridDim.x * blockDim.x)
    pair_hess_item<kind>(W, xw, C, io.work[kind][w], io.work_env[kind][w], io.g[kind], io.h[kind], io.act[kind]);
}

// ground candidates (ref contact.py:315-345): value, y-gradient, clamped y-curvature
// ground candidate k (global index) of env e; min_s: the env's minimum
__device__ __forceinline__ void ground_item(const World& W, const double* __restrict__ xw, const Cands& C,
                                            int deriv, int k, int e, double* val, double* gy, double* hyy,
                                            double* min_s) {
  int s = C.gnd[k];
  double d = xw[3 * s + 1] - W.env_ground_y[e];
  double dhat = W.env_dhat[e], shat = dhat * dhat;
  if (d <= 0.0) {
    val[k] = INFINITY;
    if (min_s) atomic_min_pos(min_s, 0.0);
    return;
  }
  double ss = d * d;
  if (min_s) atomic_min_pos(min_s, ss);
  if (!(ss < shat)) {
    val[k] = 0.0;
    if (deriv) { gy[k] = 0.0; hyy[k] = 0.0; }
    return;
  }
  double kappa = W.env_kappa[e];
  double b, db, d2b;
  barrier_d(ss, shat, &b, &db, &d2b);
  val[k] = kappa * b;
  if (deriv) {
    gy[k] = kappa * db * 2.0 * d;
    hyy[k] = fmax(kappa * (d2b * 4.0 * d * d + db * 2.0), 0.0);
  }
}

IPC_GLOBAL void k_ground(World W, const double* __restrict__ xw, Cands C, int deriv,
                         const int* env_flag, double* val, double* gy, double* hyy,
                         double* env_min_s) {
  ipc_pdl_wait();
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  int e = blockIdx.y;
  if (k >= C.n_gnd[e]) return;
  if (env_flag && !env_flag[e]) return;
  ground_item(W, xw, C, deriv, k + C.gnd_off[e], e, val, gy, hyy, env_min_s ? env_min_s + e : nullptr);
}

// ---------------------------------------------------------------------------
// friction (ref friction.py)
// ---------------------------------------------------------------------------
IPC_HD void tangent_basis(V3 n, double* T /*3x2 row-major*/) {
  V3 ref = fabs(n.x) < 0.9 ? v3(1, 0, 0) : v3(0, 1, 0);
  V3 t1 = crossx(n, ref);
  double l = sqrt(dotx(t1, t1));
  t1 = v3(t1.x / l, t1.y / l, t1.z / l);
  V3 t2 = crossx(n, t1);
  T[0] = t1.x; T[1] = t2.x;
  T[2] = t1.y; T[3] = t2.y;
  T[4] = t1.z; T[5] = t2.z;
}

// lag one candidate pair if active and λ > 0; lags are appended per env in
// candidate order (PT list then EE list) — one CTA per env for ordering.
static __device__ void lags_env(const World& W, const double* __restrict__ xw, const Cands& C, const Lags& L, int e) {
  __shared__ int warp_tot[BP_THREADS / 32];
  __shared__ int total;
  double dhat = W.env_dhat[e], shat = dhat * dhat, kappa = W.env_kappa[e];
  long long lo = L.off[e];
  int base = 0;
  for (int kind = 0; kind < 2; ++kind) {
    int n = kind == 0 ? C.n_pt[e] : C.n_ee[e];
    long long coff = kind == 0 ? C.pt_off[e] : C.ee_off[e];
    for (int k0 = 0; k0 < n; k0 += BP_THREADS) {
      int k = k0 + threadIdx.x;
      bool keep = false;
      int sl[4];
      double gam[4], T[6], lam = 0.0;
      if (k < n) {
        int2 pr = kind == 0 ? C.pt[coff + k] : C.ee[coff + k];
        if (kind == 0) {
          int3 tv = W.tri_v[pr.y];
          sl[0] = pr.x; sl[1] = tv.x; sl[2] = tv.y; sl[3] = tv.z;
        } else {
          int2 a = W.edge_v[pr.x], b = W.edge_v[pr.y];
          sl[0] = a.x; sl[1] = a.y; sl[2] = b.x; sl[3] = b.y;
        }
        V3 X[4];
        for (int i = 0; i < 4; ++i) X[i] = ld3(xw + 3 * sl[i]);
        int region;
        double d2;
        if (kind == 0) {
          region = pt_region(X[0], X[1], X[2], X[3]);
          d2 = pt_dist2(region, X[0], X[1], X[2], X[3]);
        } else {
          region = ee_region(X[0], X[1], X[2], X[3], nullptr);
          d2 = ee_dist2(region, X[0], X[1], X[2], X[3]);
        }
        if (d2 < shat) {
          double G[12];
          for (int i = 0; i < 12; ++i) G[i] = 0.0;
          double s = dist2_grad(kind == 0, region, X, G);
          double d = sqrt(s);
          double b, db, d2b;
          barrier_d(s, shat, &b, &db, &d2b);
          V3 n3;
          if (kind == 0) {
            lam = -kappa * db * 2.0 * d;
            n3 = v3(G[0] / (2.0 * d), G[1] / (2.0 * d), G[2] / (2.0 * d));
            gam[0] = 1.0;
            for (int v = 1; v < 4; ++v) {
              double w = -(G[3 * v] * n3.x + G[3 * v + 1] * n3.y + G[3 * v + 2] * n3.z) / (2.0 * d);
              gam[v] = -w;
            }
          } else {
            double eps = 1e-6 * W.edge_len2[pr.x] * W.edge_len2[pr.y];
            double m = mollifier_val(cross2(X[1] - X[0], X[3] - X[2]), eps);
            lam = -kappa * m * db * 2.0 * d;
            n3 = v3((G[0] + G[3]) / (2.0 * d), (G[1] + G[4]) / (2.0 * d), (G[2] + G[5]) / (2.0 * d));
            for (int v = 0; v < 2; ++v)
              gam[v] = (G[3 * v] * n3.x + G[3 * v + 1] * n3.y + G[3 * v + 2] * n3.z) / (2.0 * d);
            for (int v = 2; v < 4; ++v) {
              double wb = -(G[3 * v] * n3.x + G[3 * v + 1] * n3.y + G[3 * v + 2] * n3.z) / (2.0 * d);
              gam[v] = -wb;
            }
          }
          tangent_basis(n3, T);
          keep = lam > 0.0;
        }
      }
      int o = block_ordered_offset<BP_THREADS>(keep, warp_tot, &total);
      if (keep) {
        long long dst = lo + base + o;
        L.slots[dst] = make_int4(sl[0], sl[1], sl[2], sl[3]);
        for (int i = 0; i < 4; ++i) L.gamma[4 * dst + i] = gam[i];
        for (int i = 0; i < 6; ++i) L.tangent[6 * dst + i] = T[i];
        L.lam[dst] = lam;
      }
      base += total;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) L.n[e] = base;
  // ground lags
  int gbase = 0;
  int ng = C.n_gnd[e];
  int goff = C.gnd_off[e];
  for (int k0 = 0; k0 < ng; k0 += BP_THREADS) {
    int k = k0 + threadIdx.x;
    bool keep = false;
    int s = 0;
    double lam = 0.0;
    if (k < ng) {
      s = C.gnd[goff + k];
      double d = xw[3 * s + 1] - W.env_ground_y[e];
      double ss = d * d;
      if (ss < shat) {
        double b, db, d2b;
        barrier_d(ss, shat, &b, &db, &d2b);
        lam = -kappa * db * 2.0 * d;
        keep = lam > 0.0;
      }
    }
    int o = block_ordered_offset<BP_THREADS>(keep, warp_tot, &total);
    if (keep) {
      L.g_slot[goff + gbase + o] = s;
      L.g_lam[goff + gbase + o] = lam;
    }
    gbase += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) L.g_n[e] = gbase;
}

IPC_GLOBAL void k_lags(World W, const double* __restrict__ xw, Cands C, Lags L, const int* env_flag,
                       const int* order) {
  ipc_pdl_wait();
  int e = order ? order[blockIdx.x] : blockIdx.x;
  if (env_flag && !env_flag[e]) return;
  lags_env(W, xw, C, L, e);
}

IPC_HD double f0s(double y, double eh) {
  return y < eh ? y * y / eh - y * y * y / (3.0 * eh * eh) + eh / 3.0 : y;
}
IPC_HD double f1s(double y, double eh) { return y < eh ? 2.0 * y / eh - y * y / (eh * eh) : 1.0; }

// smoothed tangential norm: value, 2-vector gradient, 2x2 Hessian (ref friction.py:177)
IPC_HD double smooth_norm(double u0, double u1, double ml, double eh, double* gu, double* hu) {
  double y = sqrt(u0 * u0 + u1 * u1);
  double v = ml * f0s(y, eh);
  if (gu) {
    double fac = y > 0 ? f1s(y, eh) / fmax(y, 1e-300) : 2.0 / eh;
    gu[0] = ml * fac * u0;
    gu[1] = ml * fac * u1;
    double df1 = y < eh ? 2.0 / eh - 2.0 * y / (eh * eh) : 0.0;
    double coef = y > 1e-300 ? df1 - fac : 0.0;
    double iy = 1.0 / fmax(y, 1e-300);
    double h0 = u0 * iy, h1 = u1 * iy;
    hu[0] = ml * (fac + coef * h0 * h0);
    hu[1] = ml * (coef * h0 * h1);
    hu[2] = hu[1];
    hu[3] = ml * (fac + coef * h1 * h1);
  }
  return v;
}

__device__ __forceinline__ void friction_item(const World& W, const double* __restrict__ xw,
                                              const double* __restrict__ xw0, const Lags& L, double h, int deriv,
                                              long long q, int e, double* val, double* g12, double* hp) {
  int4 s4 = L.slots[q];
  int sl[4] = {s4.x, s4.y, s4.z, s4.w};
  const double* gam = L.gamma + 4 * q;
  const double* T = L.tangent + 6 * q;
  double u3[3] = {0, 0, 0};
  for (int i = 0; i < 4; ++i)
    for (int c = 0; c < 3; ++c) u3[c] += gam[i] * (xw[3 * sl[i] + c] - xw0[3 * sl[i] + c]);
  double u0 = T[0] * u3[0] + T[2] * u3[1] + T[4] * u3[2];
  double u1 = T[1] * u3[0] + T[3] * u3[1] + T[5] * u3[2];
  double ml = W.env_mu[e] * L.lam[q];
  double eh = W.env_epsv[e] * h;
  double gu[2], hu[4];
  val[q] = smooth_norm(u0, u1, ml, eh, deriv ? gu : nullptr, hu);
  if (!deriv) return;
  double g3[3], h3[9];
  for (int a = 0; a < 3; ++a) {
    g3[a] = T[2 * a] * gu[0] + T[2 * a + 1] * gu[1];
    for (int b = 0; b < 3; ++b)
      h3[3 * a + b] = T[2 * a] * (hu[0] * T[2 * b] + hu[1] * T[2 * b + 1]) +
                      T[2 * a + 1] * (hu[2] * T[2 * b] + hu[3] * T[2 * b + 1]);
  }
  for (int i = 0; i < 4; ++i)
    for (int a = 0; a < 3; ++a) g12[12 * q + 3 * i + a] = gam[i] * g3[a];
  for (int r = 0; r < 12; ++r)
    for (int c = r; c < 12; ++c) hp[PK * q + pk(r, c)] = gam[r / 3] * gam[c / 3] * h3[3 * (r % 3) + c % 3];
}

IPC_GLOBAL void k_friction(World W, const double* __restrict__ xw, const double* __restrict__ xw0,
                           Lags L, double h, int deriv, const int* env_flag, double* val,
                           double* g12, double* hp) {
  ipc_pdl_wait();
  int total = L.pre[W.n_env];
  for (int gi = blockIdx.x * blockDim.x + threadIdx.x; gi < total; gi += gridDim.x * blockDim.x) {
    int e = find_env(L.pre, W.n_env, gi);
    if (env_flag && !env_flag[e]) continue;
    friction_item(W, xw, xw0, L, h, deriv, L.off[e] + (gi - L.pre[e]), e, val, g12, hp);
  }
}

// ground friction: tangent frame (x, z)
__device__ __forceinline__ void friction_gnd_item(const World& W, const double* __restrict__ xw,
                                                  const double* __restrict__ xw0, const Lags& L, double h,
                                                  int deriv, int q, int e, double* val, double* g3, double* h3) {
  int s = L.g_slot[q];
  double u0 = xw[3 * s] - xw0[3 * s], u1 = xw[3 * s + 2] - xw0[3 * s + 2];
  double ml = W.env_mu[e] * L.g_lam[q];
  double eh = W.env_epsv[e] * h;
  double gu[2], hu[4];
  val[q] = smooth_norm(u0, u1, ml, eh, deriv ? gu : nullptr, hu);
  if (!deriv) return;
  g3[3 * q] = gu[0]; g3[3 * q + 1] = 0.0; g3[3 * q + 2] = gu[1];
  h3[9 * q + 0] = hu[0]; h3[9 * q + 1] = 0.0; h3[9 * q + 2] = hu[1];
  h3[9 * q + 3] = 0.0; h3[9 * q + 4] = 0.0; h3[9 * q + 5] = 0.0;
  h3[9 * q + 6] = hu[2]; h3[9 * q + 7] = 0.0; h3[9 * q + 8] = hu[3];
}

IPC_GLOBAL void k_friction_gnd(World W, const double* __restrict__ xw, const double* __restrict__ xw0,
                               Lags L, double h, int deriv, const int* env_flag, double* val,
                               double* g3, double* h3) {
  ipc_pdl_wait();
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  int e = blockIdx.y;
  if (k >= L.g_n[e]) return;
  if (env_flag && !env_flag[e]) return;
  friction_gnd_item(W, xw, xw0, L, h, deriv, W.env_slot[e] + k, e, val, g3, h3);
}

// ---------------------------------------------------------------------------
// CCD: per-pair conservative advancement (ref ccd.py:34) and ground crossing
// ---------------------------------------------------------------------------
static __device__ double stencil_dist(int kind, const V3* X) {
  if (kind == 0) {
    int r = pt_region(X[0], X[1], X[2], X[3]);
    return sqrt(pt_dist2(r, X[0], X[1], X[2], X[3]));
  }
  int r = ee_region(X[0], X[1], X[2], X[3], nullptr);
  return sqrt(ee_dist2(r, X[0], X[1], X[2], X[3]));
}

static __device__ double pair_ccd_alpha(int kind, const V3* X, const V3* D, double conservative) {
  V3 sum = ((D[0] + D[1]) + D[2]) + D[3];
  V3 mean = v3(__ddiv_rn(sum.x, 4.0), __ddiv_rn(sum.y, 4.0), __ddiv_rn(sum.z, 4.0));
  double sp[4];
  for (int i = 0; i < 4; ++i) {
    V3 r = D[i] - mean;
    sp[i] = sqrt(dotx(r, r));
  }
  double l = kind == 0 ? sp[0] + fmax(fmax(sp[1], sp[2]), sp[3]) : fmax(sp[0], sp[1]) + fmax(sp[2], sp[3]);
  double d0 = stencil_dist(kind, X);
  if (!(l > 1e-300)) return 1.0;
  double t = 0.0, d = d0, g = 0.01 * d0;
  for (int it = 0; it < 64; ++it) {
    double tn = t + d / l;
    if (tn >= 1.0) return 1.0;
    V3 Y[4];
    for (int i = 0; i < 4; ++i)
      Y[i] = v3(__dadd_rn(X[i].x, __dmul_rn(tn, D[i].x)), __dadd_rn(X[i].y, __dmul_rn(tn, D[i].y)),
                __dadd_rn(X[i].z, __dmul_rn(tn, D[i].z)));
    d = stencil_dist(kind, Y);
    t = tn;
    if (d <= g) return conservative * t;
  }
  return fmin(1.0, fmax(conservative * t, 1e-12));
}

__device__ __forceinline__ double ccd_pair_item(const World& W, const double* __restrict__ xw,
                                                const double* __restrict__ dxw, const Cands& C, int kind,
                                                long long q, double conservative) {
  int2 pr = kind == 0 ? C.pt[q] : C.ee[q];
  int sl[4];
  pair_slots(W, kind, pr, sl);
  V3 X[4], D[4];
  for (int i = 0; i < 4; ++i) {
    X[i] = ld3(xw + 3 * sl[i]);
    D[i] = ld3(dxw + 3 * sl[i]);
  }
  return pair_ccd_alpha(kind, X, D, conservative);
}

// ground crossing time of ground candidate k (global index) of env e, or 2 (none)
__device__ __forceinline__ double ccd_ground_item(const World& W, const double* __restrict__ xw,
                                                  const double* __restrict__ dxw, const Cands& C, int k, int e,
                                                  double conservative) {
  int s = C.gnd[k];
  double y = xw[3 * s + 1], dy = dxw[3 * s + 1];
  if (!(dy < 0.0)) return 2.0;
  double t = (y - W.env_ground_y[e]) / -dy;
  if (!(t <= 1.0)) return 2.0;
  return fmin(1.0, conservative * t);
}

IPC_GLOBAL void k_ccd_pairs(World W, const double* __restrict__ xw, const double* __restrict__ dxw,
                            Cands C, double conservative, const int* env_flag, double* env_alpha) {
  ipc_pdl_wait();
  const int kind = blockIdx.y;
  const int* pre = kind == 0 ? C.pre_pt : C.pre_ee;
  int total = pre[W.n_env];
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    int e = find_env(pre, W.n_env, g);
    if (env_flag && !env_flag[e]) continue;
    long long q = (kind == 0 ? C.pt_off[e] : C.ee_off[e]) + (g - pre[e]);
    double a = ccd_pair_item(W, xw, dxw, C, kind, q, conservative);
    if (a < 1.0) atomic_min_pos(env_alpha + e, a);
  }
}

IPC_GLOBAL void k_ccd_ground(World W, const double* __restrict__ xw, const double* __restrict__ dxw,
                             Cands C, double conservative, const int* env_flag, double* env_alpha) {
  ipc_pdl_wait();
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  int e = blockIdx.y;
  if (k >= C.n_gnd[e]) return;
  if (env_flag && !env_flag[e]) return;
  double a = ccd_ground_item(W, xw, dxw, C, C.gnd_off[e] + k, e, conservative);
  if (a <= 1.0) atomic_min_pos(env_alpha + e, a);
}

}  // namespace ipc
