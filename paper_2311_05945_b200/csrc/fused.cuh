// Fused per-environment time step for dense worlds: one 256-thread CTA runs
// the whole of ref solver.py:355-454 for one environment — feasibility check,
// predictor, lagged-friction fixed point, augmented-Lagrangian outer loop,
// Newton iterations (DCD broad phase, every energy term, dense LDLᵀ solve,
// CCD sweep + conservative advancement, backtracking line search), post-step
// distance and κ adaptation — with block barriers between phases and no host
// round trip. CTAs pull environments from an atomic queue, so a long
// contact-onset solve in one env overlaps with the rest of the batch instead
// of serialising the launch sequence of the batched path.
//
// Every per-element formula is the batched path's own item function
// (kernels.cuh / solve.cuh), so both paths produce the same values; only
// the schedule differs (sequential line-search trials instead of speculative
// ones, which accept the same α).
#pragma once
#include "solve.cuh"

namespace ipc {

// optional phase timers (IPC_FUSED_TIMERS=1): SM cycles per phase,
// summed over envs into FusedArgs::timers
enum { FT_WORLD, FT_BROAD_DCD, FT_TERMS, FT_ENERGY, FT_DENSE, FT_CCD_PREP, FT_BROAD_CCD, FT_CCD, FT_LS, FT_OTHER,
       FT_N };
// per-item latency of the terms phase's heavy items, after the phases:
// (cycle sum, count, max) for PT pair Hessians, EE pair Hessians, affine
// bodies, friction stencils
enum { FT_IT_PT, FT_IT_EE, FT_IT_BODY, FT_IT_FR, FT_NIT };
// sub-phases of the dense solve (dense_solve_block dtm), after the items
constexpr int FT_DENSE_SUB = FT_N + 3 * FT_NIT, FT_NDS = 9;
constexpr int FT_TOTAL = FT_DENSE_SUB + FT_NDS;
__device__ __forceinline__ void ft_item(long long* timers, int type, long long t0) {
  if (!timers) return;
  long long dt = clock64() - t0;
  unsigned long long* p = (unsigned long long*)timers + FT_N + 3 * type;
  atomicAdd(p, (unsigned long long)dt);
  atomicAdd(p + 1, 1ull);
  atomicMax(p + 2, (unsigned long long)dt);
}
// phase timers are on when FusedArgs::timers is set (IPC_FUSED_TIMERS=1 at
// world creation): a block-uniform branch, no cost when off
#define FT_MARK(A, k)                                                     \
  do {                                                                    \
    if ((A).timers) {                                                     \
      __syncthreads();                                                    \
      if (threadIdx.x < 32) { /* whole warp 0: no lane-0 divergence */    \
        long long now = clock64();                                        \
        atomicAdd((unsigned long long*)(A).timers + (k),                  \
                  threadIdx.x == 0 ? (unsigned long long)(now - ft_t0) : 0ull); \
        ft_t0 = now;                                                      \
      }                                                                   \
    }                                                                     \
  } while (0)
#define FT_START long long ft_t0 = clock64()

struct FusedArgs {
  World W;
  EnvState S;
  Cands dc, sw;  // DCD / CCD-sweep candidate stores
  Cands ss;      // cached candidate superset (env_candidates)
  double *bb_lo, *bb_hi;  // per-slot build boxes of the superset
  double ss_pad;          // build-box padding in units of d̂ (0: superset off)
  Lags L;
  Derivs D;      // derivative buffers of the DCD store
  Terms T;       // value buffers of the DCD store
  double *xwt, *xlo, *xhi;
  const int* enable;
  int *ok, *accepted, *ls_count;
  const double* targets;
  int* queue;        // [0]: next env
  const int* order;  // queue position -> env (nullptr: identity)
  long long* stat;   // [0] Newton iterations, [1] line-search trials
  long long* timers; // [FT_N] phase cycles, or nullptr (timers off)
  double h, newton_tol, ccd_cons;
  int max_newton, max_halvings, fp_iters, al_max_outer;
  int smem_doubles;  // dynamic shared memory per CTA (time-shared scratch)
};

static __device__ __noinline__ void fused_pair_hess0(const World& W, const double* xw, const Cands& C, long long q, int e,
                                              const Derivs& D) {
  pair_hess_item<0>(W, xw, C, q, e, D.pt_g, D.pt_h, D.pt_act);
}
static __device__ __noinline__ void fused_pair_hess1(const World& W, const double* xw, const Cands& C, long long q, int e,
                                              const Derivs& D) {
  pair_hess_item<1>(W, xw, C, q, e, D.ee_g, D.ee_h, D.ee_act);
}
static __device__ __noinline__ void fused_body(const World& W, const double* x, const double* xhat, double h2, int deriv,
                                        int b, double* val, double* g, double* hh) {
  body_item(W, x, xhat, h2, deriv, b, val, g, hh);
}
static __device__ __noinline__ void fused_tet(const World& W, const double* x, double h2, int deriv, int t, double* val,
                                       double* g, double* hp) {
  tet_item(W, x, h2, deriv, t, val, g, hp);
}

__device__ __forceinline__ void env_world(const World& W, const double* x, double* xw, int e) {
  for (int s = W.env_slot[e] + threadIdx.x; s < W.env_slot[e + 1]; s += blockDim.x) world_slot(W, x, xw, s);
  __syncthreads();
}

// broad phase of env e over [lo, hi] into C; returns false on capacity
// overflow (sticky flag: the host replays the whole step with more room)
static __device__ bool env_broad(const World& W, const double* lo, const double* hi, const Cands& C, int e) {
  __shared__ int s_ov;
  int b0 = W.env_cbody[e], b1 = W.env_cbody[e + 1];
  int t0 = W.cbody_tchunk[b0], t1 = W.cbody_tchunk[b1];
  int q0 = W.cbody_echunk[b0], q1 = W.cbody_echunk[b1];
  for (int c = t0 + threadIdx.x; c < t1; c += blockDim.x) chunk_box(W, lo, hi, c);
  for (int c = q0 + threadIdx.x; c < q1; c += blockDim.x) chunk_box(W, lo, hi, W.n_tchunk + c);
  __syncthreads();
  for (int kind = 0; kind < 3; ++kind) {
    broad_env(W, lo, hi, C, kind, e, 0, 1, -1, nullptr);
    __syncthreads();
  }
  if (threadIdx.x == 0) s_ov = *(volatile int*)C.overflow;
  __syncthreads();
  return !s_ov;
}

// Broad phase of env e with every box staged in shared memory (buf, cap
// doubles): slot boxes, triangle / edge boxes, 32-primitive chunk boxes, body
// boxes. Same tests, same box arithmetic and the same (row, primitive)
// output order as broad_env; the global-memory version runs when the env's
// boxes do not fit. Returns false on capacity overflow.
static __device__ bool env_broad_sm(const World& W, const double* __restrict__ lo, const double* __restrict__ hi,
                             const Cands& C, int e, double* buf, int cap_d) {
  __shared__ double blo[3 * MAX_BODIES], bhi[3 * MAX_BODIES];
  __shared__ int surv[BP_WIN], soff[BP_WIN];
  __shared__ int wtot[BP_THREADS / 32];
  __shared__ int s_ov, s_total;
  int s0 = W.env_slot[e], s1 = W.env_slot[e + 1], ns = s1 - s0;
  int t0 = W.env_tri[e], nt = W.env_tri[e + 1] - t0;
  int e0 = W.env_edge[e], ne = W.env_edge[e + 1] - e0;
  int cb0 = W.env_cbody[e], nb = W.env_cbody[e + 1] - cb0;
  int tc0 = W.cbody_tchunk[cb0], ntc = W.cbody_tchunk[cb0 + nb] - tc0;
  int ec0 = W.cbody_echunk[cb0], nec = W.cbody_echunk[cb0 + nb] - ec0;
  if (6 * (ns + nt + ne + ntc + nec) > cap_d) return env_broad(W, lo, hi, C, e);
  double* sb = buf;            // slot boxes (lo xyz, hi xyz)
  double* tb = sb + 6 * ns;    // triangle boxes
  double* eb = tb + 6 * nt;    // edge boxes
  double* tcb = eb + 6 * ne;   // triangle chunk boxes
  double* ecb = tcb + 6 * ntc; // edge chunk boxes
  int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < 3 * ns; i += blockDim.x) {
    int s = i / 3, c = i - 3 * s;
    sb[6 * s + c] = lo[3 * (s0 + s) + c];
    sb[6 * s + 3 + c] = hi[3 * (s0 + s) + c];
  }
  __syncthreads();
  for (int t = tid; t < nt; t += blockDim.x) {
    int3 v = W.tri_v[t0 + t];
    const double *a = sb + 6 * (v.x - s0), *b = sb + 6 * (v.y - s0), *c = sb + 6 * (v.z - s0);
    for (int k = 0; k < 3; ++k) {
      tb[6 * t + k] = fmin(fmin(a[k], b[k]), c[k]);
      tb[6 * t + 3 + k] = fmax(fmax(a[3 + k], b[3 + k]), c[3 + k]);
    }
  }
  for (int t = tid; t < ne; t += blockDim.x) {
    int2 v = W.edge_v[e0 + t];
    const double *a = sb + 6 * (v.x - s0), *b = sb + 6 * (v.y - s0);
    for (int k = 0; k < 3; ++k) {
      eb[6 * t + k] = fmin(a[k], b[k]);
      eb[6 * t + 3 + k] = fmax(a[3 + k], b[3 + k]);
    }
  }
  __syncthreads();
  for (int i = tid; i < ntc + nec; i += blockDim.x) {
    bool tri = i < ntc;
    int ch = tri ? tc0 + i : ec0 + (i - ntc);
    const int* cp0 = tri ? W.tchunk_p0 : W.echunk_p0;
    const double* pb = tri ? tb - 6 * t0 : eb - 6 * e0;  // indexed by global primitive id below
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int q = cp0[ch]; q < cp0[ch + 1]; ++q)
      for (int k = 0; k < 3; ++k) {
        mn[k] = fmin(mn[k], pb[6 * q + k]);
        mx[k] = fmax(mx[k], pb[6 * q + 3 + k]);
      }
    double* o = (tri ? tcb : ecb) + 6 * (tri ? i : i - ntc);
    for (int k = 0; k < 3; ++k) {
      o[k] = mn[k];
      o[3 + k] = mx[k];
    }
  }
  for (int B = wid; B < nb; B += BP_THREADS / 32) {  // body boxes, one warp per body
    int a0 = W.cbody_slot[cb0 + B] - s0, a1 = W.cbody_slot[cb0 + B + 1] - s0;
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int v = a0 + lane; v < a1; v += 32)
      for (int c = 0; c < 3; ++c) {
        mn[c] = fmin(mn[c], sb[6 * v + c]);
        mx[c] = fmax(mx[c], sb[6 * v + 3 + c]);
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
  double margin = W.env_dhat[e];
  // ground candidates (kind 2)
  if (!W.env_has_ground[e]) {
    if (tid == 0) C.n_gnd[e] = 0;
  } else {
    double lim = __dadd_rn(W.env_ground_y[e], margin);
    int off = C.gnd_off[e], base = 0;
    for (int v0 = 0; v0 < ns; v0 += BP_THREADS) {
      int v = v0 + tid;
      bool hit = v < ns && sb[6 * v + 1] < lim && !W.cbody_kin[W.slot_cbody[s0 + v]];
      int o = block_ordered_offset<BP_THREADS>(hit, wtot, &s_total);
      if (hit) C.gnd[off + base + o] = s0 + v;
      base += s_total;
      __syncthreads();
    }
    if (tid == 0) C.n_gnd[e] = base;
  }
  for (int kind = 0; kind < 2; ++kind) {
    if (!W.env_pairs[e]) {
      if (tid == 0) {
        if (kind == 0) C.n_pt[e] = 0; else C.n_ee[e] = 0;
      }
      continue;
    }
    int r0 = kind == 0 ? s0 : e0, nrow = kind == 0 ? ns : ne;
    long long off = kind == 0 ? C.pt_off[e] : C.ee_off[e];
    long long cap = (kind == 0 ? C.pt_off[e + 1] : C.ee_off[e + 1]) - off;
    int n_items = nrow * nb;
    // query box of row r (local index): slot box or edge box
    const double* qb = kind == 0 ? sb : eb;
    const int* cp0 = kind == 0 ? W.tchunk_p0 : W.echunk_p0;
    const int* cbc = kind == 0 ? W.cbody_tchunk : W.cbody_echunk;
    const double* chb = kind == 0 ? tcb : ecb;
    int chbase = kind == 0 ? tc0 : ec0;
    const double* pbx = kind == 0 ? tb : eb;
    int pbase = kind == 0 ? t0 : e0;
    auto range = [&](int it, int& row, int& B, int& c0, int& c1) {
      row = it / nb;
      B = it - row * nb;
      if (kind == 0) {
        c0 = W.cbody_tri[cb0 + B];
        c1 = W.cbody_tri[cb0 + B + 1];
      } else {
        c0 = max(W.cbody_edge[cb0 + B], r0 + row + 1);
        c1 = W.cbody_edge[cb0 + B + 1];
      }
    };
    // visit the hits of item (row, B) in primitive order
    auto visit = [&](int row, int B, int c0, int c1, auto f) {
      const double* q = qb + 6 * row;
      int grow = r0 + row;
      int2 er = kind == 1 ? W.edge_v[grow] : make_int2(0, 0);
      for (int ch = cbc[cb0 + B]; ch < cbc[cb0 + B + 1]; ++ch) {
        int p0 = max(cp0[ch], c0), p1 = min(cp0[ch + 1], c1);
        if (p0 >= p1) continue;
        const double* cb = chb + 6 * (ch - chbase);
        if (!box_hit(q, q + 3, cb, cb + 3, margin)) continue;
        for (int t = p0; t < p1; ++t) {
          const double* pb = pbx + 6 * (t - pbase);
          if (!box_hit(q, q + 3, pb, pb + 3, margin)) continue;
          if (kind == 0) {
            int3 tv = W.tri_v[t];
            if (tv.x == grow || tv.y == grow || tv.z == grow) continue;
          } else {
            int2 ej = W.edge_v[t];
            if (er.x == ej.x || er.x == ej.y || er.y == ej.x || er.y == ej.y) continue;
          }
          f(t);
        }
      }
    };
    constexpr int SEG = BP_WIN / (BP_THREADS / 32);
    long long base = 0;
    for (int win = 0; win < n_items; win += BP_WIN) {
      int nsv = 0;
      int seg0 = win + wid * SEG;
      for (int j = 0; j < SEG; j += 32) {
        int it = seg0 + j + lane;
        bool live = false;
        if (it < n_items) {
          int row, B, c0, c1;
          range(it, row, B, c0, c1);
          int rb = kind == 0 ? W.slot_cbody[r0 + row] : W.edge_cbody[r0 + row];
          const double* q = qb + 6 * row;
          live = c0 < c1 && !cull_item(W, cb0, rb, B, q, q + 3, blo, bhi, margin);
        }
        unsigned m = __ballot_sync(0xffffffffu, live);
        if (live) surv[wid * SEG + nsv + __popc(m & ((1u << lane) - 1u))] = it - win;
        nsv += __popc(m);
      }
      __syncwarp();
      int run = 0;
      for (int j0 = 0; j0 < nsv; j0 += 32) {
        int j = j0 + lane, n_hit = 0;
        if (j < nsv) {
          int row, B, c0, c1;
          range(win + surv[wid * SEG + j], row, B, c0, c1);
          visit(row, B, c0, c1, [&](int) { ++n_hit; });
        }
        int incl = n_hit;
        for (int o = 1; o < 32; o <<= 1) {
          int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        if (j < nsv) soff[wid * SEG + j] = run + incl - n_hit;
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) wtot[wid] = run;
      __syncthreads();
      long long wbase = base, wsum = 0;
      for (int w = 0; w < BP_THREADS / 32; ++w) {
        if (w < wid) wbase += wtot[w];
        wsum += wtot[w];
      }
      for (int j = lane; j < nsv; j += 32) {
        int row, B, c0, c1;
        range(win + surv[wid * SEG + j], row, B, c0, c1);
        long long dst = wbase + soff[wid * SEG + j];
        int grow = r0 + row;
        visit(row, B, c0, c1, [&](int t) {
          if (dst < cap) {
            if (kind == 0) C.pt[off + dst] = make_int2(grow, t);
            else C.ee[off + dst] = make_int2(grow, t);
          }
          ++dst;
        });
      }
      base += wsum;
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

// ---------------------------------------------------------------------------
// Cached candidate superset (ref broadphase.py:74 BroadPhaseCache keeps its
// trees across queries and rebuilds only after large motion). The superset S
// of env e is the exact broad phase over every slot's *build box*: the query
// box the slot had at build time grown by ss_pad·d̂ on every side. For any
// later configuration in which each slot's query box (a point for DCD, the
// sweep box for CCD) lies inside its build box, every pair the exact broad
// phase reports is in S (primitive boxes are unions of slot boxes, the pair
// margin is d̂ in both). The exact list is S filtered with the prim-level box
// test of env_broad_sm (identical arithmetic) in S's lexicographic order, so
// it is bit-identical to a fresh broad phase at the cost of one ordered
// compaction; S is rebuilt when a query box leaves its build box.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool env_ss_covers(const FusedArgs& A, const double* lo, const double* hi, int e) {
  const World& W = A.W;
  int ok = 1;
  for (int i = 3 * W.env_slot[e] + threadIdx.x; i < 3 * W.env_slot[e + 1]; i += blockDim.x)
    ok &= (lo[i] >= A.bb_lo[i]) & (hi[i] <= A.bb_hi[i]);
  return __syncthreads_and(ok);
}

static __device__ bool env_ss_build(const FusedArgs& A, const double* lo, const double* hi, int e, double* sm) {
  const World& W = A.W;
  double pad = A.ss_pad * W.env_dhat[e];
  for (int i = 3 * W.env_slot[e] + threadIdx.x; i < 3 * W.env_slot[e + 1]; i += blockDim.x) {
    A.bb_lo[i] = __dsub_rn(lo[i], pad);
    A.bb_hi[i] = __dadd_rn(hi[i], pad);
  }
  __syncthreads();
  return env_broad_sm(W, A.bb_lo, A.bb_hi, A.ss, e, sm, A.smem_doubles);
}

// exact candidates of the query boxes [lo, hi] from the env's superset into C
static __device__ bool env_ss_filter(const FusedArgs& A, const double* lo, const double* hi, const Cands& C, int e) {
  return ss_filter_env(A.W, A.ss, lo, hi, C, e);
}

// candidates of the query boxes [lo, hi] into C: through the env's cached
// superset (*ss_ok: block-uniform shared flag, 0 = no valid superset) or a
// fresh broad phase when the cache is off (ss_pad == 0)
static __device__ bool env_candidates(const FusedArgs& A, const double* lo, const double* hi, const Cands& C, int e,
                                      double* sm, int* ss_ok) {
  if (A.ss_pad <= 0.0) return env_broad_sm(A.W, lo, hi, C, e, sm, A.smem_doubles);
  if (!(*ss_ok && env_ss_covers(A, lo, hi, e))) {
    if (!env_ss_build(A, lo, hi, e, sm)) return false;
    if (threadIdx.x == 0) *ss_ok = 1;
  }
  return env_ss_filter(A, lo, hi, C, e);
}

// Batched schedule: the shared-memory broad phase, one CTA per flagged env
// (all three kinds; chunk boxes built in shared memory).
IPC_GLOBAL void __launch_bounds__(BP_THREADS) k_broad_sm(World W, const double* __restrict__ lo,
                                                          const double* __restrict__ hi, Cands C,
                                                          const int* env_mask, int cap_d, const int* order) {
  ipc_pdl_wait();
  extern __shared__ double bsm[];
  int e = order ? order[blockIdx.x] : blockIdx.x;
  if (env_mask && !env_mask[e]) return;
  env_broad_sm(W, lo, hi, C, e, bsm, cap_d);
}

// element values (deriv = 0) or values + derivatives of every term at x / xw;
// returns the env's minimum squared distance over candidates and ground.
// Derivative pass: one value sweep over all candidates (PT and EE together)
// appends the active pairs to a shared work list, then bodies, tets and the
// active pairs are spread over the block in one round, so the latency is one
// pair Hessian rather than one per kind.
constexpr int FUSED_WORK = 1024;
static __device__ double env_terms(const FusedArgs& A, const double* x, const double* xw, int deriv, int e) {
  const World& W = A.W;
  __shared__ double s_min;
  __shared__ int s_nw;
  __shared__ int s_work[FUSED_WORK];  // kind << 30 | local candidate index
  if (threadIdx.x == 0) {
    s_min = INFINITY;
    s_nw = 0;
  }
  __syncthreads();
  double h2 = A.h * A.h;
  const Cands& C = A.dc;
  int n_pt = C.n_pt[e], n_ee = C.n_ee[e];
  long long pt_off = C.pt_off[e], ee_off = C.ee_off[e];
  for (int k = threadIdx.x; k < n_pt + n_ee; k += blockDim.x) {
    int kind = k < n_pt ? 0 : 1;
    int j = kind == 0 ? k : k - n_pt;
    long long q = (kind == 0 ? pt_off : ee_off) + j;
    bool on = pair_value_item(W, xw, C, kind, q, e, kind == 0 ? A.T.pt_val : A.T.ee_val,
                              kind == 0 ? A.D.pt_act : A.D.ee_act, &s_min);
    if (on && deriv) {
      int slot = atomicAdd(&s_nw, 1);
      if (slot < FUSED_WORK) s_work[slot] = (kind << 30) | j;
      else if (kind == 0) fused_pair_hess0(W, xw, C, q, e, A.D);
      else fused_pair_hess1(W, xw, C, q, e, A.D);
    }
  }
  for (int k = threadIdx.x; k < C.n_gnd[e]; k += blockDim.x)
    ground_item(W, xw, C, deriv, C.gnd_off[e] + k, e, A.T.gnd_val, A.D.gnd_gy, A.D.gnd_hyy, &s_min);
  if (deriv) {
    __syncthreads();
    int nw = min(s_nw, FUSED_WORK);
    int b0 = W.env_aff[e], nbody = W.env_aff[e + 1] - b0;
    int t0 = W.env_tet[e], ntet = W.env_tet[e + 1] - t0;
    int total = nbody + ntet + nw;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      long long c0 = clock64();
      if (i < nbody) {
        fused_body(W, x, W.xhat, h2, 1, b0 + i, A.T.body_val, A.D.body_g, A.D.body_h);
        ft_item(A.timers, FT_IT_BODY, c0);
      } else if (i < nbody + ntet) {
        fused_tet(W, x, h2, 1, t0 + (i - nbody), A.T.tet_val, A.D.tet_g, A.D.tet_h);
      } else {
        int w = s_work[i - nbody - ntet];
        int kind = w >> 30, j = w & ((1 << 30) - 1);
        if (kind == 0) fused_pair_hess0(W, xw, C, pt_off + j, e, A.D);
        else fused_pair_hess1(W, xw, C, ee_off + j, e, A.D);
        ft_item(A.timers, kind == 0 ? FT_IT_PT : FT_IT_EE, c0);
      }
    }
    const Lags& L = A.L;
    for (int k = threadIdx.x; k < L.n[e]; k += blockDim.x) {
      long long c0 = clock64();
      friction_item(W, xw, W.xw0, L, A.h, 1, L.off[e] + k, e, A.T.fr_val, A.D.fr_g, A.D.fr_h);
      ft_item(A.timers, FT_IT_FR, c0);
    }
    for (int k = threadIdx.x; k < L.g_n[e]; k += blockDim.x)
      friction_gnd_item(W, xw, W.xw0, L, A.h, 1, W.env_slot[e] + k, e, A.T.frg_val, A.D.frg_g, A.D.frg_h);
  }
  __syncthreads();
  double m = s_min;
  __syncthreads();
  return m;
}

// any non-finite candidate value of the incoming state (k_start_check)
static __device__ bool env_infeasible(const FusedArgs& A, int e) {
  const Cands& C = A.dc;
  int bad = 0;
  for (int k = threadIdx.x; k < C.n_pt[e]; k += blockDim.x) bad |= isinf(A.T.pt_val[C.pt_off[e] + k]);
  for (int k = threadIdx.x; k < C.n_ee[e]; k += blockDim.x) bad |= isinf(A.T.ee_val[C.ee_off[e] + k]);
  for (int k = threadIdx.x; k < C.n_gnd[e]; k += blockDim.x) bad |= isinf(A.T.gnd_val[C.gnd_off[e] + k]);
  return __syncthreads_or(bad);
}

__device__ __forceinline__ int env_flag_read(const int* f, int e) {
  __shared__ int s_f;
  __syncthreads();
  if (threadIdx.x == 0) s_f = f[e];
  __syncthreads();
  return s_f;
}

// Newton loop of one env (ref solver.py:295-352) from iteration it0 (begin:
// fresh loop state); false on overflow
static __device__ bool env_newton(const FusedArgs& A, int e, double* sm, bool begin = true, int it0 = 0) {
  const World& W = A.W;
  const EnvState& S = A.S;
  __shared__ double s_amin;
  __shared__ int s_ss_ok;  // the env's candidate superset is valid (env_candidates)
  int d0 = W.env_dof[e], d1 = W.env_dof[e + 1];
  int s0 = W.env_slot[e], s1 = W.env_slot[e + 1];
  if (threadIdx.x == 0) s_ss_ok = 0;
  if (threadIdx.x == 0 && begin) newton_begin_env(S, S.al_active, e);
  FT_START;
  for (int it = it0; it < A.max_newton; ++it) {
    if (!env_flag_read(S.newton_active, e)) break;
    // head: DCD candidates at x, derivatives, E0, Newton direction
    FT_MARK(A, FT_OTHER);
    env_world(W, W.x, W.xw, e);
    FT_MARK(A, FT_WORLD);
    if (!env_candidates(A, W.xw, W.xw, A.dc, e, sm, &s_ss_ok)) return false;
    FT_MARK(A, FT_BROAD_DCD);
    double ms = env_terms(A, W.x, W.xw, 1, e);
    FT_MARK(A, FT_TERMS);
    double e0 = env_energy_block(W, W.x, W.xhat, A.T, A.dc, A.L, e);
    if (threadIdx.x == 0) {
      S.min_s[e] = ms;
      S.e0[e] = e0;
    }
    FT_MARK(A, FT_ENERGY);
    dense_solve_block(W, S, A.D, A.dc, A.L, W.x, W.xhat, W.p, W.grad, e, sm,
                      A.timers ? A.timers + FT_DENSE_SUB : nullptr);
    FT_MARK(A, FT_DENSE);
    if (threadIdx.x == 0) {
      newton_check_env(S, A.h, A.newton_tol, e);
      atomicAdd((unsigned long long*)A.stat, 1ull);
    }
    if (!env_flag_read(S.ls_active, e)) continue;  // converged (newton_active cleared)
    // CCD bound along p: sweep boxes of x -> x + p
    for (int i = d0 + threadIdx.x; i < d1; i += blockDim.x) W.xt[i] = __dadd_rn(W.x[i], __dmul_rn(1.0, W.p[i]));
    __syncthreads();
    env_world(W, W.xt, A.xwt, e);
    for (int i = 3 * s0 + threadIdx.x; i < 3 * s1; i += blockDim.x) {
      double dd = __dsub_rn(A.xwt[i], W.xw[i]);
      W.dxw[i] = dd;
      double a = W.xw[i], b = __dadd_rn(W.xw[i], dd);
      A.xlo[i] = fmin(a, b);
      A.xhi[i] = fmax(a, b);
    }
    FT_MARK(A, FT_CCD_PREP);
    if (!env_candidates(A, A.xlo, A.xhi, A.sw, e, sm, &s_ss_ok)) return false;
    FT_MARK(A, FT_BROAD_CCD);
    if (threadIdx.x == 0) s_amin = 1.0;
    __syncthreads();
    {
      const Cands& C = A.sw;
      for (int kind = 0; kind < 2; ++kind) {
        int n = kind == 0 ? C.n_pt[e] : C.n_ee[e];
        long long off = kind == 0 ? C.pt_off[e] : C.ee_off[e];
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
          double a = ccd_pair_item(W, W.xw, W.dxw, C, kind, off + k, A.ccd_cons);
          if (a < 1.0) atomic_min_pos(&s_amin, a);
        }
      }
      for (int k = threadIdx.x; k < C.n_gnd[e]; k += blockDim.x) {
        double a = ccd_ground_item(W, W.xw, W.dxw, C, C.gnd_off[e] + k, e, A.ccd_cons);
        if (a <= 1.0) atomic_min_pos(&s_amin, a);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      S.alpha_max[e] = s_amin;
      ls_begin_env(S, A.ls_count, e);
      A.accepted[e] = 0;
    }
    FT_MARK(A, FT_CCD);
    // backtracking (ref solver.py:257): E(x + α p) <= E0, α halved
    while (env_flag_read(S.ls_active, e)) {
      double a = S.alpha[e];
      double en = ls_value_block(W, A.sw, A.L, W.x, W.p, W.xhat, A.h * A.h, A.h, a, e, sm);
      if (threadIdx.x == 0) {
        S.e_new[e] = en;
        ls_check_env(S, A.ls_count, A.max_halvings, A.accepted, e);
        atomicAdd((unsigned long long*)A.stat + 1, 1ull);
      }
    }
    FT_MARK(A, FT_LS);
    if (env_flag_read(A.accepted, e)) {
      double a = S.alpha[e];
      for (int i = d0 + threadIdx.x; i < d1; i += blockDim.x) W.x[i] = __dadd_rn(W.x[i], __dmul_rn(a, W.p[i]));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && S.newton_active[e]) {  // iteration cap: not converged
    S.converged[e] = 0;
    S.newton_active[e] = 0;
  }
  __syncthreads();
  return true;
}

// whole step of env e; false when a candidate store overflowed
static __device__ bool env_step(const FusedArgs& A, int e, double* sm) {
  const World& W = A.W;
  const EnvState& S = A.S;
  int tid = threadIdx.x;
  int d0 = W.env_dof[e], d1 = W.env_dof[e + 1];
  if (tid == 0) {
    S.newton_iters[e] = 0; S.ccd_calls[e] = 0; S.al_outer[e] = 0; S.ls_failed[e] = 0;
    S.converged[e] = 1; S.err[e] = 0; S.min_s_before[e] = INFINITY; S.gnorm[e] = 0.0;
    A.ok[e] = A.enable[e] ? 1 : 0;
  }
  env_world(W, W.x, W.xw0, e);
  bool ok = env_flag_read(A.ok, e);
  if (ok) {
    // feasibility of the incoming state (ref solver.py:372-385)
    if (!env_broad_sm(W, W.xw0, W.xw0, A.dc, e, sm, A.smem_doubles)) return false;
    env_terms(A, W.x, W.xw0, 0, e);
    if (env_infeasible(A, e)) {
      ok = false;
      if (tid == 0) {
        A.ok[e] = 0;
        S.err[e] = 1;
      }
    }
  }
  // predictor x̂ = x + h v + h² a_g (ref bodies.py:292)
  double h = A.h, hh = h * h;
  for (int i = d0 + tid; i < d1; i += blockDim.x) W.xhat[i] = W.x[i] + h * W.v[i];
  __syncthreads();
  for (int v = W.env_vert[e] + tid; v < W.env_vert[e + 1]; v += blockDim.x) {
    int d = W.vert_dof[v];
    const double* g = W.env_gravity + 3 * e;
    for (int c = 0; c < 3; ++c) W.xhat[d + c] += hh * g[c];
  }
  for (int b = W.env_aff[e] + tid; b < W.env_aff[e + 1]; b += blockDim.x) {
    int o = W.aff_dof[b];
    for (int c = 0; c < 12; ++c) W.xhat[o + c] += hh * W.aff_acc[12 * b + c];
  }
  // fresh AL cycle (ref solver.py:394-400)
  for (int k = W.env_cons[e] + tid; k < W.env_cons[e + 1]; k += blockDim.x) {
    for (int i = 0; i < 12; ++i) {
      W.cons_lam[12 * k + i] = 0.0;
      W.cons_target[12 * k + i] = A.targets[12 * k + i];
    }
    W.cons_kappa[k] = W.cons_kappa0[k];
    W.cons_lastres[k] = INFINITY;
  }
  __syncthreads();
  for (int fp = 0; fp < A.fp_iters; ++fp) {
    if (ok) {
      if (fp == 0) {
        lags_env(W, W.xw0, A.dc, A.L, e);
      } else {
        env_world(W, W.x, W.xw, e);
        if (!env_broad_sm(W, W.xw, W.xw, A.dc, e, sm, A.smem_doubles)) return false;
        lags_env(W, W.xw, A.dc, A.L, e);
      }
    }
    if (tid == 0) S.al_active[e] = ok ? 1 : 0;
    __syncthreads();
    for (int outer = 0; outer < A.al_max_outer; ++outer) {
      if (!env_flag_read(S.al_active, e)) break;
      if (!env_newton(A, e, sm)) return false;
      if (tid == 0) al_update_env(W, S, outer, e);
    }
    if (tid == 0 && S.ls_failed[e]) A.ok[e] = 0;
    ok = env_flag_read(A.ok, e);
  }
  // post-step distance and barrier adaptation (ref solver.py:440-450)
  ok = A.enable[e] && !env_flag_read(S.err, e);
  if (tid == 0) {
    A.ok[e] = ok ? 1 : 0;
    S.min_s[e] = INFINITY;
  }
  __syncthreads();
  if (ok) {
    env_world(W, W.x, W.xw, e);
    if (!env_broad_sm(W, W.xw, W.xw, A.dc, e, sm, A.smem_doubles)) return false;
    double ms = env_terms(A, W.x, W.xw, 0, e);
    if (tid == 0) {
      S.min_s[e] = ms;
      kappa_adapt_env(W, S, e);
    }
  }
  for (int i = d0 + tid; i < d1; i += blockDim.x) {
    if (!ok) W.x[i] = W.x_prev[i];
    else W.v[i] = (W.x[i] - W.x_prev[i]) / h;
  }
  __syncthreads();
  return true;
}

#ifdef IPC_FUSED_TU
// Hand-off from the batched schedule: once few envs are still iterating, each
// continues its Newton loop from iteration it0 in its own CTA (same state in
// EnvState / World, same item functions), without per-iteration launches.
__global__ void __launch_bounds__(256, 1) k_env_newton_rest(FusedArgs A, int it0) {
  ipc_pdl_wait();
  extern __shared__ double sm[];
  __shared__ int s_e;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      int e = A.W.n_env;
      if (!*(volatile int*)A.dc.overflow && !*(volatile int*)A.sw.overflow)
        do {  // heaviest envs first (k_env_order of the last batched iteration)
          e = atomicAdd(A.queue, 1);
          if (e < A.W.n_env && A.order) e = A.order[e];
        } while (e < A.W.n_env && !A.S.newton_active[e]);
      s_e = e;
    }
    __syncthreads();
    int e = s_e;
    if (e >= A.W.n_env) return;
    env_newton(A, e, sm, false, it0);
  }
}

// Asynchronous range: each env runs its own steps k0..k1-1 of the
// device-resident command stream back to back in one CTA (envs never
// interact, so only the per-env step order matters); a contact-onset solve
// in one env overlaps with the other envs' later steps.
__global__ void __launch_bounds__(256, 1) k_env_steps(FusedArgs A, const double* sched, int n_cons, int k0, int k1) {
  ipc_pdl_wait();
  extern __shared__ double sm[];
  __shared__ int s_e;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_e = *(volatile int*)A.dc.overflow || *(volatile int*)A.sw.overflow
                                    ? A.W.n_env : atomicAdd(A.queue, 1);
    __syncthreads();
    int e = s_e;
    if (e >= A.W.n_env) return;
    for (int k = k0; k < k1; ++k) {
      FusedArgs Ak = A;
      Ak.targets = sched + 12 * (size_t)n_cons * k;
      for (int i = A.W.env_dof[e] + threadIdx.x; i < A.W.env_dof[e + 1]; i += blockDim.x) A.W.x_prev[i] = A.W.x[i];
      __syncthreads();
      if (!env_step(Ak, e, sm)) break;
    }
  }
}

__global__ void __launch_bounds__(256, 1) k_env_step(FusedArgs A) {
  ipc_pdl_wait();
  extern __shared__ double sm[];
  __shared__ int s_e;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_e = *(volatile int*)A.dc.overflow || *(volatile int*)A.sw.overflow
                                    ? A.W.n_env : atomicAdd(A.queue, 1);
    __syncthreads();
    int e = s_e;
    if (e >= A.W.n_env) return;
    env_step(A, e, sm);
  }
}

#else
// defined in fused.cu
__global__ void __launch_bounds__(256, 1) k_env_newton_rest(FusedArgs A, int it0);
__global__ void __launch_bounds__(256, 1) k_env_steps(FusedArgs A, const double* sched, int n_cons, int k0, int k1);
__global__ void __launch_bounds__(256, 1) k_env_step(FusedArgs A);
#endif

}  // namespace ipc
