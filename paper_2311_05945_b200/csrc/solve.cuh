// Per-environment reductions, dense Newton solve and the Newton / line-search /
// augmented-Lagrangian bookkeeping of ref solver.py:295-454.
#pragma once
#include "kernels.cuh"

namespace ipc {

constexpr int RED_THREADS = 256;

static __device__ double block_sum(double v, double* sh) {
  // fixed-shape tree: deterministic for a fixed thread->item assignment
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += sh[w];
  __syncthreads();
  return r;  // valid on thread 0
}

static __device__ double block_max(double v, double* sh) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, sh[w]);
  __syncthreads();
  return r;
}

// block_sum over RED_THREADS virtual lanes: part(vt) is virtual lane vt's
// partial sum; thread t holds lanes t, t + blockDim.x, ...; the tree (warp
// shuffles, then the virtual warps in order on thread 0) is block_sum's at
// RED_THREADS threads. Valid on thread 0.
template <class F>
static __device__ double block_sum_virtual(F part, double* sh) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int vt = threadIdx.x; vt < RED_THREADS; vt += blockDim.x) {
    double v = part(vt);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[wid + nw * (vt / blockDim.x)] = v;
  }
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < RED_THREADS / 32; ++w) r += sh[w];
  __syncthreads();
  return r;
}

// Element value buffers of one energy evaluation.
struct Terms {
  double *body_val, *tet_val, *pt_val, *ee_val, *gnd_val, *fr_val, *frg_val;
  const Cands* C;  // candidates the pair values refer to (device copy)
};

// E(x) per env = ½(x−x̂)ᵀM(x−x̂) [soft part here, affine in body_val] + Σ element values
// block function: env e's energy, valid on thread 0
static __device__ double env_energy_block(const World& W, const double* __restrict__ x, const double* __restrict__ xhat,
                                   const Terms& T, const Cands& C, const Lags& L, int e) {
  __shared__ double sh[RED_THREADS / 32];
  double acc = 0.0;
  int tid = threadIdx.x;
  for (int v = W.env_vert[e] + tid; v < W.env_vert[e + 1]; v += RED_THREADS) {
    int d = W.vert_dof[v];
    double m = W.vert_mass[v], s = 0.0;
    for (int c = 0; c < 3; ++c) {
      double dd = x[d + c] - xhat[d + c];
      s += dd * m * dd;
    }
    acc += 0.5 * s;
  }
  for (int b = W.env_aff[e] + tid; b < W.env_aff[e + 1]; b += RED_THREADS) acc += T.body_val[b];
  for (int t = W.env_tet[e] + tid; t < W.env_tet[e + 1]; t += RED_THREADS) acc += T.tet_val[t];
  for (int k = tid; k < C.n_pt[e]; k += RED_THREADS) acc += T.pt_val[C.pt_off[e] + k];
  for (int k = tid; k < C.n_ee[e]; k += RED_THREADS) acc += T.ee_val[C.ee_off[e] + k];
  for (int k = tid; k < C.n_gnd[e]; k += RED_THREADS) acc += T.gnd_val[C.gnd_off[e] + k];
  for (int k = tid; k < L.n[e]; k += RED_THREADS) acc += T.fr_val[L.off[e] + k];
  for (int k = tid; k < L.g_n[e]; k += RED_THREADS) acc += T.frg_val[W.env_slot[e] + k];
  return block_sum(acc, sh);
}

IPC_GLOBAL void __launch_bounds__(RED_THREADS) k_env_energy(World W, const double* __restrict__ x,
                                                             const double* __restrict__ xhat, Terms T,
                                                             Cands C, Lags L, const int* env_flag,
                                                             double* out, const int* order) {
  ipc_pdl_wait();
  int e = order ? order[blockIdx.x] : blockIdx.x;
  if (env_flag && !env_flag[e]) return;
  double s = env_energy_block(W, x, xhat, T, C, L, e);
  if (threadIdx.x == 0) out[e] = s;
}

// ---------------------------------------------------------------------------
// Fused line-search energy: one CTA per (env, trial m) evaluates
// E(x + α 2^-m p) — trial world positions staged in shared memory, then
// inertia, h²-scaled elasticity and orthogonality, kinematic targets, barrier
// over the swept candidates, ground, lagged friction — and reduces it in a
// fixed order. Per-element formulas and operation order are those of the
// element kernels (k_body, k_tet, k_pair_dist, k_ground, k_friction), so the
// values are the same bits; a whole M-trial backtracking round is one launch.
// ---------------------------------------------------------------------------
static __device__ double body_value(const World& W, int b, int e, const double* q, const double* xh, double h2) {
  const double* M = W.aff_M + 144 * b;
  double d[12];
  for (int i = 0; i < 12; ++i) d[i] = q[i] - xh[i];
  double v = 0.0;
  for (int i = 0; i < 12; ++i) {
    double s = 0.0;
    for (int j = 0; j < 12; ++j) s += M[12 * i + j] * d[j];
    v += d[i] * s;
  }
  v *= 0.5;
  double c = W.aff_ortho[b];
  M3 A;
  for (int i = 0; i < 9; ++i) A.m[i] = q[3 + i];
  M3 Mm = m3_mul(A, m3_T(A));
  m3_add_diag(Mm, -1.0);
  double ov = 0.0;
  for (int i = 0; i < 9; ++i) ov += Mm.m[i] * Mm.m[i];
  v += h2 * c * ov;
  for (int k = W.env_cons[e]; k < W.env_cons[e + 1]; ++k) {
    if (W.cons_aff[k] != b) continue;
    double kap = W.cons_kappa[k], sm = sqrt(W.cons_mass[k]);
    const double* tg = W.cons_target + 12 * k;
    const double* lam = W.cons_lam + 12 * k;
    double dd = 0.0, ld = 0.0;
    for (int i = 0; i < 12; ++i) {
      double di = q[i] - tg[i];
      dd += di * di;
      ld += lam[i] * di;
    }
    v += 0.5 * kap * dd - sm * ld;
  }
  return v;
}

__device__ __forceinline__ double axpy_rn(double x, double a, double p) { return __dadd_rn(x, __dmul_rn(a, p)); }

// block function: E(x + a p) of env e (valid on thread 0); sxw: 3 doubles
// per env slot of shared scratch
static __device__ double ls_value_block(const World& W, const Cands& C, const Lags& L, const double* __restrict__ x,
                                 const double* __restrict__ p, const double* __restrict__ xhat, double h2, double h,
                                 double a, int e, double* sxw) {
  __shared__ double sh[RED_THREADS / 32];
  int tid = threadIdx.x;
  int s0 = W.env_slot[e], s1 = W.env_slot[e + 1];
  for (int s = s0 + tid; s < s1; s += blockDim.x) {
    int d = W.slot_dof[s];
    double* o = sxw + 3 * (s - s0);
    if (!W.slot_aff[s]) {
      for (int c = 0; c < 3; ++c) o[c] = axpy_rn(x[d + c], a, p[d + c]);
    } else {
      const double* r = W.slot_rest + 3 * s;
      for (int i = 0; i < 3; ++i) {
        double a0 = axpy_rn(x[d + 3 + 3 * i], a, p[d + 3 + 3 * i]);
        double a1 = axpy_rn(x[d + 4 + 3 * i], a, p[d + 4 + 3 * i]);
        double a2 = axpy_rn(x[d + 5 + 3 * i], a, p[d + 5 + 3 * i]);
        double mm = __dadd_rn(__dadd_rn(__dmul_rn(a0, r[0]), __dmul_rn(a1, r[1])), __dmul_rn(a2, r[2]));
        o[i] = __dadd_rn(axpy_rn(x[d + i], a, p[d + i]), mm);
      }
    }
  }
  __syncthreads();
  auto XW = [&](int s) { return ld3(sxw + 3 * (s - s0)); };
  // every item sweep runs over RED_THREADS virtual lanes (stride RED_THREADS),
  // each thread taking RED_THREADS / blockDim.x of them: the per-lane sums and
  // the reduction tree are those of a RED_THREADS-thread block whatever the
  // launch width, so E(x + a p) has the same bits at 128 and at 256 threads
  auto sweep = [&](int tid) {
    double acc = 0.0;
    for (int v = W.env_vert[e] + tid; v < W.env_vert[e + 1]; v += RED_THREADS) {
      int d = W.vert_dof[v];
      double mass = W.vert_mass[v], sv = 0.0;
      for (int c = 0; c < 3; ++c) {
        double dd = axpy_rn(x[d + c], a, p[d + c]) - xhat[d + c];
        sv += dd * mass * dd;
      }
      acc += 0.5 * sv;
    }
    for (int b = W.env_aff[e] + tid; b < W.env_aff[e + 1]; b += RED_THREADS) {
      int o = W.aff_dof[b];
      double q[12];
      for (int i = 0; i < 12; ++i) q[i] = axpy_rn(x[o + i], a, p[o + i]);
      acc += body_value(W, b, e, q, xhat + o, h2);
    }
    for (int t = W.env_tet[e] + tid; t < W.env_tet[e + 1]; t += RED_THREADS) {
      int4 td = W.tet_dof[t];
      int dv[4] = {td.x, td.y, td.z, td.w};
      V3 X[4];
      for (int k = 0; k < 4; ++k)
        X[k] = v3(axpy_rn(x[dv[k]], a, p[dv[k]]), axpy_rn(x[dv[k] + 1], a, p[dv[k] + 1]),
                  axpy_rn(x[dv[k] + 2], a, p[dv[k] + 2]));
      V3 e1 = X[1] - X[0], e2 = X[2] - X[0], e3 = X[3] - X[0];
      M3 Ds;
      Ds.m[0] = e1.x; Ds.m[1] = e2.x; Ds.m[2] = e3.x;
      Ds.m[3] = e1.y; Ds.m[4] = e2.y; Ds.m[5] = e3.y;
      Ds.m[6] = e1.z; Ds.m[7] = e2.z; Ds.m[8] = e3.z;
      M3 Dmi;
      for (int i = 0; i < 9; ++i) Dmi.m[i] = W.tet_Dminv[9 * t + i];
      M3 F = m3_mul(Ds, Dmi);
      double psi = psi_value(W.tet_model[t], F, W.tet_mu[t], W.tet_lam[t]);
      acc += isinf(psi) ? INFINITY : (h2 * W.tet_vol[t]) * psi;
    }
    double dhat = W.env_dhat[e], shat = dhat * dhat, kappa = W.env_kappa[e];
    for (int kind = 0; kind < 2; ++kind) {
      int n = kind == 0 ? C.n_pt[e] : C.n_ee[e];
      long long off = kind == 0 ? C.pt_off[e] : C.ee_off[e];
      for (int k = tid; k < n; k += RED_THREADS) {
        int2 pr = kind == 0 ? C.pt[off + k] : C.ee[off + k];
        int sl[4];
        pair_slots(W, kind, pr, sl);
        V3 X[4];
        for (int i = 0; i < 4; ++i) X[i] = XW(sl[i]);
        double d2;
        if (kind == 0) d2 = pt_dist2(pt_region(X[0], X[1], X[2], X[3]), X[0], X[1], X[2], X[3]);
        else d2 = ee_dist2(ee_region(X[0], X[1], X[2], X[3], nullptr), X[0], X[1], X[2], X[3]);
        if (!(d2 < shat)) continue;
        if (d2 <= 0.0) {
          acc += INFINITY;
          continue;
        }
        double bv = barrier_val(d2, shat);
        if (kind == 0) {
          acc += kappa * bv;
        } else {
          double mo = mollifier_val(cross2(X[1] - X[0], X[3] - X[2]), 1e-6 * W.edge_len2[pr.x] * W.edge_len2[pr.y]);
          acc += kappa * (mo * bv);
        }
      }
    }
    if (W.env_has_ground[e]) {
      double gy = W.env_ground_y[e];
      for (int k = tid; k < C.n_gnd[e]; k += RED_THREADS) {
        int s = C.gnd[C.gnd_off[e] + k];
        double d = sxw[3 * (s - s0) + 1] - gy;
        if (d <= 0.0) {
          acc += INFINITY;
          continue;
        }
        double ss = d * d;
        if (ss < shat) acc += kappa * barrier_val(ss, shat);
      }
    }
    double eh = W.env_epsv[e] * h, mu = W.env_mu[e];
    for (int k = tid; k < L.n[e]; k += RED_THREADS) {
      long long q = L.off[e] + k;
      int4 s4 = L.slots[q];
      int sl[4] = {s4.x, s4.y, s4.z, s4.w};
      const double* gam = L.gamma + 4 * q;
      const double* T = L.tangent + 6 * q;
      double u3[3] = {0, 0, 0};
      for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) u3[c] += gam[i] * (sxw[3 * (sl[i] - s0) + c] - W.xw0[3 * sl[i] + c]);
      double u0 = T[0] * u3[0] + T[2] * u3[1] + T[4] * u3[2];
      double u1 = T[1] * u3[0] + T[3] * u3[1] + T[5] * u3[2];
      double hu[4];
      acc += smooth_norm(u0, u1, mu * L.lam[q], eh, nullptr, hu);
    }
    for (int k = tid; k < L.g_n[e]; k += RED_THREADS) {
      int q = W.env_slot[e] + k;
      int s = L.g_slot[q];
      double u0 = sxw[3 * (s - s0)] - W.xw0[3 * s], u1 = sxw[3 * (s - s0) + 2] - W.xw0[3 * s + 2];
      double hu[4];
      acc += smooth_norm(u0, u1, mu * L.g_lam[q], eh, nullptr, hu);
    }
    return acc;
  };
  double tot = block_sum_virtual(sweep, sh);
  __syncthreads();  // sxw is reused by the caller
  return tot;
}

constexpr int LS_THREADS = 128;  // launch width of k_ls_value (the sums are RED_THREADS-lane sums)
IPC_GLOBAL void __launch_bounds__(LS_THREADS) k_ls_value(World W, EnvState S, Cands C, Lags L,
                                                           const double* __restrict__ x,
                                                           const double* __restrict__ p,
                                                           const double* __restrict__ xhat, double h2, double h,
                                                           double* e_multi, const int* order, int* ls_count) {
  ipc_pdl_wait();
  extern __shared__ double sxw[];
  int e = order ? order[blockIdx.x] : blockIdx.x, m = blockIdx.y;
  if (!S.ls_active[e]) return;
  double a0;
  if (ls_count) {  // first round of an iteration: the line-search start (k_ls_begin) folded in
    a0 = S.alpha_max[e];
    if (threadIdx.x == 0 && m == 0) {
      S.ccd_calls[e] += 1;
      S.alpha[e] = a0;
      ls_count[e] = 0;
      if (a0 < 1e-12) {  // ALPHA_FLOOR before any evaluation
        S.ls_active[e] = 0;
        S.ls_failed[e] = 1;
        S.converged[e] = 0;
        S.newton_active[e] = 0;
      }
    }
    if (a0 < 1e-12) return;
  } else {
    a0 = S.alpha[e];
  }
  double a = a0 * ldexp(1.0, -m);
  double tot = ls_value_block(W, C, L, x, p, xhat, h2, h, a, e, sxw);
  if (threadIdx.x == 0) e_multi[(long long)m * W.n_env + e] = tot;
}

// Derivative buffers of one assembly.
struct Derivs {
  double *body_g, *body_h;           // 12, 144 per affine body
  double *tet_g, *tet_h;             // 12, 78 per tet
  double *pt_g, *pt_h, *ee_g, *ee_h; // 12, 78 per candidate
  unsigned char *pt_act, *ee_act;
  double *gnd_gy, *gnd_hyy;
  double *fr_g, *fr_h;               // 12, 78 per lag
  double *frg_g, *frg_h;             // 3, 9 per ground lag
};

constexpr int DENSE_THREADS = 256;  // launch width of k_dense_solve and the fused kernels
constexpr int DENSE_MAX_N = 160;  // largest env system on the dense path (engine.cu DENSE_MAX)
constexpr int DENSE_REG_N = 64;   // warp-register substitution up to this size
constexpr int LDL_NB = 12;        // panel width of the blocked LDLᵀ

// dynamic shared memory of the dense solve of an n-DoF env: system n² + 2n,
// the record staging area, the per-DoF group keys
__host__ __device__ inline int dense_smem_doubles(int n);

// ---------------------------------------------------------------------------
// Group-tile dense assembly. Every stencil (tet, active PT / EE pair, ground
// barrier, friction lag, ground friction lag) is a *record* of ≤4 slots with a
// slot-space gradient (3·ns) and Hessian (12x12). The env's DoFs fall into
// *groups* (a soft vertex: 3 DoFs, an affine body: 12), numbered 0..G-1 in DoF
// order; a record touches the groups of its slots (bit mask rm). Records are
// staged REC_CHUNK at a time in shared memory; for every group pair (A ≥ B)
// one warp ballot gives the chunk's records touching it (pm). The lower
// triangle is cut into *tiles* — one row × three consecutive DoFs of one group
// (a translation triple, or one row of A) — each owned by one thread, which
// adds the lifted contribution of exactly the records in pm of its group
// pair, in record order (ref contact.py:346 lifting through J(x0), slots of
// one body merged): deterministic sums and no per-record barrier, and the
// arithmetic of every entry is Σ_a w_a (Σ_b w_b Hs[ia][ib]) per record, the
// same operation order as the entry-owner assembly it replaces.
// ---------------------------------------------------------------------------
constexpr int REC_CHUNK = 32;
struct RecStage {  // carved from dynamic shared memory (rec_stage_doubles)
  double* h;       // [REC_CHUNK][144] slot-space Hessian, unpacked
  double* g;       // [REC_CHUNK][12]
  double* rest;    // [REC_CHUNK][12] slot lever arms (affine slots)
  unsigned long long* rm;  // [REC_CHUNK] groups touched
  int* grp;        // [REC_CHUNK][4] group of the slot (-1: unused)
};
__host__ __device__ constexpr int rec_stage_doubles() { return REC_CHUNK * (144 + 12 + 12 + 1 + 2); }
// per-DoF group key / ordinal (2n ints) and the chunk's pair masks (one u32 per
// group pair, G ≤ n/3 groups)
__host__ __device__ inline int dense_pairs(int n) { return (n / 3) * (n / 3 + 1) / 2; }
__host__ __device__ inline int dense_smem_doubles(int n) {
  return n * n + 2 * n + rec_stage_doubles() + n + (dense_pairs(n) + 1) / 2 + 4;
}
__device__ __forceinline__ RecStage rec_stage(double* base) {
  RecStage R;
  R.h = base;
  R.g = R.h + REC_CHUNK * 144;
  R.rest = R.g + REC_CHUNK * 12;
  R.rm = reinterpret_cast<unsigned long long*>(R.rest + REC_CHUNK * 12);
  R.grp = reinterpret_cast<int*>(R.rm + REC_CHUNK);
  return R;
}

// record types of the virtual index space, in assembly order
enum { REC_TET, REC_PT, REC_EE, REC_GND, REC_FR, REC_FRG };

// lower-triangle tile T -> (row r, first column c0 = 3 t3): rows come in
// triples; row triple R3 holds 3 (R3 + 1) tiles
__device__ __forceinline__ void tile_rc(int T, int* r, int* c0) {
  int R3 = (int)((sqrtf(8.0f * (float)T / 3.0f + 1.0f) - 1.0f) * 0.5f);
  while (3 * (R3 + 1) * (R3 + 2) / 2 <= T) ++R3;
  while (3 * R3 * (R3 + 1) / 2 > T) --R3;
  int rem = T - 3 * R3 * (R3 + 1) / 2;
  *r = 3 * R3 + rem / (R3 + 1);
  *c0 = 3 * (rem % (R3 + 1));
}

// lifted row index of DoF offset R inside its group: coordinate i, lever column
// j (0: translation, 1..3: lever arm component j-1)
__device__ __forceinline__ void lift_ij(int R, int* i, int* j) {
  *i = R < 3 ? R : (R - 3) / 3;
  *j = R < 3 ? 0 : 1 + (R - 3) % 3;
}
__device__ __forceinline__ double lift_w(const RecStage& R, int k, int a, int j) {
  return j == 0 ? 1.0 : R.rest[12 * k + 3 * a + j - 1];
}

static __device__ void assemble_records(const World& W, const Derivs& D, const Cands& C, const Lags& L, int e, int d0,
                                 int n, double* H, double* g, const int* dkey, const int* gi, unsigned* pm,
                                 double* stage_mem) {
  // headers of the window's active records, resolved once by the compacting
  // thread (source, slots, groups): the chunk loop then reads the derivative
  // buffers and lever arms with a single level of indirection
  __shared__ int hsrc[DENSE_THREADS];                 // type << 28 | index in type
  __shared__ int hsl[4 * DENSE_THREADS];              // slots (-1: none / tet vertex)
  __shared__ signed char hgrp[4 * DENSE_THREADS];     // groups (-1: unused)
  __shared__ unsigned long long hrm[DENSE_THREADS];   // groups touched
  __shared__ unsigned char s_pkrc[78];                // packed 12x12 index -> row << 4 | col
  __shared__ int wtot[DENSE_THREADS / 32];
  __shared__ int atot;
  RecStage R = rec_stage(stage_mem);
  int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int t0 = W.env_tet[e], ntet = W.env_tet[e + 1] - t0;
  int npt = C.n_pt[e], nee = C.n_ee[e], ngnd = C.n_gnd[e], nfr = L.n[e], nfrg = L.g_n[e];
  long long pt0 = C.pt_off[e], ee0 = C.ee_off[e], fr0 = L.off[e];
  int gnd0 = C.gnd_off[e], frg0 = W.env_slot[e];
  int lim[6] = {ntet, npt, nee, ngnd, nfr, nfrg};
  int total = ntet + npt + nee + ngnd + nfr + nfrg;
  int G = gi[n - 1] + 1, npairs = G * (G + 1) / 2;
  if (tid < 78) {
    int r = 0, rem = tid;
    while (rem >= 12 - r) rem -= 12 - r++;
    s_pkrc[tid] = (unsigned char)(r << 4 | (r + rem));
  }
  int ntile = 3 * (n / 3) * (n / 3 + 1) / 2;
  const int nthr = blockDim.x, nwarp = nthr >> 5;
  for (int v0 = 0; v0 < total; v0 += nthr) {
    // ordered compaction of the contributing records of this window
    int v = v0 + tid, t = 0, j = v;
    bool on = false;
    if (v < total) {
      while (j >= lim[t]) j -= lim[t++];
      if (t == REC_PT) on = D.pt_act[pt0 + j];
      else if (t == REC_EE) on = D.ee_act[ee0 + j];
      else if (t == REC_GND) on = D.gnd_hyy[gnd0 + j] != 0.0 || D.gnd_gy[gnd0 + j] != 0.0;
      else on = true;
    }
    unsigned m = __ballot_sync(0xffffffffu, on);
    if (lane == 0) wtot[wid] = __popc(m);
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int w = 0; w < nwarp; ++w) {
        int c = wtot[w];
        wtot[w] = acc;
        acc += c;
      }
      atot = acc;
    }
    __syncthreads();
    if (on) {
      int pos = wtot[wid] + __popc(m & ((1u << lane) - 1u));
      hsrc[pos] = (t << 28) | j;
      int sl[4] = {-1, -1, -1, -1}, gg[4] = {-1, -1, -1, -1};
      if (t == REC_TET) {
        int4 td = W.tet_dof[t0 + j];
        gg[0] = gi[td.x - d0]; gg[1] = gi[td.y - d0]; gg[2] = gi[td.z - d0]; gg[3] = gi[td.w - d0];
      } else {
        if (t == REC_PT) {
          int2 pr = C.pt[pt0 + j];
          int3 tv = W.tri_v[pr.y];
          sl[0] = pr.x; sl[1] = tv.x; sl[2] = tv.y; sl[3] = tv.z;
        } else if (t == REC_EE) {
          int2 pr = C.ee[ee0 + j];
          int2 a = W.edge_v[pr.x], b = W.edge_v[pr.y];
          sl[0] = a.x; sl[1] = a.y; sl[2] = b.x; sl[3] = b.y;
        } else if (t == REC_FR) {
          int4 s4 = L.slots[fr0 + j];
          sl[0] = s4.x; sl[1] = s4.y; sl[2] = s4.z; sl[3] = s4.w;
        } else if (t == REC_GND) {
          sl[0] = C.gnd[gnd0 + j];
        } else {
          sl[0] = L.g_slot[frg0 + j];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
          if (sl[a] >= 0) gg[a] = gi[W.slot_dof[sl[a]] - d0];
      }
      unsigned long long rm = 0ull;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        hsl[4 * pos + a] = sl[a];
        hgrp[4 * pos + a] = (signed char)gg[a];
        if (gg[a] >= 0) rm |= 1ull << gg[a];
      }
      hrm[pos] = rm;
    }
    __syncthreads();
    int na = atot;
    for (int k0 = 0; k0 < na; k0 += REC_CHUNK) {
      int nr = min(REC_CHUNK, na - k0);
      if (tid < nr) {
        R.rm[tid] = hrm[k0 + tid];
#pragma unroll
        for (int a = 0; a < 4; ++a) R.grp[4 * tid + a] = hgrp[4 * (k0 + tid) + a];
      }
      // stage Hessians (unpacked), gradients and lever arms (all threads)
      for (int i = tid; i < nr * 102; i += nthr) {
        int k = i / 102, q = i - 102 * k;
        int src = hsrc[k0 + k], t = src >> 28, j = src & ((1 << 28) - 1);
        double val = 0.0;
        if (q < 78) {
          if (t == REC_TET) val = D.tet_h[PK * (long long)(t0 + j) + q];
          else if (t == REC_PT) val = D.pt_h[PK * (pt0 + j) + q];
          else if (t == REC_EE) val = D.ee_h[PK * (ee0 + j) + q];
          else if (t == REC_FR) val = D.fr_h[PK * (fr0 + j) + q];
          else if (q == pk(1, 1) || (t == REC_FRG && (q < 3 || (q >= 12 && q < 14) || q == 23))) {
            // 3x3 slot-space block of a one-slot record in the packed 12x12 layout
            int r = q < 12 ? 0 : (q < 23 ? 1 : 2), c = q < 12 ? q : (q < 23 ? q - 11 : 2);
            if (t == REC_GND) val = D.gnd_hyy[gnd0 + j];
            else val = D.frg_h[9 * (long long)(frg0 + j) + 3 * r + c];
          }
          // packed upper index q -> (r, c), mirrored into the full block
          int rc = s_pkrc[q], r = rc >> 4, c = rc & 15;
          R.h[144 * k + 12 * r + c] = val;
          R.h[144 * k + 12 * c + r] = val;
        } else if (q < 90) {
          int c = q - 78;
          if (t == REC_TET) val = D.tet_g[12 * (long long)(t0 + j) + c];
          else if (t == REC_PT) val = D.pt_g[12 * (pt0 + j) + c];
          else if (t == REC_EE) val = D.ee_g[12 * (ee0 + j) + c];
          else if (t == REC_FR) val = D.fr_g[12 * (fr0 + j) + c];
          else if (t == REC_GND) val = c == 1 ? D.gnd_gy[gnd0 + j] : 0.0;
          else if (c < 3) val = D.frg_g[3 * (long long)(frg0 + j) + c];
          R.g[12 * k + c] = val;
        } else {
          int a = (q - 90) / 3, c = q - 90 - 3 * a;
          int sa = hsl[4 * (k0 + k) + a];
          if (sa >= 0) R.rest[12 * k + 3 * a + c] = W.slot_rest[3 * sa + c];
        }
      }
      __syncthreads();
      // records of the chunk touching each group pair (A ≥ B)
      for (int P = wid; P < npairs; P += nwarp) {
        int A = (int)((sqrtf(8.0f * (float)P + 1.0f) - 1.0f) * 0.5f);
        while ((A + 1) * (A + 2) / 2 <= P) ++A;
        while (A * (A + 1) / 2 > P) --A;
        int B = P - A * (A + 1) / 2;
        bool t = false;
        if (lane < nr) {
          unsigned long long rm = R.rm[lane];
          t = ((rm >> A) & (rm >> B) & 1ull) != 0ull;
        }
        unsigned bm = __ballot_sync(0xffffffffu, t);
        if (lane == 0) pm[P] = bm;
      }
      __syncthreads();
      // tile owners: H[r][c0..c0+2] += Σ_a w_a(r) Σ_b w_b(c) Hs[ia][ib] per record
      for (int T = tid; T < ntile; T += nthr) {
        int r, c0;
        tile_rc(T, &r, &c0);
        int gr = gi[r], gc = gi[c0];
        int iR, jR, iC, jC;
        lift_ij(r - dkey[r], &iR, &jR);
        lift_ij(c0 - dkey[c0], &iC, &jC);
        unsigned bm = pm[gr * (gr + 1) / 2 + gc];
        if (!bm) continue;
        int ncol = min(3, r - c0 + 1);  // columns c0..c0+ncol-1 are in the lower triangle
        double h0 = H[r * n + c0], h1 = ncol > 1 ? H[r * n + c0 + 1] : 0.0, h2 = ncol > 2 ? H[r * n + c0 + 2] : 0.0;
        while (bm) {
          int k = __ffs(bm) - 1;
          bm &= bm - 1;
          const double* hk = R.h + 144 * k;
          double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            if (R.grp[4 * k + a] != gr) continue;
            double wa = lift_w(R, k, a, jR);
            const double* hrow = hk + 12 * (3 * a + iR);
            double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              if (R.grp[4 * k + b] != gc) continue;
              if (jC == 0) {  // translation triple: columns (i = 0..2, j = 0)
                s0 += 1.0 * hrow[3 * b];
                s1 += 1.0 * hrow[3 * b + 1];
                s2 += 1.0 * hrow[3 * b + 2];
              } else {  // row iC of A: columns (i = iC, j = 1..3)
                double hv = hrow[3 * b + iC];
                s0 += lift_w(R, k, b, 1) * hv;
                s1 += lift_w(R, k, b, 2) * hv;
                s2 += lift_w(R, k, b, 3) * hv;
              }
            }
            acc0 += wa * s0;
            acc1 += wa * s1;
            acc2 += wa * s2;
          }
          h0 += acc0;
          h1 += acc1;
          h2 += acc2;
        }
        H[r * n + c0] = h0;
        if (ncol > 1) H[r * n + c0 + 1] = h1;
        if (ncol > 2) H[r * n + c0 + 2] = h2;
      }
      // owners of the gradient: records touching the DoF's group
      for (int r = tid; r < n; r += nthr) {
        int gr = gi[r], iR, jR;
        lift_ij(r - dkey[r], &iR, &jR);
        unsigned bm = pm[gr * (gr + 1) / 2 + gr];
        double gv = g[r];
        while (bm) {
          int k = __ffs(bm) - 1;
          bm &= bm - 1;
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            if (R.grp[4 * k + a] != gr) continue;
            acc += lift_w(R, k, a, jR) * R.g[12 * k + 3 * a + iR];
          }
          gv += acc;
        }
        g[r] = gv;
      }
      __syncthreads();
    }
  }
}

// Forward / backward substitution of the factored small env system by one
// warp (y in two registers per lane, the pivot / column values broadcast by
// shuffles). Its own function so that the caller's register pressure (the
// fused kernels run at 255) cannot turn the loop's predicated updates into
// branches and re-materialised special-register reads (8x slower, measured).
static __device__ __noinline__ void warp_substitute(const double* H, const double* dinv, double* y, int n) {
  const unsigned FULL = 0xffffffffu;
  __syncwarp();  // enter converged: a diverged warp takes every SHFL's slow path (measured 7x)
  int lane = threadIdx.x & 31, i1 = lane + 32;
  double y0 = lane < n ? y[lane] : 0.0, y1 = i1 < n ? y[i1] : 0.0;
  // forward: L' u = -g (y holds -g); column k of L' is read from its mirror
  // in the upper triangle (row k: consecutive, conflict-free)
  for (int k = 0; k < n; ++k) {
    double uk = __shfl_sync(FULL, k < 32 ? y0 : y1, k & 31);
    double dk = dinv[k];
    double c0 = (lane > k && lane < n) ? H[k * n + lane] * dk : 0.0;
    double c1 = (i1 > k && i1 < n) ? H[k * n + i1] * dk : 0.0;
    y0 -= c0 * uk;
    y1 -= c1 * uk;
  }
  if (lane < n) y0 *= dinv[lane];
  if (i1 < n) y1 *= dinv[i1];
  // backward: L'ᵀ p = D⁻¹ u
  double dl0 = lane < n ? dinv[lane] : 0.0, dl1 = i1 < n ? dinv[i1] : 0.0;
  for (int k = n - 1; k >= 0; --k) {
    double xk = __shfl_sync(FULL, k < 32 ? y0 : y1, k & 31);
    double c0 = lane < k ? H[k * n + lane] * dl0 : 0.0;
    double c1 = i1 < k ? H[k * n + i1] * dl1 : 0.0;
    y0 -= c0 * xk;
    y1 -= c1 * xk;
  }
  if (lane < n) y[lane] = y0;
  if (i1 < n) y[i1] = y1;
}

// Assemble the env's dense Hessian/gradient, Cholesky-solve H p = −g with the
// gradient fallback of ref solver.py:241, write p, ‖p‖∞, ‖g‖∞.
// block function: assemble + solve env e; sm holds n² + 2n doubles
// dtm (optional phase timers, IPC_FUSED_TIMERS=1): SM cycles of the solve's
// sub-phases — setup, record assembly, gradient norm, LDLᵀ, substitution, tail
static __device__ void dense_solve_block(const World& W, const EnvState& S, const Derivs& D, const Cands& C,
                                  const Lags& L, const double* __restrict__ x, const double* __restrict__ xhat,
                                  double* p_out, double* g_out, int e, double* sm, long long* dtm = nullptr) {
  long long dt0 = dtm ? clock64() : 0;
  auto dmark = [&](int k) {
    if (dtm) {
      __syncthreads();
      if (threadIdx.x < 32) {  // all of warp 0 (a lane-0 branch would leave it diverged)
        long long now = clock64();
        atomicAdd((unsigned long long*)dtm + k, threadIdx.x == 0 ? (unsigned long long)(now - dt0) : 0ull);
        dt0 = now;
      }
    }
  };
  __shared__ double red[DENSE_THREADS / 32];
  __shared__ int fail;
  int d0 = W.env_dof[e], n = W.env_dof[e + 1] - d0;
  double* H = sm;
  double* g = sm + n * n;
  double* y = g + n;
  int tid = threadIdx.x;
  for (int i = tid; i < n * n; i += blockDim.x) H[i] = 0.0;
  for (int i = tid; i < n; i += blockDim.x) g[i] = 0.0;
  if (tid == 0) fail = 0;
  __syncthreads();
  // soft inertia (diagonal) and affine per-body blocks: disjoint entries
  for (int v = W.env_vert[e] + tid; v < W.env_vert[e + 1]; v += blockDim.x) {
    int d = W.vert_dof[v] - d0;
    double m = W.vert_mass[v];
    for (int c = 0; c < 3; ++c) {
      H[(d + c) * n + d + c] += m;
      g[d + c] += m * (x[d0 + d + c] - xhat[d0 + d + c]);
    }
  }
  for (int b = W.env_aff[e]; b < W.env_aff[e + 1]; ++b) {
    int o = W.aff_dof[b] - d0;
    for (int i = tid; i < 144; i += blockDim.x) H[(o + i / 12) * n + o + i % 12] += D.body_h[144 * b + i];
    for (int i = tid; i < 12; i += blockDim.x) g[o + i] += D.body_g[12 * b + i];
  }
  __syncthreads();
  // group key (local DoF offset of the owning soft vertex / affine body) of
  // every DoF, then the record-parallel assembly of every stencil
  int* dkey = reinterpret_cast<int*>(y + n + rec_stage_doubles());
  int* gi = dkey + n;
  unsigned* pm = reinterpret_cast<unsigned*>(gi + n);
  for (int v = W.env_vert[e] + tid; v < W.env_vert[e + 1]; v += blockDim.x) {
    int d = W.vert_dof[v] - d0;
    for (int c = 0; c < 3; ++c) dkey[d + c] = d;
  }
  for (int b = W.env_aff[e]; b < W.env_aff[e + 1]; ++b) {
    int o = W.aff_dof[b] - d0;
    for (int i = tid; i < 12; i += blockDim.x) dkey[o + i] = o;
  }
  __syncthreads();
  // group ordinal of every DoF: the number of group starts (dkey[d] == d) before it
  {
    __shared__ unsigned sb[DENSE_MAX_N / 32 + 1];
    int nw = (n + 31) / 32;
    for (int w0 = 0; w0 < nw; w0 += (int)(blockDim.x >> 5)) {
      int d = 32 * (w0 + (tid >> 5)) + (tid & 31);
      unsigned b = __ballot_sync(0xffffffffu, d < n && dkey[d] == d);
      if ((tid & 31) == 0 && w0 + (tid >> 5) < nw) sb[w0 + (tid >> 5)] = b;
    }
    __syncthreads();
    for (int d = tid; d < n; d += blockDim.x) {
      int c = 0;
      for (int w = 0; w < d / 32; ++w) c += __popc(sb[w]);
      c += __popc(sb[d / 32] & (0xffffffffu >> (31 - (d & 31))));
      gi[d] = c - 1;
    }
    __syncthreads();
  }
  dmark(0);
  assemble_records(W, D, C, L, e, d0, n, H, g, dkey, gi, pm, y + n);
  dmark(1);
  // keep the gradient for the report / descent test
  double gmax = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    g_out[d0 + i] = g[i];
    gmax = fmax(gmax, fabs(g[i]));
    y[i] = -g[i];
  }
  double gn = block_max(gmax, red);
  if (tid == 0) S.gnorm[e] = gn;
  __syncthreads();
  dmark(2);
  // LDLᵀ without scaling: after step k the lower column c_k = H[k+1:, k] and
  // pivot a_k = H[k][k] give H = Σ c_k c_kᵀ / a_k, i.e. L' = c / a (unit
  // lower), D = diag(a); same factorization as Cholesky (SPD input).
  __shared__ double s_dinv[DENSE_MAX_N];
  if (n <= DENSE_REG_N) {
    // Small envs (every grasp env: 4 affine bodies, n = 48): 3x3 register
    // tiles of the lower triangle, one per thread, and 3-column panels. Per
    // panel the diagonal tile factors its 3 columns, the tiles below it apply
    // those 3 steps to their rows, and every trailing tile takes the rank-3
    // update from the published panel — two barriers per 3 columns. Each
    // entry receives exactly the column-by-column sequence
    // a_ij -= (c_i / a_k) c_j, k increasing, with the same operands.
    __shared__ double pan[2][3 * DENSE_REG_N];  // panel columns, double-buffered
    const int T3 = n / 3, ntile = T3 * (T3 + 1) / 2;
    int I = -1, J = -1;
    double t[9];
    if (tid < ntile) {
      I = (int)((sqrtf(8.0f * (float)tid + 1.0f) - 1.0f) * 0.5f);
      while ((I + 1) * (I + 2) / 2 <= tid) ++I;
      while (I * (I + 1) / 2 > tid) --I;
      J = tid - I * (I + 1) / 2;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) t[3 * a + b] = (I > J || b <= a) ? H[(3 * I + a) * n + 3 * J + b] : 0.0;
    }
    for (int P = 0; P < T3; ++P) {
      double* pc = pan[P & 1];
      if (I == P && J == P) {  // diagonal tile: its three steps
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          double akk = t[4 * k];
          double inv = __drcp_rn(akk);  // correctly rounded: the bits of 1.0 / akk
          s_dinv[3 * P + k] = inv;
          if (!(akk > 0.0)) fail = 1;
#pragma unroll
          for (int a = k + 1; a < 3; ++a)
#pragma unroll
            for (int b = k + 1; b <= a; ++b) t[3 * a + b] -= (t[3 * a + k] * inv) * t[3 * b + k];
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b <= a; ++b) pc[3 * (3 * P + a) + b] = t[3 * a + b];
      }
      __syncthreads();
      if (J == P && I > P) {  // panel tile: the three steps on its rows
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          double inv = s_dinv[3 * P + k];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = k + 1; b < 3; ++b) t[3 * a + b] -= (t[3 * a + k] * inv) * pc[3 * (3 * P + b) + k];
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) pc[9 * I + q] = t[q];
      }
      __syncthreads();
      if (J > P) {  // trailing tile: rank-3 update, steps in order
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          double inv = s_dinv[3 * P + k];
          double ci[3], cj[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            ci[a] = pc[3 * (3 * I + a) + k];
            cj[a] = pc[3 * (3 * J + a) + k];
          }
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
              if (I > J || b <= a) t[3 * a + b] -= (ci[a] * inv) * cj[b];
        }
      }
    }
    if (tid < ntile) {  // L' and D, mirrored into the upper triangle for the forward substitution
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          if (I > J || b <= a) {
            H[(3 * I + a) * n + 3 * J + b] = t[3 * a + b];
            H[(3 * J + b) * n + 3 * I + a] = t[3 * a + b];
          }
    }
    __syncthreads();
  } else {
  // Blocked right-looking form: panels of LDL_NB columns; warp 0 factors the
    // diagonal block, one thread per row applies the panel's steps to the rows
    // below it, then every trailing entry takes the panel's rank-LDL_NB update.
    // Each entry receives exactly the column-by-column update sequence
    // a_ij -= (c_i / a_k) c_j, k increasing, with the same operands (so the same
    // bits), at three block barriers per panel instead of one per column.
    for (int K0 = 0; K0 < n; K0 += LDL_NB) {
      int K1 = min(n, K0 + LDL_NB);
      if (tid < 32) {
        for (int k = K0; k < K1; ++k) {
          double akk = H[k * n + k];
          double inv = __drcp_rn(akk);  // correctly rounded: the bits of 1.0 / akk
          if (tid == 0) {
            s_dinv[k] = inv;
            if (!(akk > 0.0)) fail = 1;
          }
          int i = K0 + tid;
          if (i > k && i < K1) {
            double ci = H[i * n + k] * inv;
            for (int j = k + 1; j <= i; ++j) H[i * n + j] -= ci * H[j * n + k];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      for (int i = K1 + tid; i < n; i += blockDim.x) {
        for (int k = K0; k < K1; ++k) {
          double ci = H[i * n + k] * s_dinv[k];
          for (int j = k + 1; j < K1; ++j) H[i * n + j] -= ci * H[j * n + k];
        }
      }
      __syncthreads();
      int m = n - K1;
      for (int idx = tid; idx < m * (m + 1) / 2; idx += blockDim.x) {
        int ii = (int)((sqrtf(8.0f * (float)idx + 1.0f) - 1.0f) * 0.5f);
        while ((ii + 1) * (ii + 2) / 2 <= idx) ++ii;
        while (ii * (ii + 1) / 2 > idx) --ii;
        int i = K1 + ii, j = K1 + (idx - ii * (ii + 1) / 2);
        double a = H[i * n + j];
        for (int k = K0; k < K1; ++k) a -= (H[i * n + k] * s_dinv[k]) * H[j * n + k];
        H[i * n + j] = a;
      }
      __syncthreads();
    }
  }
  dmark(3);
  if (n <= DENSE_REG_N) {
    // Small envs (every grasp env: 4 affine bodies, n = 48): warp 0
    // substitutes with y in registers, the pivot / column values broadcast by
    // shuffles.
    if (tid < 32) warp_substitute(H, s_dinv, y, n);
    __syncthreads();
    dmark(4);
  } else {
    // forward: L' u = -g  (y holds -g)
    for (int k = 0; k < n; ++k) {
      double uk = y[k], inv = 1.0 / H[k * n + k];
      for (int i = k + 1 + tid; i < n; i += blockDim.x) y[i] -= (H[i * n + k] * inv) * uk;
      __syncthreads();
    }
    for (int i = tid; i < n; i += blockDim.x) y[i] /= H[i * n + i];
    __syncthreads();
    // backward: L'ᵀ p = D⁻¹ u
    for (int k = n - 1; k >= 0; --k) {
      double xk = y[k];
      for (int i = tid; i < k; i += blockDim.x) y[i] -= (H[k * n + i] / H[i * n + i]) * xk;
      __syncthreads();
    }
  }
  double pg = 0.0;
  int bad = 0;
  for (int i = tid; i < n; i += blockDim.x) {
    pg += y[i] * g[i];
    if (!isfinite(y[i])) bad = 1;
  }
  double spg = block_sum(pg, red);
  __shared__ int nonfinite;
  if (tid == 0) nonfinite = 0;
  __syncthreads();
  if (bad) atomicExch(&nonfinite, 1);
  __syncthreads();
  __shared__ int use_grad;
  if (tid == 0) use_grad = fail || nonfinite || spg > 0.0;
  __syncthreads();
  double pmax = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    double pi = use_grad ? -g[i] : y[i];
    p_out[d0 + i] = pi;
    pmax = fmax(pmax, fabs(pi));
  }
  double pn = block_max(pmax, red);
  if (tid == 0) S.pnorm[e] = pn;
  dmark(5);
}

// Order in which the per-env CTAs of the dense solve start: most records
// first (a heavy env starting in the last wave is the kernel's tail), active
// before converged envs, ties by env index. Keys (records << 12 | (4095 -
// env)) are unique, so an env's slot is its rank = the number of larger keys:
// ORDER_ENVS envs per CTA, one warp per env counting over the keys staged in
// shared memory (no sorting network, no serial stages; grid = n_env / 32).
// Identity beyond 4096 envs.
constexpr int ORDER_MAX = 4096;
constexpr int ORDER_ENVS = 32;  // envs ranked per CTA (one warp each)
IPC_GLOBAL void __launch_bounds__(ORDER_ENVS * 32) k_env_order(int n_env, const int* active, Cands C, Lags L,
                                                               int* order) {
  ipc_pdl_wait();
  __shared__ long long key[ORDER_MAX];
  int tid = threadIdx.x;
  if (n_env > ORDER_MAX) {
    for (int e = blockIdx.x * blockDim.x + tid; e < n_env; e += gridDim.x * blockDim.x) order[e] = e;
    return;
  }
  for (int i = tid; i < n_env; i += blockDim.x) {
    long long w = active[i] ? 1 + (long long)C.n_pt[i] + C.n_ee[i] + L.n[i] : 0;
    key[i] = (w << 12) | (ORDER_MAX - 1 - i);
  }
  __syncthreads();
  int lane = tid & 31, e = blockIdx.x * ORDER_ENVS + (tid >> 5);
  if (e >= n_env) return;
  long long k = key[e];
  unsigned cnt = 0;
  for (int j = lane; j < n_env; j += 32) cnt += key[j] > k;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) order[cnt] = e;
}

IPC_GLOBAL void __launch_bounds__(DENSE_THREADS) k_dense_solve(World W, EnvState S, Derivs D, Cands C,
                                                                Lags L, const double* __restrict__ x,
                                                                const double* __restrict__ xhat,
                                                                double* p_out, double* g_out, long long* dtm,
                                                                const int* order) {
  ipc_pdl_wait();
  extern __shared__ double sm[];
  int e = order ? order[blockIdx.x] : blockIdx.x;
  if (!S.newton_active[e]) return;
  dense_solve_block(W, S, D, C, L, x, xhat, p_out, g_out, e, sm, dtm);
}

// ---------------------------------------------------------------------------
// bookkeeping kernels (one thread per env)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void newton_begin_env(const EnvState& S, const int* flag, int e) {
  int on = flag[e] ? 1 : 0;
  S.newton_active[e] = on;
  if (on) {
    S.small_run[e] = 0;
    S.prev_pnorm[e] = INFINITY;
  }
}
IPC_GLOBAL void k_newton_begin(int n_env, EnvState S, const int* flag) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n_env) newton_begin_env(S, flag, e);
}

// two-consecutive-small-steps rule of ref solver.py:326-332
__device__ __forceinline__ void newton_check_env(const EnvState& S, double h, double tol, int e) {
  if (!S.newton_active[e]) {
    S.ls_active[e] = 0;
    return;
  }
  S.newton_iters[e] += 1;
  S.min_s_before[e] = fmin(S.min_s_before[e], S.min_s[e]);
  double pn = S.pnorm[e];
  bool small = __ddiv_rn(pn, h) <= tol;
  int run = S.small_run[e];
  if (small && run >= 1 && (pn <= S.prev_pnorm[e] || run >= 7)) {
    S.newton_active[e] = 0;
    S.ls_active[e] = 0;
    return;
  }
  S.small_run[e] = small ? run + 1 : 0;
  S.prev_pnorm[e] = pn;
  S.ls_active[e] = 1;
  S.alpha_max[e] = 1.0;
}
IPC_GLOBAL void k_newton_check(int n_env, EnvState S, double h, double tol) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n_env) newton_check_env(S, h, tol, e);
}

__device__ __forceinline__ void ls_begin_env(const EnvState& S, int* ls_count, int e) {
  if (!S.ls_active[e]) return;
  S.ccd_calls[e] += 1;
  S.alpha[e] = S.alpha_max[e];
  ls_count[e] = 0;
  if (S.alpha[e] < 1e-12) {  // ALPHA_FLOOR before any evaluation
    S.ls_active[e] = 0;
    S.ls_failed[e] = 1;
    S.converged[e] = 0;
    S.newton_active[e] = 0;
  }
}
IPC_GLOBAL void k_ls_begin(int n_env, EnvState S, int* ls_count) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n_env) ls_begin_env(S, ls_count, e);
}

// Armijo with c = 0 (ref solver.py:257); accepted envs copy xt -> x
__device__ __forceinline__ void ls_check_env(const EnvState& S, int* ls_count, int max_halvings, int* accepted,
                                             int e) {
  accepted[e] = 0;
  if (!S.ls_active[e]) return;
  if (S.e_new[e] <= S.e0[e]) {
    accepted[e] = 1;
    S.ls_active[e] = 0;
    return;
  }
  double a = S.alpha[e] * 0.5;
  int c = ls_count[e] + 1;
  ls_count[e] = c;
  S.alpha[e] = a;
  if (c >= max_halvings || a < 1e-12) {
    S.ls_active[e] = 0;
    S.ls_failed[e] = 1;
    S.converged[e] = 0;
    S.newton_active[e] = 0;
  }
}
IPC_GLOBAL void k_ls_check(World W, EnvState S, int* ls_count, int max_halvings, int* accepted) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < W.n_env) ls_check_env(S, ls_count, max_halvings, accepted, e);
}

// speculative backtracking: trials m = 0..M-1 evaluated E(x + α 2^-m p) into
// e_multi[m * n_env + e]; take the first trial the sequential search would
// have accepted (same floor / halving-count rules, ref solver.py:257-272)
__device__ __forceinline__ void ls_check_multi_env(const World& W, const EnvState& S, int* ls_count,
                                                   int max_halvings, int M, const double* e_multi, int* accepted,
                                                   int e) {
  accepted[e] = 0;
  if (!S.ls_active[e]) return;
  double a = S.alpha[e];
  int c = ls_count[e];
  for (int m = 0; m < M; ++m) {
    if (c >= max_halvings || a < 1e-12) {
      S.ls_active[e] = 0;
      S.ls_failed[e] = 1;
      S.converged[e] = 0;
      S.newton_active[e] = 0;
      return;
    }
    if (e_multi[(long long)m * W.n_env + e] <= S.e0[e]) {
      S.alpha[e] = a;
      accepted[e] = 1;
      S.ls_active[e] = 0;
      return;
    }
    a *= 0.5;
    ++c;
  }
  S.alpha[e] = a;
  ls_count[e] = c;
  if (c >= max_halvings || a < 1e-12) {
    S.ls_active[e] = 0;
    S.ls_failed[e] = 1;
    S.converged[e] = 0;
    S.newton_active[e] = 0;
  }
}
// the round's Armijo check and, for an accepted env, x += alpha p over its
// DoFs (the per-env check and k_axpy_env in one launch, one CTA per env;
// same operations, same bits)
IPC_GLOBAL void k_ls_check_apply(World W, EnvState S, int* ls_count, int max_halvings, int M,
                                 const double* e_multi, int* accepted, double* x, const double* __restrict__ p) {
  ipc_pdl_wait();
  __shared__ int acc;
  int e = blockIdx.x;
  if (threadIdx.x == 0) {
    ls_check_multi_env(W, S, ls_count, max_halvings, M, e_multi, accepted, e);
    acc = accepted[e];
  }
  __syncthreads();
  if (!acc) return;
  double a = S.alpha[e] * 1.0;
  for (int i = W.env_dof[e] + threadIdx.x; i < W.env_dof[e + 1]; i += blockDim.x)
    x[i] = __dadd_rn(x[i], __dmul_rn(a, p[i]));
}

IPC_GLOBAL void k_copy_env(World W, const double* src, double* dst, const int* flag) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W.n_dof) return;
  if (flag[W.dof_env[i]]) dst[i] = src[i];
}

// multiplier update after each inner solve (ref constraints.py:215, solver.py:414-434)
__device__ __forceinline__ void al_update_env(const World& W, const EnvState& S, int outer, int e) {
  if (!S.al_active[e]) return;
  double res = 0.0;
  for (int k = W.env_cons[e]; k < W.env_cons[e + 1]; ++k) {
    int o = W.aff_dof[W.cons_aff[k]];
    double dd = 0.0;
    double d[12];
    for (int i = 0; i < 12; ++i) {
      d[i] = W.x[o + i] - W.cons_target[12 * k + i];
      dd += d[i] * d[i];
    }
    double r = sqrt(dd);
    double kap = W.cons_kappa[k], sm = sqrt(W.cons_mass[k]);
    for (int i = 0; i < 12; ++i) W.cons_lam[12 * k + i] -= kap * d[i] / sm;
    if (r > 0.5 * W.cons_lastres[k]) W.cons_kappa[k] = fmin(2.0 * kap, 1e6 * W.cons_kappa0[k]);
    W.cons_lastres[k] = r;
    res = fmax(res, r);
  }
  S.res[e] = res;
  S.al_outer[e] = max(S.al_outer[e], outer + 1);
  bool has = W.env_cons[e + 1] > W.env_cons[e];
  if (!has || res <= 1e-6 || S.ls_failed[e]) S.al_active[e] = 0;
}
IPC_GLOBAL void k_al_update(World W, EnvState S, int outer) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < W.n_env) al_update_env(W, S, outer, e);
}

IPC_GLOBAL void k_cons_reset(World W, const double* targets) {
  ipc_pdl_wait();
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= W.n_cons) return;
  for (int i = 0; i < 12; ++i) {
    W.cons_lam[12 * k + i] = 0.0;
    W.cons_target[12 * k + i] = targets[12 * k + i];
  }
  W.cons_kappa[k] = W.cons_kappa0[k];
  W.cons_lastres[k] = INFINITY;
}

// x̂ = x + h v + h² a_g (ref bodies.py:292)
IPC_GLOBAL void k_predictor(World W, double h) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < W.n_dof) W.xhat[i] = W.x[i] + h * W.v[i];
}
IPC_GLOBAL void k_predictor_forces(World W, double h) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double hh = h * h;
  if (i < W.n_vert) {
    int d = W.vert_dof[i];
    const double* g = W.env_gravity + 3 * W.vert_env[i];
    for (int c = 0; c < 3; ++c) W.xhat[d + c] += hh * g[c];
  }
  if (i < W.n_aff) {
    int o = W.aff_dof[i];
    for (int c = 0; c < 12; ++c) W.xhat[o + c] += hh * W.aff_acc[12 * i + c];
  }
}

IPC_GLOBAL void k_finalize(World W, double h, const int* ok) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W.n_dof) return;
  int e = W.dof_env[i];
  if (!ok[e]) {  // failed to start: leave state untouched
    W.x[i] = W.x_prev[i];
    return;
  }
  W.v[i] = (W.x[i] - W.x_prev[i]) / h;
}

// post-step: min distance + κ doubling (ref barrier.py:85, solver.py:440-450)
__device__ __forceinline__ void kappa_adapt_env(const World& W, const EnvState& S, int e) {
  double md = isinf(S.min_s[e]) ? INFINITY : sqrt(S.min_s[e]);
  S.min_s[e] = md;  // now a distance
  double k = W.env_kappa[e], k0 = W.env_kappa0[e], dhat = W.env_dhat[e];
  if (md < 1e-4 * dhat && k < 1e8 * k0) W.env_kappa[e] = fmin(2.0 * k, 1e8 * k0);
}
IPC_GLOBAL void k_kappa_adapt(World W, EnvState S, const int* ok) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < W.n_env && ok[e]) kappa_adapt_env(W, S, e);
}

IPC_GLOBAL void k_fill(int n, double* a, double v) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
IPC_GLOBAL void k_fill_flag(int n, double* a, double v, const int* flag) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) a[i] = v;
}
IPC_GLOBAL void k_fill_int(int n, int* a, int v) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
IPC_GLOBAL void k_count(int n, const int* flag, int* out) {
  ipc_pdl_wait();
  __shared__ int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (flag[i]) atomicAdd(&s, 1);
  __syncthreads();
  if (threadIdx.x == 0) *out = s;
}
IPC_GLOBAL void k_sweep_box(int n, const double* xw, const double* dxw, double* lo, double* hi) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  double a = xw[i], b = __dadd_rn(xw[i], dxw[i]);
  lo[i] = fmin(a, b);
  hi[i] = fmax(a, b);
}

}  // namespace ipc
