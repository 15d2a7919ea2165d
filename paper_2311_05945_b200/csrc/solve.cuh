// Per-environment reductions, dense Newton solve and the Newton / line-search /
// augmented-Lagrangian bookkeeping of ref solver.py:295-454.
#pragma once
#include "kernels.cuh"

namespace ipc {

constexpr int RED_THREADS = 256;

__device__ double block_sum(double v, double* sh) {
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

__device__ double block_max(double v, double* sh) {
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

// Element value buffers of one energy evaluation.
struct Terms {
  double *body_val, *tet_val, *pt_val, *ee_val, *gnd_val, *fr_val, *frg_val;
  const Cands* C;  // candidates the pair values refer to (device copy)
};

// E(x) per env = ½(x−x̂)ᵀM(x−x̂) [soft part here, affine in body_val] + Σ element values
__global__ void __launch_bounds__(RED_THREADS) k_env_energy(World W, const double* __restrict__ x,
                                                             const double* __restrict__ xhat, Terms T,
                                                             Cands C, Lags L, const int* env_flag,
                                                             double* out) {
  __shared__ double sh[RED_THREADS / 32];
  int e = blockIdx.x;
  if (env_flag && !env_flag[e]) return;
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
  double s = block_sum(acc, sh);
  if (tid == 0) out[e] = s;
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

// Add one stencil (ns slots, slot-space gradient gs[3ns] and Hessian hs)
// to the dense env system, lifting affine slots through J(x0) and merging
// slots that ride the same body (ref contact.py:346). One call = one element;
// each thread owns distinct output entries, so no atomics are needed.
template <typename HGet>
__device__ void add_stencil(const World& W, int d0, int n, double* H, double* g, int ns, const int* sl,
                            const double* gs, HGet hget) {
  int key[4], wid[4], grp[4], gstart[5];
  int ng = 0;
  for (int a = 0; a < ns; ++a) {
    int s = sl[a];
    int k = W.slot_dof[s] - d0;
    bool aff = W.slot_aff[s];
    int gi = -1;
    for (int q = 0; q < ng; ++q)
      if (key[q] == k) gi = q;
    if (gi < 0) {
      gi = ng++;
      key[gi] = k;
      wid[gi] = aff ? 12 : 3;
    }
    grp[a] = gi;
  }
  gstart[0] = 0;
  for (int q = 0; q < ng; ++q) gstart[q + 1] = gstart[q] + wid[q];
  int tot = gstart[ng];
  // row index R within group q: (component i, weight w) of J_a[:, R]
  auto sel = [&](int a, int R, int* i) -> double {
    int s = sl[a];
    if (!W.slot_aff[s] || R < 3) {
      *i = R;
      return 1.0;
    }
    *i = (R - 3) / 3;
    return W.slot_rest[3 * s + (R - 3) % 3];
  };
  for (int idx = threadIdx.x; idx < tot * tot; idx += blockDim.x) {
    int r = idx / tot, c = idx - r * tot;
    int qr = 0, qc = 0;
    while (r >= gstart[qr + 1]) ++qr;
    while (c >= gstart[qc + 1]) ++qc;
    int R = r - gstart[qr], Cc = c - gstart[qc];
    double acc = 0.0;
    for (int a = 0; a < ns; ++a) {
      if (grp[a] != qr) continue;
      int ia;
      double wa = sel(a, R, &ia);
      for (int b = 0; b < ns; ++b) {
        if (grp[b] != qc) continue;
        int ib;
        double wb = sel(b, Cc, &ib);
        acc += wa * wb * hget(3 * a + ia, 3 * b + ib);
      }
    }
    H[(key[qr] + R) * n + key[qc] + Cc] += acc;
  }
  for (int r = threadIdx.x; r < tot; r += blockDim.x) {
    int qr = 0;
    while (r >= gstart[qr + 1]) ++qr;
    int R = r - gstart[qr];
    double acc = 0.0;
    for (int a = 0; a < ns; ++a) {
      if (grp[a] != qr) continue;
      int ia;
      double wa = sel(a, R, &ia);
      acc += wa * gs[3 * a + ia];
    }
    g[key[qr] + R] += acc;
  }
  __syncthreads();
}

constexpr int DENSE_THREADS = 256;

// Assemble the env's dense Hessian/gradient, Cholesky-solve H p = −g with the
// gradient fallback of ref solver.py:241, write p, ‖p‖∞, ‖g‖∞.
__global__ void __launch_bounds__(DENSE_THREADS) k_dense_solve(World W, EnvState S, Derivs D, Cands C,
                                                                Lags L, const double* __restrict__ x,
                                                                const double* __restrict__ xhat,
                                                                double* p_out, double* g_out) {
  extern __shared__ double sm[];
  __shared__ double red[DENSE_THREADS / 32];
  __shared__ int fail;
  int e = blockIdx.x;
  if (!S.newton_active[e]) return;
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
  // tets
  for (int t = W.env_tet[e]; t < W.env_tet[e + 1]; ++t) {
    int4 td = W.tet_dof[t];
    int dv[4] = {td.x - d0, td.y - d0, td.z - d0, td.w - d0};
    const double* hp = D.tet_h + PK * t;
    for (int i = tid; i < 144; i += blockDim.x) {
      int r = i / 12, c = i % 12;
      H[(dv[r / 3] + r % 3) * n + dv[c / 3] + c % 3] += pk_get(hp, r, c);
    }
    for (int i = tid; i < 12; i += blockDim.x) g[dv[i / 3] + i % 3] += D.tet_g[12 * t + i];
    __syncthreads();
  }
  // contact pairs
  for (int kind = 0; kind < 2; ++kind) {
    int nn = kind == 0 ? C.n_pt[e] : C.n_ee[e];
    long long off = kind == 0 ? C.pt_off[e] : C.ee_off[e];
    const unsigned char* act = kind == 0 ? D.pt_act : D.ee_act;
    const double* gg = kind == 0 ? D.pt_g : D.ee_g;
    const double* hh = kind == 0 ? D.pt_h : D.ee_h;
    for (int k = 0; k < nn; ++k) {
      long long q = off + k;
      if (!act[q]) continue;
      int2 pr = kind == 0 ? C.pt[q] : C.ee[q];
      int sl[4];
      if (kind == 0) {
        int3 tv = W.tri_v[pr.y];
        sl[0] = pr.x; sl[1] = tv.x; sl[2] = tv.y; sl[3] = tv.z;
      } else {
        int2 a = W.edge_v[pr.x], b = W.edge_v[pr.y];
        sl[0] = a.x; sl[1] = a.y; sl[2] = b.x; sl[3] = b.y;
      }
      const double* hp = hh + PK * q;
      add_stencil(W, d0, n, H, g, 4, sl, gg + 12 * q, [&](int i, int j) { return pk_get(hp, i, j); });
    }
  }
  // ground barrier (y only)
  for (int k = 0; k < C.n_gnd[e]; ++k) {
    int q = C.gnd_off[e] + k;
    double hy = D.gnd_hyy[q], gy = D.gnd_gy[q];
    if (hy == 0.0 && gy == 0.0) continue;
    int sl[1] = {C.gnd[q]};
    double gs[3] = {0.0, gy, 0.0};
    add_stencil(W, d0, n, H, g, 1, sl, gs, [&](int i, int j) { return (i == 1 && j == 1) ? hy : 0.0; });
  }
  // friction
  for (int k = 0; k < L.n[e]; ++k) {
    long long q = L.off[e] + k;
    int4 s4 = L.slots[q];
    int sl[4] = {s4.x, s4.y, s4.z, s4.w};
    const double* hp = D.fr_h + PK * q;
    add_stencil(W, d0, n, H, g, 4, sl, D.fr_g + 12 * q, [&](int i, int j) { return pk_get(hp, i, j); });
  }
  for (int k = 0; k < L.g_n[e]; ++k) {
    int q = W.env_slot[e] + k;
    int sl[1] = {L.g_slot[q]};
    const double* hp = D.frg_h + 9 * q;
    add_stencil(W, d0, n, H, g, 1, sl, D.frg_g + 3 * q, [&](int i, int j) { return hp[3 * i + j]; });
  }
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
  // Cholesky H = L Lᵀ (lower, in place)
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      double akk = H[k * n + k];
      if (!(akk > 0.0)) fail = 1;
      H[k * n + k] = sqrt(fmax(akk, 1e-300));
    }
    __syncthreads();
    double lkk = H[k * n + k];
    for (int i = k + 1 + tid; i < n; i += blockDim.x) H[i * n + k] /= lkk;
    __syncthreads();
    int m = n - k - 1;
    for (int idx = tid; idx < m * m; idx += blockDim.x) {
      int i = k + 1 + idx / m, j = k + 1 + idx % m;
      if (j <= i) H[i * n + j] -= H[i * n + k] * H[j * n + k];
    }
    __syncthreads();
  }
  // forward: L z = -g
  for (int k = 0; k < n; ++k) {
    if (tid == 0) y[k] /= H[k * n + k];
    __syncthreads();
    for (int i = k + 1 + tid; i < n; i += blockDim.x) y[i] -= H[i * n + k] * y[k];
    __syncthreads();
  }
  // backward: Lᵀ p = z
  for (int k = n - 1; k >= 0; --k) {
    if (tid == 0) y[k] /= H[k * n + k];
    __syncthreads();
    for (int i = tid; i < k; i += blockDim.x) y[i] -= H[k * n + i] * y[k];
    __syncthreads();
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
}

// ---------------------------------------------------------------------------
// bookkeeping kernels (one thread per env)
// ---------------------------------------------------------------------------
__global__ void k_newton_begin(int n_env, EnvState S, const int* flag) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_env) return;
  int on = flag[e] ? 1 : 0;
  S.newton_active[e] = on;
  if (on) {
    S.small_run[e] = 0;
    S.prev_pnorm[e] = INFINITY;
  }
}

// two-consecutive-small-steps rule of ref solver.py:326-332
__global__ void k_newton_check(int n_env, EnvState S, double h, double tol) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_env || !S.newton_active[e]) {
    if (e < n_env) S.ls_active[e] = 0;
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

__global__ void k_ls_begin(int n_env, EnvState S, int* ls_count) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_env || !S.ls_active[e]) return;
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

// Armijo with c = 0 (ref solver.py:257); accepted envs copy xt -> x
__global__ void k_ls_check(World W, EnvState S, int* ls_count, int max_halvings, int* accepted) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= W.n_env) return;
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

__global__ void k_copy_env(World W, const double* src, double* dst, const int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W.n_dof) return;
  if (flag[W.dof_env[i]]) dst[i] = src[i];
}

// multiplier update after each inner solve (ref constraints.py:215, solver.py:414-434)
__global__ void k_al_update(World W, EnvState S, int outer) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= W.n_env || !S.al_active[e]) return;
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

__global__ void k_cons_reset(World W, const double* targets) {
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
__global__ void k_predictor(World W, double h) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < W.n_dof) W.xhat[i] = W.x[i] + h * W.v[i];
}
__global__ void k_predictor_forces(World W, double h) {
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

__global__ void k_finalize(World W, double h, const int* ok) {
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
__global__ void k_kappa_adapt(World W, EnvState S, const int* ok) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= W.n_env || !ok[e]) return;
  double md = isinf(S.min_s[e]) ? INFINITY : sqrt(S.min_s[e]);
  S.min_s[e] = md;  // now a distance
  double k = W.env_kappa[e], k0 = W.env_kappa0[e], dhat = W.env_dhat[e];
  if (md < 1e-4 * dhat && k < 1e8 * k0) W.env_kappa[e] = fmin(2.0 * k, 1e8 * k0);
}

__global__ void k_fill(int n, double* a, double v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
__global__ void k_fill_flag(int n, double* a, double v, const int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) a[i] = v;
}
__global__ void k_fill_int(int n, int* a, int v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
__global__ void k_count(int n, const int* flag, int* out) {
  __shared__ int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (flag[i]) atomicAdd(&s, 1);
  __syncthreads();
  if (threadIdx.x == 0) *out = s;
}
__global__ void k_sweep_box(int n, const double* xw, const double* dxw, double* lo, double* hi) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  double a = xw[i], b = __dadd_rn(xw[i], dxw[i]);
  lo[i] = fmin(a, b);
  hi[i] = fmax(a, b);
}

}  // namespace ipc
