// Sparse Newton system for large environments: deterministic BSR assembly by
// sort + segmented reduction, and block-Jacobi preconditioned CG.
//
// Nodes are 3-DoF groups: node = dof / 3 (a soft vertex, or one of the four
// (p, a1, a2, a3) triples of an affine body). Every element (soft-vertex
// inertia, affine body, tet, active contact pair, ground pair, friction
// stencil) emits 3x3 node blocks keyed (row << 32 | col) and gradient
// 3-vectors keyed (row << 32 | GRAD_COL). A stable radix sort groups equal
// keys in emission order, so the segmented sums — and the whole solve — are
// bit-reproducible (ref solver.py:223 _combine sums duplicates likewise).
#pragma once
#include "solve.cuh"

namespace ipc {

constexpr unsigned GRAD_COL = 0xFFFFFFFFu;

// lifted Jacobian row selector of slot `s` for node `k` of its group:
// row component i(r) and weight w(r) of J[:, 3k + r]
__device__ __forceinline__ double jsel(const World& W, int s, int k, int r, int* i) {
  if (!W.slot_aff[s] || k == 0) {
    *i = r;
    return 1.0;
  }
  *i = k - 1;
  return W.slot_rest[3 * s + r];
}
__device__ __forceinline__ int slot_nodes(const World& W, int s) { return W.slot_aff[s] ? 4 : 1; }
__device__ __forceinline__ int slot_node0(const World& W, int s) { return W.slot_dof[s] / 3; }

// element index space, in emission order
struct ElemSpace {
  long long n_vert, n_aff, n_tet, n_pt, n_ee, n_gnd, n_fr, n_frg;
  __device__ __forceinline__ long long total() const {
    return n_vert + n_aff + n_tet + n_pt + n_ee + n_gnd + n_fr + n_frg;
  }
};

// locate element q's type and local index
__device__ __forceinline__ int elem_type(const ElemSpace& S, long long q, long long* loc) {
  long long b[8] = {S.n_vert, S.n_aff, S.n_tet, S.n_pt, S.n_ee, S.n_gnd, S.n_fr, S.n_frg};
  for (int t = 0; t < 8; ++t) {
    if (q < b[t]) {
      *loc = q;
      return t;
    }
    q -= b[t];
  }
  *loc = 0;
  return -1;
}

__device__ __forceinline__ int find_env_ll(const long long* __restrict__ pre, int n_env, long long g) {
  int lo = 0, hi = n_env;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pre[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

struct AsmIn {  // everything an element needs
  World W;
  EnvState S;
  Derivs D;
  Cands C;
  Lags L;
  const double *x, *xhat;
  ElemSpace sp;
};

// Visit element q: returns its stencil (slots) or fixed-DoF description and
// calls emit(row_node, col_node_or_GRAD, v[9]) for each block / gradient.
// Modes: counting (emit counts) or writing.
template <typename Emit>
static __device__ void visit_element(const AsmIn& A, long long q, Emit emit) {
  const World& W = A.W;
  long long l;
  int t = elem_type(A.sp, q, &l);
  double v[9];
  if (t == 0) {  // soft vertex inertia
    int vi = (int)l;
    if (!A.S.newton_active[W.vert_env[vi]]) return;
    int d = W.vert_dof[vi];
    double m = W.vert_mass[vi];
    for (int i = 0; i < 9; ++i) v[i] = 0.0;
    v[0] = v[4] = v[8] = m;
    emit(d / 3, d / 3, v);
    v[0] = m * (A.x[d] - A.xhat[d]);
    v[1] = m * (A.x[d + 1] - A.xhat[d + 1]);
    v[2] = m * (A.x[d + 2] - A.xhat[d + 2]);
    emit(d / 3, GRAD_COL, v);
    return;
  }
  if (t == 1) {  // affine body 12x12 (inertia + h² ortho + kinematic)
    int b = (int)l;
    if (!A.S.newton_active[W.aff_env[b]]) return;
    int n0 = W.aff_dof[b] / 3;
    const double* H = A.D.body_h + 144 * b;
    for (int bi = 0; bi < 4; ++bi)
      for (int bj = 0; bj < 4; ++bj) {
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) v[3 * r + c] = H[(3 * bi + r) * 12 + 3 * bj + c];
        emit(n0 + bi, n0 + bj, v);
      }
    for (int bi = 0; bi < 4; ++bi) {
      for (int r = 0; r < 3; ++r) v[r] = A.D.body_g[12 * b + 3 * bi + r];
      emit(n0 + bi, GRAD_COL, v);
    }
    return;
  }
  if (t == 2) {  // tet
    int tt = (int)l;
    if (!A.S.newton_active[W.tet_env[tt]]) return;
    int4 td = W.tet_dof[tt];
    int nd[4] = {td.x / 3, td.y / 3, td.z / 3, td.w / 3};
    const double* hp = A.D.tet_h + PK * tt;
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) v[3 * r + c] = pk_get(hp, 3 * a + r, 3 * b + c);
        emit(nd[a], nd[b], v);
      }
    for (int a = 0; a < 4; ++a) {
      for (int r = 0; r < 3; ++r) v[r] = A.D.tet_g[12 * tt + 3 * a + r];
      emit(nd[a], GRAD_COL, v);
    }
    return;
  }
  // slot stencils
  int ns = 0, sl[4];
  const double* gs = nullptr;
  const double* hp = nullptr;
  double gbuf[3], hbuf[9];
  int hmode = 0;  // 0 packed 12x12, 1 dense 3x3
  if (t == 3 || t == 4) {
    int kind = t - 3;
    const long long* off = kind == 0 ? A.C.pt_off : A.C.ee_off;
    int e = find_env_ll(off, W.n_env, l);
    if (!A.S.newton_active[e]) return;
    int n = kind == 0 ? A.C.n_pt[e] : A.C.n_ee[e];
    if (l - off[e] >= n) return;
    const unsigned char* act = kind == 0 ? A.D.pt_act : A.D.ee_act;
    if (!act[l]) return;
    pair_slots(W, kind, kind == 0 ? A.C.pt[l] : A.C.ee[l], sl);
    ns = 4;
    gs = (kind == 0 ? A.D.pt_g : A.D.ee_g) + 12 * l;
    hp = (kind == 0 ? A.D.pt_h : A.D.ee_h) + PK * l;
  } else if (t == 5) {  // ground candidate (slot-indexed capacity)
    int e = W.slot_env[(int)l];
    if (!A.S.newton_active[e]) return;
    int k = (int)l - A.C.gnd_off[e];
    if (k >= A.C.n_gnd[e]) return;
    double gy = A.D.gnd_gy[l], hy = A.D.gnd_hyy[l];
    if (gy == 0.0 && hy == 0.0) return;
    sl[0] = A.C.gnd[l];
    ns = 1;
    gbuf[0] = 0.0; gbuf[1] = gy; gbuf[2] = 0.0;
    for (int i = 0; i < 9; ++i) hbuf[i] = 0.0;
    hbuf[4] = hy;
    gs = gbuf;
    hmode = 1;
  } else if (t == 6) {  // friction stencil
    int e = find_env_ll(A.L.off, W.n_env, l);
    if (!A.S.newton_active[e]) return;
    if (l - A.L.off[e] >= A.L.n[e]) return;
    int4 s4 = A.L.slots[l];
    sl[0] = s4.x; sl[1] = s4.y; sl[2] = s4.z; sl[3] = s4.w;
    ns = 4;
    gs = A.D.fr_g + 12 * l;
    hp = A.D.fr_h + PK * l;
  } else if (t == 7) {  // ground friction (slot-indexed)
    int e = W.slot_env[(int)l];
    if (!A.S.newton_active[e]) return;
    int k = (int)l - W.env_slot[e];
    if (k >= A.L.g_n[e]) return;
    sl[0] = A.L.g_slot[l];
    ns = 1;
    gs = A.D.frg_g + 3 * l;
    for (int i = 0; i < 9; ++i) hbuf[i] = A.D.frg_h[9 * l + i];
    hmode = 1;
  } else {
    return;
  }
  for (int a = 0; a < ns; ++a)
    for (int ka = 0; ka < slot_nodes(W, sl[a]); ++ka) {
      for (int b = 0; b < ns; ++b)
        for (int kb = 0; kb < slot_nodes(W, sl[b]); ++kb) {
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
              int ia, ib;
              double wa = jsel(W, sl[a], ka, r, &ia), wb = jsel(W, sl[b], kb, c, &ib);
              double h = hmode ? hbuf[3 * ia + ib] : pk_get(hp, 3 * a + ia, 3 * b + ib);
              v[3 * r + c] = wa * wb * h;
            }
          emit(slot_node0(W, sl[a]) + ka, slot_node0(W, sl[b]) + kb, v);
        }
      for (int r = 0; r < 3; ++r) {
        int ia;
        double wa = jsel(W, sl[a], ka, r, &ia);
        v[r] = wa * gs[3 * a + ia];
      }
      emit(slot_node0(W, sl[a]) + ka, GRAD_COL, v);
    }
}

IPC_GLOBAL void k_asm_count(AsmIn A, int* counts) {
  ipc_pdl_wait();
  long long n = A.sp.total();
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    int c = 0;
    visit_element(A, q, [&](int, unsigned, const double*) { ++c; });
    counts[q] = c;
  }
}

IPC_GLOBAL void k_asm_emit(AsmIn A, const long long* offs, unsigned long long* keys, double* vals, int* idx) {
  ipc_pdl_wait();
  long long n = A.sp.total();
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    long long o = offs[q];
    visit_element(A, q, [&](int row, unsigned col, const double* v) {
      keys[o] = ((unsigned long long)(unsigned)row << 32) | col;
      for (int i = 0; i < 9; ++i) vals[9 * o + i] = v[i];
      idx[o] = (int)o;
      ++o;
    });
  }
}

// head flags of sorted keys (1 at the first item of every run)
IPC_GLOBAL void k_asm_heads(long long n, const unsigned long long* keys, int* heads) {
  ipc_pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    heads[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// run starts: seg_start[u] = first sorted position of unique key u
IPC_GLOBAL void k_asm_starts(long long n, const int* heads, const long long* uidx, long long* seg_start) {
  ipc_pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (heads[i]) seg_start[uidx[i]] = i;
}

// sum each run in sorted (= emission) order; gradient runs go to g, blocks
// to the BSR value array; also count blocks per row
IPC_GLOBAL void k_asm_reduce(long long n_items, long long n_unique, const unsigned long long* keys,
                             const long long* seg_start, const int* perm, const double* vals, double* g,
                             unsigned* bcol, double* bval, int* row_cnt, int* bpos) {
  ipc_pdl_wait();
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n_unique; u += (long long)gridDim.x * blockDim.x) {
    long long a = seg_start[u], b = (u + 1 < n_unique) ? seg_start[u + 1] : n_items;
    unsigned long long key = keys[a];
    unsigned row = (unsigned)(key >> 32), col = (unsigned)(key & 0xFFFFFFFFu);
    double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (long long i = a; i < b; ++i) {
      const double* v = vals + 9 * (long long)perm[i];
      for (int k = 0; k < 9; ++k) s[k] += v[k];
    }
    if (col == GRAD_COL) {
      g[3 * row] = s[0];
      g[3 * row + 1] = s[1];
      g[3 * row + 2] = s[2];
      bpos[u] = -1;
    } else {
      for (int k = 0; k < 9; ++k) bval[9 * u + k] = s[k];
      bcol[u] = col;
      atomicAdd(row_cnt + row, 1);  // counts only (order-free)
      bpos[u] = 1;
    }
  }
}

// BSR (row-sorted by construction of the keys): row_ptr over the block
// entries; block entry j of row r is unique index row_first[r] + j (gradient
// entries sit at the end of each row's run: col GRAD_COL sorts last)
IPC_GLOBAL void k_bsr_rowfirst(long long n_unique, const unsigned long long* keys, const long long* seg_start,
                               int* row_first) {
  ipc_pdl_wait();
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n_unique; u += (long long)gridDim.x * blockDim.x) {
    unsigned row = (unsigned)(keys[seg_start[u]] >> 32);
    if (u == 0 || (unsigned)(keys[seg_start[u - 1]] >> 32) != row) row_first[row] = (int)u;
  }
}

// ---------------------------------------------------------------------------
// block-Jacobi PCG over all active envs. Rows = nodes. Reductions are
// deterministic: per-chunk partial sums (chunks never straddle envs), then
// per-env sums over the env's chunks in order.
// ---------------------------------------------------------------------------
struct Pcg {
  int n_node, n_chunk;
  const int *chunk_env, *chunk_n0, *chunk_n1;  // chunk -> env, node range
  const int *env_chunk;                         // [n_env+1]
  const int* node_env;
  const int *row_first, *row_cnt;  // BSR rows (row_cnt = #block entries)
  const unsigned* bcol;
  const double* bval;
  double *x, *r, *z, *p, *Ap, *Minv;  // 3 per node; Minv 9 per node
  double *part, *env_rz, *env_rz_new, *env_pap, *env_bb, *env_rr;
  int* env_live;  // per env: still iterating
  const int* env_on;  // newton_active
  // affine bodies are preconditioned by the inverse of their whole 12x12
  // diagonal block (the 4 nodes of a body never straddle a chunk):
  // node_aff[node] = global affine body index or -1, aff_node0[b] = its first node
  const int *node_aff, *aff_node0;
  double* Minv12;  // 144 per affine body
  int aff_blocks;  // 0: plain 3x3 node blocks everywhere
};

// z (3 values) of node nd = M⁻¹ r: the node's 3x3 block inverse, or its 3
// rows of the owning affine body's 12x12 block inverse
__device__ __forceinline__ void pcg_precond_node(const Pcg& P, int nd, double* z) {
  int b = P.aff_blocks ? P.node_aff[nd] : -1;
  if (b < 0) {
    const double* M = P.Minv + 9 * (long long)nd;
    const double* r = P.r + 3 * (long long)nd;
    for (int k = 0; k < 3; ++k) z[k] = M[3 * k] * r[0] + M[3 * k + 1] * r[1] + M[3 * k + 2] * r[2];
    return;
  }
  int n0 = P.aff_node0[b];
  const double* M = P.Minv12 + 144 * (long long)b + 36 * (nd - n0);
  const double* r = P.r + 3 * (long long)n0;
  for (int k = 0; k < 3; ++k) {
    double s = 0.0;
    for (int j = 0; j < 12; ++j) s += M[12 * k + j] * r[j];
    z[k] = s;
  }
}

// in-place inverse of a 12x12 matrix (Gauss-Jordan, partial pivoting); false
// when singular
static __device__ bool inv12(double* A) {
  int piv[12];
  for (int c = 0; c < 12; ++c) {
    int pr = c;
    double best = fabs(A[12 * c + c]);
    for (int r = c + 1; r < 12; ++r)
      if (fabs(A[12 * r + c]) > best) { best = fabs(A[12 * r + c]); pr = r; }
    if (!(best > 0.0)) return false;
    piv[c] = pr;
    if (pr != c)
      for (int j = 0; j < 12; ++j) { double t = A[12 * c + j]; A[12 * c + j] = A[12 * pr + j]; A[12 * pr + j] = t; }
    double d = 1.0 / A[12 * c + c];
    A[12 * c + c] = 1.0;
    for (int j = 0; j < 12; ++j) A[12 * c + j] *= d;
    for (int r = 0; r < 12; ++r) {
      if (r == c) continue;
      double f = A[12 * r + c];
      A[12 * r + c] = 0.0;
      for (int j = 0; j < 12; ++j) A[12 * r + j] -= f * A[12 * c + j];
    }
  }
  for (int c = 11; c >= 0; --c)
    if (piv[c] != c)
      for (int r = 0; r < 12; ++r) { double t = A[12 * r + c]; A[12 * r + c] = A[12 * r + piv[c]]; A[12 * r + piv[c]] = t; }
  return true;
}

__device__ __forceinline__ bool row_live(const Pcg& P, int node) { return P.env_live[P.node_env[node]]; }

// M⁻¹ = inverse of each node's diagonal 3x3 block, and of each affine body's
// 12x12 diagonal block (aff_blocks); x = 0, r = b = -g, z = p = M⁻¹ r
IPC_GLOBAL void k_pcg_setup(Pcg P, const double* g) {
  ipc_pdl_wait();
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < P.n_node; nd += gridDim.x * blockDim.x) {
    int e = P.node_env[nd];
    if (!P.env_on[e]) continue;
    const double* D = nullptr;
    int f = P.row_first[nd];
    for (int j = 0; j < P.row_cnt[nd]; ++j)
      if ((int)P.bcol[f + j] == nd) D = P.bval + 9 * (long long)(f + j);
    M3 m;
    for (int i = 0; i < 9; ++i) m.m[i] = D ? D[i] : (i % 4 == 0 ? 1.0 : 0.0);
    double det = m3_det(m);
    M3 inv = m3_T(m3_inv_T(m, det));
    for (int i = 0; i < 9; ++i) P.Minv[9 * nd + i] = inv.m[i];
    for (int c = 0; c < 3; ++c) {
      P.x[3 * nd + c] = 0.0;
      P.r[3 * nd + c] = -g[3 * nd + c];
    }
    int b = P.aff_blocks ? P.node_aff[nd] : -1;
    if (b >= 0 && P.aff_node0[b] == nd) {  // the body's first node gathers its 12x12 block
      double A[144];
      for (int i = 0; i < 144; ++i) A[i] = 0.0;
      for (int q = 0; q < 4; ++q) {
        int fq = P.row_first[nd + q];
        for (int j = 0; j < P.row_cnt[nd + q]; ++j) {
          int cq = (int)P.bcol[fq + j] - nd;
          if (cq < 0 || cq >= 4) continue;
          const double* B = P.bval + 9 * (long long)(fq + j);
          for (int u = 0; u < 3; ++u)
            for (int v = 0; v < 3; ++v) A[12 * (3 * q + u) + 3 * cq + v] = B[3 * u + v];
        }
      }
      bool ok = inv12(A);
      double* M = P.Minv12 + 144 * (long long)b;
      for (int i = 0; i < 144; ++i) M[i] = ok ? A[i] : 0.0;
      if (!ok)  // singular block: fall back to the 3x3 node blocks on the diagonal
        for (int q = 0; q < 4; ++q)
          for (int u = 0; u < 3; ++u)
            for (int v = 0; v < 3; ++v) M[12 * (3 * q + u) + 3 * q + v] = P.Minv[9 * (nd + q) + 3 * u + v];
    }
  }
}

// z = p = M⁻¹ r after k_pcg_setup (a separate pass: affine rows need the
// whole body's r and Minv12)
IPC_GLOBAL void k_pcg_setup_z(Pcg P) {
  ipc_pdl_wait();
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < P.n_node; nd += gridDim.x * blockDim.x) {
    if (!P.env_on[P.node_env[nd]]) continue;
    double z[3];
    pcg_precond_node(P, nd, z);
    for (int c = 0; c < 3; ++c) {
      P.z[3 * nd + c] = z[c];
      P.p[3 * nd + c] = z[c];
    }
  }
}

// chunk partial dots: which 0 -> (r·z, b·b) ; 1 -> p·Ap ; 2 -> (r·z, r·r)
IPC_GLOBAL void k_pcg_partial(Pcg P, int which) {
  ipc_pdl_wait();
  __shared__ double sh[2][8];
  int c = blockIdx.x;
  if (c >= P.n_chunk) return;
  int e = P.chunk_env[c];
  if (!P.env_on[e] || (which != 0 && !P.env_live[e])) return;
  double a = 0.0, b = 0.0;
  for (int nd = P.chunk_n0[c] + threadIdx.x; nd < P.chunk_n1[c]; nd += blockDim.x)
    for (int k = 0; k < 3; ++k) {
      int i = 3 * nd + k;
      if (which == 1) a += P.p[i] * P.Ap[i];
      else {
        a += P.r[i] * P.z[i];
        b += P.r[i] * P.r[i];
      }
    }
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    sh[0][w] = a;
    sh[1][w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      sa += sh[0][k];
      sb += sh[1][k];
    }
    P.part[2 * c] = sa;
    P.part[2 * c + 1] = sb;
  }
}

// per-env scalar step. stage 0: init rz, bb; 1: pAp; 2: new rz / rr, β, convergence
IPC_GLOBAL void k_pcg_env(Pcg P, int n_env, int stage, double rtol2) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_env || !P.env_on[e]) return;
  if (stage != 0 && !P.env_live[e]) return;
  double a = 0.0, b = 0.0;
  for (int c = P.env_chunk[e]; c < P.env_chunk[e + 1]; ++c) {
    a += P.part[2 * c];
    b += P.part[2 * c + 1];
  }
  if (stage == 0) {
    P.env_rz[e] = a;
    P.env_bb[e] = b;
    P.env_live[e] = b > 0.0 ? 1 : 0;
  } else if (stage == 1) {
    P.env_pap[e] = a;
  } else {
    P.env_rz_new[e] = a;
    P.env_rr[e] = b;
    if (!(b > rtol2 * P.env_bb[e])) P.env_live[e] = 0;
  }
}

// direction, fallback and norms per env (ref solver.py:241): p = x unless the
// solve produced non-finite values or an ascent direction, then p = -g
IPC_GLOBAL void k_pcg_finish(World W, EnvState S, Pcg P, const double* g, double* p_out, double* g_out) {
  ipc_pdl_wait();
  __shared__ double sh[3][8];
  int e = blockIdx.x;
  if (!S.newton_active[e]) return;
  int d0 = W.env_dof[e], d1 = W.env_dof[e + 1];
  double pg = 0.0, gm = 0.0;
  int bad = 0;
  for (int i = d0 + threadIdx.x; i < d1; i += blockDim.x) {
    pg += P.x[i] * g[i];
    gm = fmax(gm, fabs(g[i]));
    if (!isfinite(P.x[i])) bad = 1;
  }
  bad = __syncthreads_or(bad);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    pg += __shfl_down_sync(0xffffffffu, pg, o);
    gm = fmax(gm, __shfl_down_sync(0xffffffffu, gm, o));
  }
  if (lane == 0) { sh[0][w] = pg; sh[1][w] = gm; }
  __syncthreads();
  __shared__ int use_grad;
  if (threadIdx.x == 0) {
    double a = 0.0, m = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { a += sh[0][k]; m = fmax(m, sh[1][k]); }
    use_grad = bad || a > 0.0;
    S.gnorm[e] = m;
  }
  __syncthreads();
  double pm = 0.0;
  for (int i = d0 + threadIdx.x; i < d1; i += blockDim.x) {
    double pi = use_grad ? -g[i] : P.x[i];
    p_out[i] = pi;
    g_out[i] = g[i];
    pm = fmax(pm, fabs(pi));
  }
  for (int o = 16; o > 0; o >>= 1) pm = fmax(pm, __shfl_down_sync(0xffffffffu, pm, o));
  if (lane == 0) sh[2][w] = pm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmax(m, sh[2][k]);
    S.pnorm[e] = m;
  }
}

}  // namespace ipc

#include <cooperative_groups.h>

namespace ipc {
namespace cg = cooperative_groups;

// The whole block-Jacobi PCG loop as one cooperative persistent kernel:
// phases separated by grid-wide barriers, per-env scalars updated by one
// thread per env, chunk partial sums reduced per block in a fixed order
// (same arithmetic as the per-phase kernels above, no host round trips).
__device__ __forceinline__ void coop_partial(const Pcg& P, int which, double* sh) {
  for (int c = blockIdx.x; c < P.n_chunk; c += gridDim.x) {
    int e = P.chunk_env[c];
    bool on = P.env_on[e] && P.env_live[e];
    double a = 0.0, b = 0.0;
    if (on)
      for (int nd = P.chunk_n0[c] + threadIdx.x; nd < P.chunk_n1[c]; nd += blockDim.x)
        for (int k = 0; k < 3; ++k) {
          int i = 3 * nd + k;
          if (which == 1) a += P.p[i] * P.Ap[i];
          else {
            a += P.r[i] * P.z[i];
            b += P.r[i] * P.r[i];
          }
        }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b += __shfl_down_sync(0xffffffffu, b, o);
    }
    if (lane == 0) {
      sh[w] = a;
      sh[32 + w] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0 && on) {
      double sa = 0.0, sb = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
        sa += sh[k];
        sb += sh[32 + k];
      }
      P.part[2 * c] = sa;
      P.part[2 * c + 1] = sb;
    }
    __syncthreads();
  }
}

// chunk-aligned block pass: block owns chunk c (all of its nodes), so the
// node update and the chunk's partial dot products need no extra barrier
__device__ __forceinline__ void chunk_reduce(double a, double b, double* sh, double* out2) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    sh[w] = a;
    sh[32 + w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      sa += sh[k];
      sb += sh[32 + k];
    }
    out2[0] = sa;
    out2[1] = sb;
  }
  __syncthreads();
}

__device__ __forceinline__ void env_sums(const Pcg& P, int e, const double* part, double* a, double* b) {
  double sa = 0.0, sb = 0.0;
  for (int c = P.env_chunk[e]; c < P.env_chunk[e + 1]; ++c) {
    sa += part[2 * c];
    sb += part[2 * c + 1];
  }
  *a = sa;
  *b = sb;
}

// (Σa, Σb) over env e's chunk partials, computed by warp 0 with a fixed
// lane/shuffle tree (bitwise identical in every block) and broadcast via smem
__device__ __forceinline__ void block_env_sums(const Pcg& P, int e, const double* part, double* out2) {
  __syncthreads();
  if (threadIdx.x < 32) {
    double a = 0.0, b = 0.0;
    for (int c = P.env_chunk[e] + threadIdx.x; c < P.env_chunk[e + 1]; c += 32) {
      a += part[2 * c];
      b += part[2 * c + 1];
    }
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (threadIdx.x == 0) {
      out2[0] = a;
      out2[1] = b;
    }
  }
  __syncthreads();
}

// Persistent PCG over all envs, three grid barriers per iteration. Per-chunk
// partials: part1 = p·Ap; (r·z, r·r) double-buffered in bufs[0] (= P.part,
// written by the setup pass) and bufs[1]; every block derives an env's
// liveness, α and β from the same partials, so no per-env scalar pass is
// needed. cnt[0..1]: live-env counters (alternating), cnt[2]: cumulative
// iteration count (stats).
IPC_GLOBAL void k_pcg_coop(Pcg P, int n_env, double rtol2, int max_iters, int* cnt, double* part1, double* part2) {
  ipc_pdl_wait();
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[64];
  __shared__ double es[6];  // env sums: cur (rz, rr), part1 (pAp, -), nxt (rz, rr)
  (void)n_env;
  for (int it = 0; it < max_iters; ++it) {
    const double* cur = (it & 1) ? part2 : P.part;
    double* nxt = (it & 1) ? P.part : part2;
    // phase A: Ap = H p on the block's chunks (one warp per row, lanes over
    // the row's 3x3 blocks) + chunk partial p·Ap
    for (int c = blockIdx.x; c < P.n_chunk; c += gridDim.x) {
      int e = P.chunk_env[c];
      if (!P.env_on[e] || !P.env_live[e]) continue;
      block_env_sums(P, e, cur, es);
      if (!(es[1] > rtol2 * P.env_bb[e])) continue;
      int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      double a = 0.0;
      for (int nd = P.chunk_n0[c] + wid; nd < P.chunk_n1[c]; nd += nw) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        int f = P.row_first[nd], rc = P.row_cnt[nd];
        for (int j = lane; j < rc; j += 32) {
          const double* B = P.bval + 9 * (long long)(f + j);
          const double* pv = P.p + 3 * (long long)P.bcol[f + j];
          double p0 = pv[0], p1 = pv[1], p2 = pv[2];
          s0 += B[0] * p0 + B[1] * p1 + B[2] * p2;
          s1 += B[3] * p0 + B[4] * p1 + B[5] * p2;
          s2 += B[6] * p0 + B[7] * p1 + B[8] * p2;
        }
        for (int o = 16; o > 0; o >>= 1) {
          s0 += __shfl_xor_sync(0xffffffffu, s0, o);
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (lane == 0) {
          P.Ap[3 * nd] = s0;
          P.Ap[3 * nd + 1] = s1;
          P.Ap[3 * nd + 2] = s2;
          a += P.p[3 * nd] * s0 + P.p[3 * nd + 1] * s1 + P.p[3 * nd + 2] * s2;
        }
      }
      chunk_reduce(a, 0.0, sh, part1 + 2 * c);
    }
    grid.sync();
    // phase B: α = rz / pAp; x, r, z update + next (r·z, r·r) partials
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(it + 1) & 1] = 0;
    for (int c = blockIdx.x; c < P.n_chunk; c += gridDim.x) {
      int e = P.chunk_env[c];
      bool live = P.env_on[e] && P.env_live[e];
      if (live) {
        block_env_sums(P, e, cur, es);
        live = es[1] > rtol2 * P.env_bb[e];
      }
      if (!live) {
        if (threadIdx.x == 0) {  // keep both buffers equal for finished envs
          nxt[2 * c] = cur[2 * c];
          nxt[2 * c + 1] = cur[2 * c + 1];
        }
        continue;
      }
      block_env_sums(P, e, part1, es + 2);
      double al = es[0] / es[2];
      double a = 0.0, b = 0.0;
      for (int nd = P.chunk_n0[c] + threadIdx.x; nd < P.chunk_n1[c]; nd += blockDim.x) {
        for (int k = 0; k < 3; ++k) {
          int i = 3 * nd + k;
          P.x[i] += al * P.p[i];
          P.r[i] -= al * P.Ap[i];
        }
      }
      if (P.aff_blocks) __syncthreads();  // affine rows read the whole body's r
      for (int nd = P.chunk_n0[c] + threadIdx.x; nd < P.chunk_n1[c]; nd += blockDim.x) {
        double z[3];
        pcg_precond_node(P, nd, z);
        for (int k = 0; k < 3; ++k) {
          P.z[3 * nd + k] = z[k];
          a += P.r[3 * nd + k] * z[k];
          b += P.r[3 * nd + k] * P.r[3 * nd + k];
        }
      }
      chunk_reduce(a, b, sh, nxt + 2 * c);
    }
    grid.sync();
    // phase C: convergence test and p = z + β p
    for (int c = blockIdx.x; c < P.n_chunk; c += gridDim.x) {
      int e = P.chunk_env[c];
      if (!P.env_on[e] || !P.env_live[e]) continue;
      block_env_sums(P, e, cur, es);
      if (!(es[1] > rtol2 * P.env_bb[e])) continue;
      block_env_sums(P, e, nxt, es + 4);
      if (!(es[5] > rtol2 * P.env_bb[e])) continue;  // converged this iteration
      double be = es[4] / es[0];
      for (int nd = P.chunk_n0[c] + threadIdx.x; nd < P.chunk_n1[c]; nd += blockDim.x)
        for (int k = 0; k < 3; ++k) P.p[3 * nd + k] = P.z[3 * nd + k] + be * P.p[3 * nd + k];
      if (c == P.env_chunk[e] && threadIdx.x == 0) atomicAdd(cnt + (it & 1), 1);
    }
    grid.sync();
    if (cnt[it & 1] == 0 || it + 1 == max_iters) {
      if (blockIdx.x == 0 && threadIdx.x == 0) cnt[2] += it + 1;
      break;
    }
  }
}

}  // namespace ipc
