// Host engine of libipc_b200.so: owns the device-resident world and drives
// the per-step kernel sequence (ref solver.py:360 step / :295 _newton_solve).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ipc_b200.h"
#include <cub/cub.cuh>

#include "sparse.cuh"
#include "fused.cuh"

using namespace ipc;

static thread_local std::string g_err;

static int set_err(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return -1;
}

// error sink for the other translation units of the library (repair.cu)
extern "C" int ipc__set_error(const char* msg) { return set_err("%s", msg); }

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw std::runtime_error(std::string(#call) + ": " + cudaGetErrorString(e_));  \
  } while (0)

#define GUARD(...)                                    \
  try {                                                \
    __VA_ARGS__;                                       \
    return 0;                                          \
  } catch (const std::exception& ex) {                 \
    return set_err("%s", ex.what());                   \
  }

static inline int nblk(long long n, int t) { return (int)std::max<long long>(1, (n + t - 1) / t); }

// ---------------------------------------------------------------------------
// launch accounting + optional per-kernel CUDA-event timing
// ---------------------------------------------------------------------------
enum Kid {
  K_BROAD_DCD = 0, K_BROAD_SWEEP, K_PAIRS_D, K_PAIRS_V, K_TET, K_BODY, K_GROUND, K_FRICTION, K_ENERGY,
  K_DENSE, K_CCD, K_LAGS, K_WORLD, K_SENSE, K_MISC, K_PCG, K_ASM, K_FUSED, NKID
};
struct OverflowRetry : std::exception {
  const char* what() const noexcept override { return "candidate capacity overflow"; }
};

struct Prof {
  bool on = false;
  bool capturing = false;
  unsigned mask = ~0u;
  long long launches = 0;
  struct Rec {
    int kid;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> pool;
  std::vector<Rec> pending;
  Rec cur{};
  std::vector<Rec> capture_list;  // event pairs baked into a graph being captured
  double ms[NKID] = {};
  long long cnt[NKID] = {};
  cudaEvent_t ev() {
    if (pool.empty()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void resolve() {
    for (auto& r : pending) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, r.a, r.b));
      ms[r.kid] += t;
      cnt[r.kid] += 1;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    pending.clear();
  }
  ~Prof() {
    for (auto& r : pending) { pool.push_back(r.a); pool.push_back(r.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};
static thread_local Prof* g_prof = nullptr;
static inline void prof_begin(int kid, cudaStream_t s) {
  Prof* p = g_prof;
  if (!p) return;
  p->launches++;
  if (p->on && ((p->mask >> kid) & 1u)) {
    p->cur.kid = kid;
    p->cur.a = p->ev();
    if (p->capturing) CK(cudaEventRecordWithFlags(p->cur.a, s, cudaEventRecordExternal));
    else CK(cudaEventRecord(p->cur.a, s));
  } else {
    p->cur.kid = -1;
  }
}
static inline void prof_end(int kid, cudaStream_t s) {
  Prof* p = g_prof;
  if (!p || p->cur.kid < 0) return;
  p->cur.b = p->ev();
  if (p->capturing) CK(cudaEventRecordWithFlags(p->cur.b, s, cudaEventRecordExternal));
  else CK(cudaEventRecord(p->cur.b, s));
  if (p->capturing) p->capture_list.push_back(p->cur);
  else p->pending.push_back(p->cur);
  p->cur.kid = -1;
}
// Kernel launches go through cudaLaunchKernelEx with programmatic stream
// serialization (IPC_PDL=0: plain launches): a kernel is scheduled while its
// predecessor on the stream drains and waits in ipc_pdl_wait() before its
// first memory access, so the ≈25 dependent launches of a Newton iteration
// overlap their launch latency with the previous kernel's tail.
static bool g_pdl = true;  // read at every world creation (IPC_PDL)
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#define IPC_LAUNCH(kid, stream, kern, grid, block, smem, ...)  \
  do {                                                         \
    prof_begin((kid), (stream));                               \
    CK(launch_pdl(kern, dim3(grid), dim3(block), (size_t)(smem), stream, __VA_ARGS__)); \
    prof_end((kid), (stream));                                 \
  } while (0)

namespace ipc {
__global__ void k_mark_unconverged(int n_env, EnvState S) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n_env && S.newton_active[e]) {
    S.converged[e] = 0;
    S.newton_active[e] = 0;
  }
}
__global__ void k_step_begin(int n_env, EnvState S) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_env) return;
  S.newton_iters[e] = 0; S.ccd_calls[e] = 0; S.al_outer[e] = 0; S.ls_failed[e] = 0;
  S.converged[e] = 1; S.err[e] = 0; S.min_s_before[e] = INFINITY; S.gnorm[e] = 0.0;
}
// intersection check of the incoming state: any candidate value is inf
__global__ void k_start_check(World W, EnvState S, Cands C, const double* ptv, const double* eev,
                              const double* gv, int* ok) {
  ipc_pdl_wait();
  int e = blockIdx.x;
  if (!ok[e]) {
    if (threadIdx.x == 0) S.err[e] = 0;
    return;
  }
  int bad = 0;
  for (int k = threadIdx.x; k < C.n_pt[e]; k += blockDim.x) bad |= isinf(ptv[C.pt_off[e] + k]);
  for (int k = threadIdx.x; k < C.n_ee[e]; k += blockDim.x) bad |= isinf(eev[C.ee_off[e] + k]);
  for (int k = threadIdx.x; k < C.n_gnd[e]; k += blockDim.x) bad |= isinf(gv[C.gnd_off[e] + k]);
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    ok[e] = !bad;
    S.err[e] = bad;
  }
}
__global__ void k_status(int n_env, const int* newton, const int* ls, const int* ov1, const int* ov2, int* out) {
  ipc_pdl_wait();
  __shared__ int a, b;
  if (threadIdx.x == 0) a = b = 0;
  __syncthreads();
  int ca = 0, cb = 0;
  for (int e = threadIdx.x; e < n_env; e += blockDim.x) {
    ca += newton[e] != 0;
    cb += ls[e] != 0;
  }
  atomicAdd(&a, ca);
  atomicAdd(&b, cb);
  __syncthreads();
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
    out[2] = *ov1 | *ov2;
  }
}
// Device-driven Newton loop control (the body of the loop graph's WHILE
// node, after the SWITCH that ran one Newton iteration (mode 0) or one
// line-search round of LS_M (mode 1) or, from the second round of an
// iteration, LS_M2 speculative trials (mode 2)). Mirrors the host loop of newton_solve: line
// search rounds while any env is still backtracking and fewer than
// max_halvings+1 trials were made, then the next iteration unless no env is
// active, the iteration cap is reached, the active count fits the per-env
// tail hand-off, or a candidate store overflowed (the host then replays).
// ctl: [0] iterations run, [1] line-search trials of this iteration,
// [2] line-search rounds (stats), [3] active envs at exit, [4] overflow,
// [5] mode of the body that just ran (set here for the next one; 0 at launch)
__global__ void k_loop_ctl(int n_env, const int* newton, const int* ls, const int* ov1, const int* ov2, int* ctl,
                           int max_iters, int max_halvings, int ls_m, int ls_m2, int tail,
                           cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_mode) {
  ipc_pdl_wait();
  __shared__ int a, b;
  if (threadIdx.x == 0) a = b = 0;
  __syncthreads();
  int ca = 0, cb = 0;
  for (int e = threadIdx.x; e < n_env; e += blockDim.x) {
    ca += newton[e] != 0;
    cb += ls[e] != 0;
  }
  atomicAdd(&a, ca);
  atomicAdd(&b, cb);
  __syncthreads();
  if (threadIdx.x != 0) return;
  int ov = *ov1 | *ov2;
  // the trials of the mode that just ran
  if (ctl[5] == 0) {
    ctl[0] += 1;
    ctl[1] = 1;
  } else {
    ctl[1] += ctl[5] == 1 ? ls_m : ls_m2;
  }
  ctl[2] += 1;
  ctl[3] = a;
  ctl[4] = ov;
  unsigned loop = 1, mode = 0;
  if (ov) {
    loop = 0;
  } else if (b && ctl[1] < max_halvings + 1) {
    mode = ctl[5] == 0 ? 1 : 2;  // first follow-up round: LS_M trials, then LS_M2
  } else if (a == 0 || ctl[0] >= max_iters || (tail > 0 && a <= tail)) {
    loop = 0;
  }
  ctl[5] = (int)mode;
  cudaGraphSetConditional(h_mode, mode);
  cudaGraphSetConditional(h_loop, loop);
}
// sweep boxes along p, one pass per slot: x_t = x + p on flagged envs (as
// k_axpy_env), xw(x_t) (as world_slot), dxw = xw(x_t) - xw(x) and the boxes
// over [xw, xw + dxw] (ref broadphase.py:206); x_t and xw(x_t) stay in
// registers (the batched path has no other reader of them)
__global__ void k_sweep_slots(World W, const double* __restrict__ x, const double* __restrict__ p,
                              const int* flag, const double* __restrict__ xw, double* dxw, double* lo,
                              double* hi) {
  ipc_pdl_wait();
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= W.n_slot) return;
  int d = W.slot_dof[s];
  bool on = flag == nullptr || flag[W.dof_env[d]];
  auto xt = [&](int j) { return on ? __dadd_rn(x[j], __dmul_rn(1.0, p[j])) : x[j]; };
  double t[3];
  if (!W.slot_aff[s]) {
    for (int i = 0; i < 3; ++i) t[i] = xt(d + i);
  } else {
    const double* r = W.slot_rest + 3 * s;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      int a = d + 3 + 3 * i;
      double m = __dadd_rn(__dadd_rn(__dmul_rn(xt(a), r[0]), __dmul_rn(xt(a + 1), r[1])), __dmul_rn(xt(a + 2), r[2]));
      t[i] = __dadd_rn(xt(d + i), m);
    }
  }
  for (int i = 0; i < 3; ++i) {
    int k = 3 * s + i;
    double w = xw[k], dd = __dsub_rn(t[i], w);
    dxw[k] = dd;
    double b = __dadd_rn(w, dd);
    lo[k] = fmin(w, b);
    hi[k] = fmax(w, b);
  }
}
__global__ void k_copy_int(int n, const int* a, int* b) {
  ipc_pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}
__global__ void k_and_not(int n, int* a, const int* b) {
  ipc_pdl_wait();  // a &= !b
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && b[i]) a[i] = 0;
}
// slot forces: -∂B/∂x_slot / h², each slot gathers its own contributions
// in candidate order (deterministic)
__global__ void k_slot_forces(World W, Cands C, const double* pt_g, const unsigned char* pt_act,
                              const double* ee_g, const unsigned char* ee_act, const double* gnd_gy,
                              double h, double* out) {
  ipc_pdl_wait();
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= W.n_slot) return;
  int e = W.slot_env[s];
  double f[3] = {0, 0, 0};
  for (int kind = 0; kind < 2; ++kind) {
    int n = kind == 0 ? C.n_pt[e] : C.n_ee[e];
    long long off = kind == 0 ? C.pt_off[e] : C.ee_off[e];
    const unsigned char* act = kind == 0 ? pt_act : ee_act;
    const double* g = kind == 0 ? pt_g : ee_g;
    for (int k = 0; k < n; ++k) {
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
      for (int a = 0; a < 4; ++a)
        if (sl[a] == s)
          for (int c = 0; c < 3; ++c) f[c] += g[12 * q + 3 * a + c];
    }
  }
  for (int k = 0; k < C.n_gnd[e]; ++k)
    if (C.gnd[C.gnd_off[e] + k] == s) f[1] += gnd_gy[C.gnd_off[e] + k];
  double ih = 1.0 / (h * h);
  for (int c = 0; c < 3; ++c) out[3 * s + c] = -f[c] * ih;
}
__global__ void k_group_forces(World W, const double* slot_f, const unsigned long long* groups, int ng,
                               double* out) {
  ipc_pdl_wait();
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= W.n_env * ng) return;
  int e = q / ng;
  unsigned long long m = groups[q];
  int cb0 = W.env_cbody[e];
  double f[3] = {0, 0, 0};
  for (int s = W.env_slot[e]; s < W.env_slot[e + 1]; ++s)
    if ((m >> (W.slot_cbody[s] - cb0)) & 1ull)
      for (int c = 0; c < 3; ++c) f[c] += slot_f[3 * s + c];
  for (int c = 0; c < 3; ++c) out[3 * q + c] = f[c];
}
__global__ void k_group_distance(World W, Cands C, const double* xw, const unsigned long long* ga,
                                 const unsigned long long* gb, double* out) {
  ipc_pdl_wait();
  int e = blockIdx.x;
  __shared__ double sh[8];
  int cb0 = W.env_cbody[e];
  unsigned long long A = ga[e], B = gb[e];
  double best = INFINITY;
  for (int k = threadIdx.x; k < C.n_pt[e]; k += blockDim.x) {
    int2 pr = C.pt[C.pt_off[e] + k];
    int bv = W.slot_cbody[pr.x] - cb0, bt = W.tri_cbody[pr.y] - cb0;
    bool in = (((A >> bv) & 1) && ((B >> bt) & 1)) || (((B >> bv) & 1) && ((A >> bt) & 1));
    if (!in) continue;
    int3 tv = W.tri_v[pr.y];
    V3 p = ld3(xw + 3 * pr.x), t0 = ld3(xw + 3 * tv.x), t1 = ld3(xw + 3 * tv.y), t2 = ld3(xw + 3 * tv.z);
    best = fmin(best, pt_dist2(pt_region(p, t0, t1, t2), p, t0, t1, t2));
  }
  for (int k = threadIdx.x; k < C.n_ee[e]; k += blockDim.x) {
    int2 pr = C.ee[C.ee_off[e] + k];
    int b1 = W.edge_cbody[pr.x] - cb0, b2 = W.edge_cbody[pr.y] - cb0;
    bool in = (((A >> b1) & 1) && ((B >> b2) & 1)) || (((B >> b1) & 1) && ((A >> b2) & 1));
    if (!in) continue;
    int2 a = W.edge_v[pr.x], b = W.edge_v[pr.y];
    V3 a0 = ld3(xw + 3 * a.x), a1 = ld3(xw + 3 * a.y), b0 = ld3(xw + 3 * b.x), b1v = ld3(xw + 3 * b.y);
    best = fmin(best, ee_dist2(ee_region(a0, a1, b0, b1v, nullptr), a0, a1, b0, b1v));
  }
  // min-reduce (exact, order independent)
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_down_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmin(r, sh[w]);
    out[e] = isinf(r) ? INFINITY : sqrt(r);
  }
}
__global__ void k_ground_distance(World W, const double* xw, const unsigned long long* g, double* out) {
  ipc_pdl_wait();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= W.n_env) return;
  if (!W.env_has_ground[e]) {
    out[e] = INFINITY;
    return;
  }
  int cb0 = W.env_cbody[e];
  double lo = INFINITY;
  for (int s = W.env_slot[e]; s < W.env_slot[e + 1]; ++s)
    if ((g[e] >> (W.slot_cbody[s] - cb0)) & 1ull) lo = fmin(lo, xw[3 * s + 1]);
  out[e] = isinf(lo) ? INFINITY : lo - W.env_ground_y[e];
}
}  // namespace ipc


struct Pool {
  std::vector<void*> ptrs;
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    CK(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    ptrs.push_back(p);
    return (T*)p;
  }
  template <typename T>
  T* upload(const T* host, size_t n) {
    T* d = alloc<T>(n);
    if (host && n) CK(cudaMemcpy(d, host, n * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
  void free_one(void* p) {
    auto it = std::find(ptrs.begin(), ptrs.end(), p);
    if (it != ptrs.end()) {
      cudaFree(p);
      ptrs.erase(it);
    }
  }
  ~Pool() {
    for (void* p : ptrs) cudaFree(p);
  }
};

// candidate storage with per-env capacities
struct CandStore {
  Cands c{};
  std::vector<long long> pt_cap, ee_cap;  // per env
  long long* d_pt_off = nullptr;
  long long* d_ee_off = nullptr;
  long long pt_total = 0, ee_total = 0;
  int max_pt_cap = 0, max_ee_cap = 0;
};

// element output buffers sized to a candidate store
struct PairBufs {
  double *pt_val = nullptr, *ee_val = nullptr, *gnd_val = nullptr;
  double *pt_g = nullptr, *pt_h = nullptr, *ee_g = nullptr, *ee_h = nullptr;
  unsigned char *pt_act = nullptr, *ee_act = nullptr;
  double *gnd_gy = nullptr, *gnd_hyy = nullptr;
};

struct ipc_world {
  Pool pool;
  World W{};
  EnvState S{};
  int n_env = 0;
  std::vector<int> h_env_slot, h_env_dof, h_env_tri, h_env_edge, h_env_cbody;
  int max_env_dof = 0;
  CandStore dcd, sweep;
  CandStore ss;  // cached candidate superset of the fused per-env kernels (fused.cuh env_candidates)
  double *bb_lo = nullptr, *bb_hi = nullptr;
  double ss_pad = 2.0;  // IPC_SS_PAD: superset build-box padding in units of d̂ (0: off)
  PairBufs pb_dcd, pb_sweep;
  Lags L{};
  long long* d_lag_off = nullptr;
  Derivs D{};
  double *body_val = nullptr, *tet_val = nullptr, *fr_val = nullptr, *frg_val = nullptr;
  double *xlo = nullptr, *xhi = nullptr, *xwt = nullptr;
  double *env_alpha = nullptr;
  int *enable = nullptr, *ok = nullptr, *al_flag = nullptr, *accepted = nullptr, *ls_count = nullptr, *d_count = nullptr;
  int* env_order = nullptr;  // start order of the per-env dense-solve CTAs (k_env_order)
  bool use_env_order = getenv("IPC_ENV_ORDER") == nullptr || getenv("IPC_ENV_ORDER")[0] != '0';  // 0: identity
  int* h_count = nullptr;  // pinned
  double* slot_force = nullptr;
  double* d_targets = nullptr;
  bool lags_stale = false;
  std::vector<double> h_targets;
  bool targets_set = false;
  cudaStream_t st = 0;
  Prof prof;
  int n_sm = 148;
  long long stat_iters = 0, stat_ls_rounds = 0, stat_syncs = 0;
  int max_slots = 0;
  int* d_status = nullptr;
  int* h_status = nullptr;
  long long* work[2] = {nullptr, nullptr};
  int* work_env[2] = {nullptr, nullptr};
  int* work_n = nullptr;
  double* flush_buf = nullptr;
  double* sched = nullptr;
  int sched_steps = 0;
  std::vector<cudaEvent_t> marks;

  ~ipc_world() {
    drop_graphs();
    for (auto s2 : side)
      if (s2) cudaStreamDestroy(s2);
    for (auto e2 : fj)
      if (e2) cudaEventDestroy(e2);
    if (h_count) cudaFreeHost(h_count);
    if (h_status) cudaFreeHost(h_status);
  }

  int count(const int* flag) {
    IPC_LAUNCH(K_MISC, st, k_count, 1, 256, 0, n_env, flag, d_count);
    CK(cudaMemcpyAsync(h_count, d_count, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return *h_count;
  }

  void alloc_cands(CandStore& cs, const std::vector<long long>& ptc, const std::vector<long long>& eec) {
    drop_graphs();  // captured graphs hold the old buffer pointers by value
    cs.pt_cap = ptc;
    cs.ee_cap = eec;
    std::vector<long long> po(n_env + 1, 0), eo(n_env + 1, 0);
    cs.max_pt_cap = cs.max_ee_cap = 0;
    for (int e = 0; e < n_env; ++e) {
      po[e + 1] = po[e] + ptc[e];
      eo[e + 1] = eo[e] + eec[e];
      cs.max_pt_cap = std::max<long long>(cs.max_pt_cap, ptc[e]);
      cs.max_ee_cap = std::max<long long>(cs.max_ee_cap, eec[e]);
    }
    cs.pt_total = po[n_env];
    cs.ee_total = eo[n_env];
    if (cs.d_pt_off) { pool.free_one(cs.d_pt_off); pool.free_one(cs.d_ee_off); pool.free_one(cs.c.pt); pool.free_one(cs.c.ee); }
    cs.d_pt_off = pool.upload(po.data(), po.size());
    cs.d_ee_off = pool.upload(eo.data(), eo.size());
    cs.c.pt = pool.alloc<int2>(cs.pt_total);
    cs.c.ee = pool.alloc<int2>(cs.ee_total);
    cs.c.pt_off = cs.d_pt_off;
    cs.c.ee_off = cs.d_ee_off;
    if (!cs.c.gnd) {
      cs.c.gnd = pool.alloc<int>(W.n_slot);
      cs.c.n_pt = pool.alloc<int>(n_env);
      cs.c.n_ee = pool.alloc<int>(n_env);
      cs.c.n_gnd = pool.alloc<int>(n_env);
      cs.c.gnd_off = W.env_slot;
      cs.c.overflow = pool.alloc<int>(1);
      cs.c.pre_pt = pool.alloc<int>(n_env + 1);
      cs.c.pre_ee = pool.alloc<int>(n_env + 1);
      cs.c.pre_gnd = pool.alloc<int>(n_env + 1);
      cs.c.need_pt = pool.alloc<int>(n_env);
      cs.c.need_ee = pool.alloc<int>(n_env);
    }
    if (&cs == &dcd) {  // derivative work lists track the DCD capacity
      for (int k = 0; k < 2; ++k) {
        if (work[k]) { pool.free_one(work[k]); pool.free_one(work_env[k]); }
        long long n = k == 0 ? cs.pt_total : cs.ee_total;
        work[k] = pool.alloc<long long>(n);
        work_env[k] = pool.alloc<int>(n);
      }
      if (!work_n) work_n = pool.alloc<int>(2);
    }
  }

  void alloc_pairbufs(PairBufs& b, const CandStore& cs, bool derivs) {
    drop_graphs();
    for (void* p : {(void*)b.pt_val, (void*)b.ee_val, (void*)b.pt_g, (void*)b.pt_h, (void*)b.ee_g,
                    (void*)b.ee_h, (void*)b.pt_act, (void*)b.ee_act})
      if (p) pool.free_one(p);
    b.pt_val = pool.alloc<double>(cs.pt_total);
    b.ee_val = pool.alloc<double>(cs.ee_total);
    if (!b.gnd_val) b.gnd_val = pool.alloc<double>(W.n_slot);
    if (derivs) {
      b.pt_g = pool.alloc<double>(12 * cs.pt_total);
      b.pt_h = pool.alloc<double>(PK * cs.pt_total);
      b.ee_g = pool.alloc<double>(12 * cs.ee_total);
      b.ee_h = pool.alloc<double>(PK * cs.ee_total);
      b.pt_act = pool.alloc<unsigned char>(cs.pt_total);
      b.ee_act = pool.alloc<unsigned char>(cs.ee_total);
      if (!b.gnd_gy) {
        b.gnd_gy = pool.alloc<double>(W.n_slot);
        b.gnd_hyy = pool.alloc<double>(W.n_slot);
      }
    } else {
      b.pt_g = b.pt_h = b.ee_g = b.ee_h = nullptr;
      b.pt_act = b.ee_act = nullptr;
    }
  }

  void alloc_lags() {
    drop_graphs();
    std::vector<long long> lo(n_env + 1, 0);
    for (int e = 0; e < n_env; ++e) lo[e + 1] = lo[e] + dcd.pt_cap[e] + dcd.ee_cap[e];
    long long tot = lo[n_env];
    lag_total = tot;
    for (void* p : {(void*)d_lag_off, (void*)L.slots, (void*)L.gamma, (void*)L.tangent, (void*)L.lam,
                    (void*)fr_val, (void*)D.fr_g, (void*)D.fr_h})
      if (p) pool.free_one(p);
    d_lag_off = pool.upload(lo.data(), lo.size());
    L.off = d_lag_off;
    L.slots = pool.alloc<int4>(tot);
    L.gamma = pool.alloc<double>(4 * tot);
    L.tangent = pool.alloc<double>(6 * tot);
    L.lam = pool.alloc<double>(tot);
    if (!L.n) {
      L.n = pool.alloc<int>(n_env);
      L.g_slot = pool.alloc<int>(W.n_slot);
      L.g_lam = pool.alloc<double>(W.n_slot);
      L.g_n = pool.alloc<int>(n_env);
      frg_val = pool.alloc<double>(W.n_slot);
      D.frg_g = pool.alloc<double>(3 * W.n_slot);
      D.frg_h = pool.alloc<double>(9 * W.n_slot);
      L.pre = pool.alloc<int>(n_env + 1);
      L.g_pre = pool.alloc<int>(n_env + 1);
    }
    fr_val = pool.alloc<double>(tot);
    D.fr_g = pool.alloc<double>(12 * tot);
    D.fr_h = pool.alloc<double>(PK * tot);
  }

  // broad phase without a host round trip; overflow stays sticky in the
  // store's flag and is handled by replaying the step (see ipc_world_step)
  // broad phase over [lo, hi]: chunk boxes, then one CTA per env (bp_z == 1)
  // or bp_z CTAs per env in a count pass and a write pass
  static constexpr long long BROAD_ITEMS = 8192;
  int bp_z = 1;
  int* bp_cnt = nullptr;
  size_t broad_smem = 0;  // k_broad_sm: staged boxes of the largest env (0: unused)
  // broad phase over [lo, hi] into cs: through the cached candidate superset
  // (k_ss_check flags the envs whose query boxes left their build boxes, the
  // superset of those is rebuilt over the padded build boxes, k_ss_filter
  // extracts the exact lists; fused.cuh env_candidates), or directly
  int* ss_valid = nullptr;    // [n_env] superset holds the broad phase of the current build boxes
  int* ss_rebuild = nullptr;  // [n_env] scratch: envs to rebuild in this call
  // world_x: compute the world positions xw(world_x) into lo (== hi) first
  void launch_broad(CandStore& cs, const double* lo, const double* hi, const int* env_mask,
                    const double* world_x = nullptr) {
    int kid = &cs == &sweep ? K_BROAD_SWEEP : K_BROAD_DCD;
    if (ss_pad > 0.0 && &cs != &ss) {
      IPC_LAUNCH(kid, st, k_ss_check, n_env, 256, 0, W, lo, hi, bb_lo, bb_hi, ss_pad, env_mask, ss_valid, ss_rebuild,
                 world_x, const_cast<double*>(lo));
      launch_broad_raw(ss, bb_lo, bb_hi, ss_rebuild, kid);
      IPC_LAUNCH(kid, st, k_ss_filter, n_env, BP_THREADS, 0, W, lo, hi, ss.c, cs.c, env_mask, env_order);
      return;
    }
    if (world_x) world_pos(world_x, const_cast<double*>(lo));
    launch_broad_raw(cs, lo, hi, env_mask, kid);
  }
  void launch_broad_raw(CandStore& cs, const double* lo, const double* hi, const int* env_mask, int kid) {
    if (broad_smem && bp_z == 1) {
      IPC_LAUNCH(kid, st, k_broad_sm, n_env, BP_THREADS, broad_smem, W, lo, hi, cs.c, env_mask,
                 (int)(broad_smem / sizeof(double)), env_order);
      return;
    }
    IPC_LAUNCH(kid, st, k_chunk_boxes, nblk(W.n_tchunk + W.n_echunk, 128), 128, 0, W, lo, hi);
    if (W.n_tree)
      IPC_LAUNCH(kid, st, k_lbvh_build, W.n_tree, LBVH_THREADS, 4 * LBVH_MAX * sizeof(unsigned), W, lo, hi);
    if (bp_z == 1) {
      IPC_LAUNCH(kid, st, k_broad, dim3(n_env, 3), BP_THREADS, 0, W, lo, hi, cs.c, -1, env_mask, -1, nullptr);
    } else {
      IPC_LAUNCH(kid, st, k_broad, dim3(n_env, 3, bp_z), BP_THREADS, 0, W, lo, hi, cs.c, -1, env_mask, 0, bp_cnt);
      IPC_LAUNCH(kid, st, k_broad, dim3(n_env, 2, bp_z), BP_THREADS, 0, W, lo, hi, cs.c, -1, env_mask, 1, bp_cnt);
    }
  }
  // fill: optional per-env array set to v on the masked envs in the same launch
  void broad_nosync(CandStore& cs, const double* lo, const double* hi, const int* env_mask, double* fill = nullptr,
                    double v = 0.0, const double* world_x = nullptr) {
    launch_broad(cs, lo, hi, env_mask, world_x);
    IPC_LAUNCH(K_MISC, st, k_prefix3, fill && env_mask ? 4 : 3, 1024, 0, n_env, cs.c, env_mask, fill, v);
    if (fill && !env_mask) IPC_LAUNCH(K_MISC, st, k_fill, nblk(n_env, 128), 128, 0, n_env, fill, v);
  }

  // run broad phase; grow capacities and retry on overflow
  void broad(CandStore& cs, PairBufs& pb, bool derivs, const double* lo, const double* hi,
             const int* env_mask) {
    (void)pb;
    (void)derivs;
    for (int attempt = 0; attempt < 8; ++attempt) {
      // the superset store shares the sweep store's sticky flag
      CK(cudaMemsetAsync(cs.c.overflow, 0, sizeof(int), st));
      CK(cudaMemsetAsync(sweep.c.overflow, 0, sizeof(int), st));
      launch_broad(cs, lo, hi, env_mask);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(h_count, cs.c.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_status, sweep.c.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (!*h_count && !*h_status) {
        IPC_LAUNCH(K_MISC, st, k_prefix3, 3, 1024, 0, n_env, cs.c, env_mask, nullptr, 0.0);
        return;
      }
      // grow the overflowed stores to 1.5x their unclipped counts (at least 4x)
      grow_overflowed();
    }
    throw std::runtime_error("broad phase capacity overflow persists");
  }

  // contact pairs of (cs): light distance/value pass over every candidate of
  // the envs flagged at the last broad phase, then (deriv) the heavy
  // derivative pass over the compacted active list
  void pairs(const double* xw, CandStore& cs, PairBufs& pb, int deriv, double* min_s, int kid) {
    if (!cs.pt_total && !cs.ee_total) return;
    PairIO io{};
    io.val[0] = pb.pt_val; io.val[1] = pb.ee_val;
    io.act[0] = pb.pt_act; io.act[1] = pb.ee_act;
    io.g[0] = pb.pt_g; io.g[1] = pb.ee_g;
    io.h[0] = pb.pt_h; io.h[1] = pb.ee_h;
    io.work[0] = work[0]; io.work[1] = work[1];
    io.work_env[0] = work_env[0]; io.work_env[1] = work_env[1];
    io.work_n = work_n;
    if (deriv) CK(cudaMemsetAsync(work_n, 0, 2 * sizeof(int), st));
    IPC_LAUNCH(kid, st, k_pair_dist, dim3(n_sm * 8, 2), 128, 0, W, xw, cs.c, deriv, io, min_s);
    if (deriv) {  // the two kinds' derivative passes run as parallel branches
      fork_to(side[2], fj[3]);
      IPC_LAUNCH(kid == K_SENSE ? K_SENSE : K_PAIRS_D, side[2], k_pair_hess<1>, n_sm * 8, 64, 0, W, xw, cs.c, io);
      IPC_LAUNCH(kid == K_SENSE ? K_SENSE : K_PAIRS_D, st, k_pair_hess<0>, n_sm * 8, 64, 0, W, xw, cs.c, io);
      join_from(side[2], fj[3]);
    }
  }

  void world_pos(const double* x, double* xw) {
    IPC_LAUNCH(K_WORLD, st, k_world, nblk(W.n_slot, 256), 256, 0, W, x, xw);
  }

  // derivative or value pass of every term over (cands, lags)
  // side streams: independent element kernels run as parallel branches
  // (parallel graph branches when captured); fj: fork/join events
  cudaStream_t side[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t fj[4] = {nullptr, nullptr, nullptr, nullptr};
  void fork_to(cudaStream_t s2, cudaEvent_t ev) {
    CK(cudaEventRecord(ev, st));
    CK(cudaStreamWaitEvent(s2, ev, 0));
  }
  void join_from(cudaStream_t s2, cudaEvent_t ev) {
    CK(cudaEventRecord(ev, s2));
    CK(cudaStreamWaitEvent(st, ev, 0));
  }

  void terms(const double* x, const double* xw, CandStore& cs, PairBufs& pb, bool deriv, double h,
             const int* flag, double* min_s) {
    double h2 = h * h;
    int max_slots = 0;
    for (int e = 0; e < n_env; ++e) max_slots = std::max(max_slots, h_env_slot[e + 1] - h_env_slot[e]);
    // branch 1: affine bodies + tets; branch 2: ground + friction; main: pairs
    fork_to(side[0], fj[0]);
    CK(cudaStreamWaitEvent(side[1], fj[0], 0));
    IPC_LAUNCH(K_BODY, side[0], k_body, nblk(W.n_aff, 64), 64, 0, W, x, W.xhat, h2, deriv, flag, body_val, D.body_g,
               D.body_h);
    if (W.n_tet)
      IPC_LAUNCH(K_TET, side[0], k_tet, nblk(W.n_tet, 64), 64, 0, W, x, h2, deriv, flag, tet_val, D.tet_g, D.tet_h);
    IPC_LAUNCH(K_GROUND, side[1], k_ground, dim3(nblk(max_slots, 128), n_env), 128, 0, W, xw, cs.c, deriv, flag,
               pb.gnd_val, pb.gnd_gy, pb.gnd_hyy, min_s);
    IPC_LAUNCH(K_FRICTION, side[1], k_friction, n_sm * 4, 128, 0, W, xw, W.xw0, L, h, deriv, flag, fr_val, D.fr_g,
               D.fr_h);
    IPC_LAUNCH(K_FRICTION, side[1], k_friction_gnd, dim3(nblk(max_slots, 128), n_env), 128, 0, W, xw, W.xw0, L, h,
               deriv, flag, frg_val, D.frg_g, D.frg_h);
    pairs(xw, cs, pb, deriv, min_s, K_PAIRS_V);
    join_from(side[0], fj[1]);
    join_from(side[1], fj[2]);
    CK(cudaGetLastError());
  }

  void energy(const double* x, CandStore& cs, PairBufs& pb, const int* flag, double* out) {
    Terms T{body_val, tet_val, pb.pt_val, pb.ee_val, pb.gnd_val, fr_val, frg_val, nullptr};
    IPC_LAUNCH(K_ENERGY, st, k_env_energy, n_env, RED_THREADS, 0, W, x, W.xhat, T, cs.c, L, flag, out, env_order);
  }

  // ---- one Newton iteration = three fixed launch sequences ----------------
  // head: DCD broad phase, derivative pass of every term, E0, solve, check
  void seq_head(const ipc_step_config& cfg) {
    broad_nosync(dcd, W.xw, W.xw, S.newton_active, S.min_s, INFINITY, W.x);  // xw = world(x) first
    terms(W.x, W.xw, dcd, pb_dcd, true, cfg.h, S.newton_active, S.min_s);
    if (sparse) {
      energy(W.x, dcd, pb_dcd, S.newton_active, S.e0);
      sparse_solve(cfg);
    } else {  // E0 reduction as a parallel branch of the dense solve
      fork_to(side[0], fj[0]);
      Terms T{body_val, tet_val, pb_dcd.pt_val, pb_dcd.ee_val, pb_dcd.gnd_val, fr_val, frg_val, nullptr};
      IPC_LAUNCH(K_ENERGY, side[0], k_env_energy, n_env, RED_THREADS, 0, W, W.x, W.xhat, T, dcd.c, L, S.newton_active,
                 S.e0, env_order);
      IPC_LAUNCH(K_DENSE, st, k_dense_solve, n_env, DENSE_THREADS, dense_smem, W, S, D_with(pb_dcd), dcd.c, L, W.x,
                 W.xhat, W.p, W.grad, dense_timers(), env_order);
      join_from(side[0], fj[1]);
    }
    IPC_LAUNCH(K_MISC, st, k_newton_check, nblk(n_env, 128), 128, 0, n_env, S, cfg.h, cfg.newton_tol);
  }
  // CCD bound along p (ref solver.py:333-343)
  void seq_ccd(const ipc_step_config& cfg) {
    IPC_LAUNCH(K_MISC, st, k_sweep_slots, nblk(W.n_slot, 128), 128, 0, W, W.x, W.p, S.ls_active, W.xw, W.dxw, xlo,
               xhi);
    broad_nosync(sweep, xlo, xhi, S.ls_active, S.alpha_max, 1.0);
    fork_to(side[0], fj[0]);  // ground crossings as a parallel branch
    IPC_LAUNCH(K_CCD, side[0], k_ccd_ground, dim3(nblk(max_slots, 128), n_env), 128, 0, W, W.xw, W.dxw, sweep.c,
               cfg.ccd_conservative_factor, S.ls_active, S.alpha_max);
    if (sweep.pt_total || sweep.ee_total)
      IPC_LAUNCH(K_CCD, st, k_ccd_pairs, dim3(n_sm * 8, 2), 64, 0, W, W.xw, W.dxw, sweep.c,
                 cfg.ccd_conservative_factor, S.ls_active, S.alpha_max);
    join_from(side[0], fj[1]);
    if (sparse)  // dense worlds: folded into the first k_ls_value round
      IPC_LAUNCH(K_MISC, st, k_ls_begin, nblk(n_env, 128), 128, 0, n_env, S, ls_count);
  }
  // one backtracking round (ref solver.py:257): M speculative halvings
  void seq_ls_round(const ipc_step_config& cfg, int M, bool begin = false) {
    if (!sparse) {
      IPC_LAUNCH(K_ENERGY, st, k_ls_value, dim3(n_env, M), LS_THREADS, (size_t)3 * max_slots * sizeof(double), W, S,
                 sweep.c, L, W.x, W.p, W.xhat, cfg.h * cfg.h, cfg.h, e_multi, env_order, begin ? ls_count : nullptr);
    } else {
      double scale = 1.0;
      for (int m = 0; m < M; ++m, scale *= 0.5) {
        IPC_LAUNCH(K_MISC, st, k_axpy_env, nblk(W.n_dof, 256), 256, 0, W, W.x, W.p, S.alpha, scale, S.ls_active, W.xt);
        world_pos(W.xt, xwt);
        terms(W.xt, xwt, sweep, pb_sweep, false, cfg.h, S.ls_active, nullptr);
        energy(W.xt, sweep, pb_sweep, S.ls_active, e_multi + (size_t)m * n_env);
      }
    }
    IPC_LAUNCH(K_MISC, st, k_ls_check_apply, n_env, 64, 0, W, S, ls_count, cfg.max_line_search_halvings, M, e_multi,
               accepted, W.x, W.p);
  }
  void seq_ls(const ipc_step_config& cfg) { seq_ls_round(cfg, 1, true); }

  // M speculative halvings in one round (follow-up rounds only)
  static constexpr int LS_M = 8;    // trials of an iteration's first follow-up round
  static constexpr int LS_M2 = 32;  // trials of later rounds (few envs still backtracking)
  double* e_multi = nullptr;
  void seq_ls_multi(const ipc_step_config& cfg) { seq_ls_round(cfg, LS_M); }
  void seq_ls_multi2(const ipc_step_config& cfg) { seq_ls_round(cfg, LS_M2); }

  // ---- CUDA graphs of the sequences (dense worlds) ------------------------
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    long long kernels = 0;
    std::vector<Prof::Rec> timed;  // event pairs recorded inside the graph
  };
  Graph g_iter, g_ls, g_ls2;
  bool graphs_valid = false;
  bool use_graphs = true;
  ipc_step_config graph_cfg{};

  void grow_overflowed() {
    CK(cudaStreamSynchronize(st));
    // the broad phase records each env's unclipped candidate count: grow
    // straight to 1.5x that (at least 4x), so one replay suffices. An env that
    // overflowed one store grows all three (DCD ⊆ sweep ⊆ superset in practice),
    // so a step replay does not discover the same env again in another store.
    CandStore* stores[3] = {&dcd, &sweep, &ss};
    std::vector<long long> want_pt(n_env, 0), want_ee(n_env, 0);
    std::vector<int> hit(n_env, 0);
    for (CandStore* cs : stores) {
      std::vector<int> np(n_env), ne(n_env);
      CK(cudaMemcpy(np.data(), cs->c.need_pt, 4 * n_env, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ne.data(), cs->c.need_ee, 4 * n_env, cudaMemcpyDeviceToHost));
      for (int e = 0; e < n_env; ++e) {
        // overflowed, or within 25 % of overflowing: grow now rather than in a
        // later replay of the same step
        if (4 * (long long)np[e] > 3 * cs->pt_cap[e] || 4 * (long long)ne[e] > 3 * cs->ee_cap[e]) hit[e] = 1;
        want_pt[e] = std::max(want_pt[e], (long long)np[e]);
        want_ee[e] = std::max(want_ee[e], (long long)ne[e]);
        if (getenv("IPC_DEBUG_OVERFLOW") && (np[e] > cs->pt_cap[e] || ne[e] > cs->ee_cap[e]))
          fprintf(stderr, "[overflow] store %s env %d need pt %d / cap %lld, ee %d / cap %lld\n",
                  cs == &dcd ? "dcd" : (cs == &sweep ? "sweep" : "superset"), e, np[e], cs->pt_cap[e], ne[e],
                  cs->ee_cap[e]);
      }
    }
    for (CandStore* cs : stores) {
      std::vector<long long> ptc = cs->pt_cap, eec = cs->ee_cap;
      bool grew = false;
      for (int e = 0; e < n_env; ++e) {
        if (!hit[e]) continue;
        long long nv = h_env_slot[e + 1] - h_env_slot[e], nt = h_env_tri[e + 1] - h_env_tri[e];
        long long nE = h_env_edge[e + 1] - h_env_edge[e];
        long long p2 = std::min(nv * nt, std::max(want_pt[e] * 3 / 2, ptc[e]));
        long long e2 = std::min(nE * nE, std::max(want_ee[e] * 3 / 2, eec[e]));
        if (want_pt[e] > ptc[e]) p2 = std::min(nv * nt, std::max(p2, 4 * std::max(ptc[e], 1LL)));
        if (want_ee[e] > eec[e]) e2 = std::min(nE * nE, std::max(e2, 4 * std::max(eec[e], 1LL)));
        if (p2 != ptc[e] || e2 != eec[e]) grew = true;
        ptc[e] = p2;
        eec[e] = e2;
      }
      if (!grew) continue;
      alloc_cands(*cs, ptc, eec);
      if (cs != &ss) alloc_pairbufs(cs == &dcd ? pb_dcd : pb_sweep, *cs, cs == &dcd);
      if (cs == &dcd) lags_stale = true;
    }
    if (ss_valid) CK(cudaMemsetAsync(ss_valid, 0, sizeof(int) * n_env, st));
    drop_graphs();
  }

  void drop_graphs() {
    if (loop_exec) cudaGraphExecDestroy(loop_exec);
    loop_exec = nullptr;
    for (Graph* g : {&g_iter, &g_ls, &g_ls2}) {
      if (g->exec) cudaGraphExecDestroy(g->exec);
      g->exec = nullptr;
      for (auto& r : g->timed) { prof.pool.push_back(r.a); prof.pool.push_back(r.b); }
      g->timed.clear();
    }
    graphs_valid = false;
  }

  template <typename F>
  void capture(Graph& g, F body) {
    long long l0 = prof.launches;
    prof.capturing = true;
    prof.capture_list.clear();
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    body();
    cudaGraph_t graph;
    CK(cudaStreamEndCapture(st, &graph));
    prof.capturing = false;
    CK(cudaGraphInstantiate(&g.exec, graph, 0));
    CK(cudaGraphDestroy(graph));
    g.kernels = prof.launches - l0;
    prof.launches = l0;
    g.timed = prof.capture_list;
    prof.capture_list.clear();
  }

  static bool same_cfg(const ipc_step_config& a, const ipc_step_config& b) {
    return a.h == b.h && a.newton_tol == b.newton_tol && a.max_line_search_halvings == b.max_line_search_halvings &&
           a.ccd_conservative_factor == b.ccd_conservative_factor;
  }

  void ensure_graphs(const ipc_step_config& cfg) {
    if (graphs_valid && same_cfg(cfg, graph_cfg) && graph_prof_on == prof.on && graph_prof_mask == prof.mask)
      return;
    drop_graphs();
    capture(g_iter, [&] {
      seq_head(cfg);
      seq_ccd(cfg);
      seq_ls(cfg);
    });
    capture(g_ls, [&] { seq_ls_multi(cfg); });
    capture(g_ls2, [&] { seq_ls_multi2(cfg); });
    graph_cfg = cfg;
    graph_prof_on = prof.on;
    graph_prof_mask = prof.mask;
    graphs_valid = true;
  }
  bool graph_prof_on = false;
  unsigned graph_prof_mask = 0;

  void run(Graph& g) {
    CK(cudaGraphLaunch(g.exec, st));
    prof.launches += g.kernels;
    if (!g.timed.empty()) graph_timed.push_back(&g);
  }
  std::vector<Graph*> graph_timed;  // graphs whose event pairs await a sync

  // device status after a sync: active counts + sticky overflow
  struct Status {
    int newton, ls, overflow;
  };
  Status status() {
    IPC_LAUNCH(K_MISC, st, k_status, 1, 256, 0, n_env, S.newton_active, S.ls_active, dcd.c.overflow,
               sweep.c.overflow, d_status);
    CK(cudaMemcpyAsync(h_status, d_status, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ++stat_syncs;
    for (Graph* g : graph_timed)
      for (auto& r : g->timed) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, r.a, r.b));
        prof.ms[r.kid] += t;
        prof.cnt[r.kid] += 1;
      }
    graph_timed.clear();
    if (h_status[2]) throw OverflowRetry();
    return Status{h_status[0], h_status[1], h_status[2]};
  }

  // ---- device-driven Newton loop: one graph launch per Newton solve ------
  // WHILE(h_loop) { SWITCH(h_mode) { 0: Newton iteration (g_iter's
  // sequence), 1: line-search round (g_ls's) }; k_loop_ctl } — no host round
  // trip per iteration or per line-search round. Used when no kernel of the
  // loop is being event-timed (conditional bodies take no event nodes).
  cudaGraphExec_t loop_exec = nullptr;
  ipc_step_config loop_cfg{};
  int loop_tail = -1;
  int* d_loopctl = nullptr;
  bool use_loop_graph = getenv("IPC_LOOP_GRAPH") == nullptr || getenv("IPC_LOOP_GRAPH")[0] != '0';  // 0: host loop

  void build_loop_graph(const ipc_step_config& cfg, int tail) {
    if (loop_exec) cudaGraphExecDestroy(loop_exec);
    loop_exec = nullptr;
    if (!d_loopctl) d_loopctl = pool.alloc<int>(8);
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_loop, h_mode;
    CK(cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_loop;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    CK(cudaGraphConditionalHandleCreate(&h_mode, body, 0, cudaGraphCondAssignDefault));
    cudaGraphNodeParams sp = {};
    sp.type = cudaGraphNodeTypeConditional;
    sp.conditional.handle = h_mode;
    sp.conditional.type = cudaGraphCondTypeSwitch;
    sp.conditional.size = 3;
    cudaGraphNode_t snode;
    CK(cudaGraphAddNode(&snode, body, nullptr, 0, &sp));
    cudaGraph_t b_iter = sp.conditional.phGraph_out[0], b_ls = sp.conditional.phGraph_out[1],
                b_ls2 = sp.conditional.phGraph_out[2];
    const bool prof_on = prof.on;
    prof.on = false;  // conditional bodies take no event nodes
    auto capture_into = [&](cudaGraph_t target, const cudaGraphNode_t* deps, size_t ndep, auto fn) {
      long long l0 = prof.launches;
      prof.capturing = true;
      CK(cudaStreamBeginCaptureToGraph(st, target, deps, nullptr, ndep, cudaStreamCaptureModeThreadLocal));
      fn();
      cudaGraph_t out;
      CK(cudaStreamEndCapture(st, &out));
      prof.capturing = false;
      prof.launches = l0;
    };
    capture_into(b_iter, nullptr, 0, [&] {
      seq_head(cfg);
      seq_ccd(cfg);
      seq_ls(cfg);
    });
    capture_into(b_ls, nullptr, 0, [&] { seq_ls_multi(cfg); });
    capture_into(b_ls2, nullptr, 0, [&] { seq_ls_multi2(cfg); });
    // the control kernel follows the SWITCH in the body
    capture_into(body, &snode, 1, [&] {
      k_loop_ctl<<<1, 1024, 0, st>>>(n_env, S.newton_active, S.ls_active, dcd.c.overflow, sweep.c.overflow,
                                     d_loopctl, cfg.max_newton_iters, cfg.max_line_search_halvings, LS_M, LS_M2,
                                     tail, h_loop, h_mode);
      CK(cudaPeekAtLastError());
    });
    CK(cudaGraphInstantiate(&loop_exec, g, 0));
    CK(cudaGraphDestroy(g));
    CK(cudaGraphUpload(loop_exec, st));
    prof.on = prof_on;
    loop_cfg = cfg;
    loop_tail = tail;
  }

  bool loop_graph_usable() const {
    if (!use_loop_graph || sparse || !use_graphs) return false;
    // conditional bodies take no event nodes: only when no loop kernel is timed
    const unsigned loop_kernels = ~((1u << K_FUSED) | (1u << K_SENSE));
    return !(prof.on && (prof.mask & loop_kernels));
  }

  void newton_solve(const ipc_step_config& cfg) {
    IPC_LAUNCH(K_MISC, st, k_newton_begin, nblk(n_env, 128), 128, 0, n_env, S, al_flag);
    // start order of the per-env CTAs for this solve, from the latest
    // candidate and lag counts (only scheduling: any order gives the same bits)
    if (!sparse && use_env_order)
      IPC_LAUNCH(K_MISC, st, k_env_order, n_env <= ORDER_MAX ? (n_env + ORDER_ENVS - 1) / ORDER_ENVS : 148,
                 ORDER_ENVS * 32, 0, n_env, S.newton_active, dcd.c, L, env_order);
    bool graphs = use_graphs && !sparse;
    if (graphs) ensure_graphs(cfg);
    int tail = 0;
    if (graphs && use_loop_graph) {
      // the loop hands off to the per-env tail kernel only when it can run;
      // built (and uploaded) even while kernel timing keeps the host loop in
      // use, so switching the timers off never costs an instantiation
      tail = (tail_envs > 0 && fused_setup()) ? tail_envs : 0;
      if (!loop_exec || !same_cfg(cfg, loop_cfg) || cfg.max_newton_iters != loop_cfg.max_newton_iters ||
          loop_tail != tail)
        build_loop_graph(cfg, tail);
    }
    if (graphs && loop_graph_usable()) {
      CK(cudaMemsetAsync(d_loopctl, 0, 8 * sizeof(int), st));
      CK(cudaGraphLaunch(loop_exec, st));
      int ctl[5];
      CK(cudaMemcpyAsync(h_status, d_loopctl, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_status + 4, d_loopctl + 4, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      ++stat_syncs;
      for (int i = 0; i < 5; ++i) ctl[i] = h_status[i];
      stat_iters += ctl[0];
      stat_ls_rounds += ctl[2];
      if (ctl[4]) throw OverflowRetry();
      int active = ctl[3], it = ctl[0] - 1;
      if (active > 0 && tail > 0 && active <= tail && it + 1 < cfg.max_newton_iters) {
        CK(cudaMemsetAsync(fq, 0, sizeof(int), st));
        FusedArgs A = fused_args(cfg);
        IPC_LAUNCH(K_FUSED, st, k_env_newton_rest, std::min(active, fused_blocks), 256, fused_smem, A, it + 1);
        status();
      }
      IPC_LAUNCH(K_MISC, st, k_mark_unconverged, nblk(n_env, 128), 128, 0, n_env, S);
      return;
    }
    for (int it = 0; it < cfg.max_newton_iters; ++it) {
      if (graphs) {
        run(g_iter);
      } else {
        seq_head(cfg);
        seq_ccd(cfg);
        seq_ls(cfg);
      }
      ++stat_iters;
      ++stat_ls_rounds;
      Status s = status();
      for (int ls = 1, r = 0; s.ls && ls < cfg.max_line_search_halvings + 1; ls += r++ == 0 ? LS_M : LS_M2) {
        if (r == 0) {
          if (graphs) run(g_ls); else seq_ls_multi(cfg);
        } else {
          if (graphs) run(g_ls2); else seq_ls_multi2(cfg);
        }
        ++stat_ls_rounds;
        s = status();
      }
      if (s.newton == 0) break;
      // few envs left: finish their Newton loops in per-env CTAs
      if (graphs && tail_envs > 0 && s.newton <= tail_envs && it + 1 < cfg.max_newton_iters && fused_setup()) {
        CK(cudaMemsetAsync(fq, 0, sizeof(int), st));
        FusedArgs A = fused_args(cfg);
        IPC_LAUNCH(K_FUSED, st, k_env_newton_rest, std::min(s.newton, fused_blocks), 256, fused_smem, A, it + 1);
        status();
        break;
      }
    }
    // envs still active after the iteration cap did not converge
    IPC_LAUNCH(K_MISC, st, k_mark_unconverged, nblk(n_env, 128), 128, 0, n_env, S);
  }

  // ---------------- fused per-env step (dense worlds) ----------------
  bool fused_on = false;    // IPC_FUSED=1: whole step in the fused per-env kernel
  bool fused_timers_on = false;  // IPC_FUSED_TIMERS=1: per-phase SM cycles of the fused kernels
  int tail_envs = 444;      // batched schedule: hand off to per-env CTAs at <= this many active envs (3 x SMs)
  int fused_max_dof = 128;  // dense LDLᵀ in shared memory: n² doubles
  int* fq = nullptr;
  long long* d_fstat = nullptr;
  double *v_save = nullptr, *kappa_save = nullptr;
  int fused_blocks = 0;
  size_t fused_smem = 0;
  size_t dense_smem = 0;
  int max_env_prims = 0;  // max over envs of slots + tris + edges + chunks
  int max_env_groups = 0;  // max over envs of soft vertices + affine bodies
  bool use_fused() const { return fused_on && !sparse && max_env_dof <= fused_max_dof; }

  void read_reports(ipc_step_report* rep);
  // dense sub-phase timers (IPC_FUSED_TIMERS=1) of the batched k_dense_solve:
  // the same counters as the fused kernels' dense_solve_block
  long long* dense_timers() { return (fused_timers_on && d_fstat) ? d_fstat + 2 + FT_DENSE_SUB : nullptr; }

  // shared setup of the fused kernels; false when the env systems do not fit
  bool fused_setup() {
    if (!fq) {
      fq = pool.alloc<int>(1);
      d_fstat = pool.alloc<long long>(2 + FT_TOTAL);
      CK(cudaMemset(d_fstat, 0, sizeof(long long) * (2 + FT_TOTAL)));
      v_save = pool.alloc<double>(W.n_dof);
      kappa_save = pool.alloc<double>(n_env);
    }
    if (!fused_blocks) {
      // time-shared scratch: dense system, line-search positions, staged
      // broad-phase boxes (6 doubles per slot / primitive / chunk)
      size_t need = std::max(dense_smem_doubles(max_env_dof), 3 * max_slots);
      need = std::max(need, (size_t)6 * max_env_prims);
      int dev = 0, optin = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, k_env_step));
      size_t avail = (size_t)optin - fa.sharedSizeBytes;
      size_t base = sizeof(double) * (size_t)dense_smem_doubles(max_env_dof);
      fused_smem = std::min(avail, sizeof(double) * need);
      if (fused_smem < base) {  // cannot hold the dense system: batched path
        fused_on = false;
        return false;
      }
      CK(cudaFuncSetAttribute(k_env_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem));
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_env_step, 256, fused_smem));
      fused_blocks = std::max(1, std::min(n_env, std::max(per_sm, 1) * n_sm));
      CK(cudaFuncSetAttribute(k_env_newton_rest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem));
      CK(cudaFuncSetAttribute(k_env_steps, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem));
    }
    return true;
  }

  FusedArgs fused_args(const ipc_step_config& cfg) {
    FusedArgs A{};
    A.order = env_order;
    A.W = W;
    A.S = S;
    A.dc = dcd.c;
    A.sw = sweep.c;
    A.ss = ss.c;
    A.bb_lo = bb_lo;
    A.bb_hi = bb_hi;
    A.ss_pad = ss_pad;
    A.L = L;
    A.D = D_with(pb_dcd);
    A.T = Terms{body_val, tet_val, pb_dcd.pt_val, pb_dcd.ee_val, pb_dcd.gnd_val, fr_val, frg_val, nullptr};
    A.xwt = xwt;
    A.xlo = xlo;
    A.xhi = xhi;
    A.enable = enable;
    A.ok = ok;
    A.accepted = accepted;
    A.ls_count = ls_count;
    A.targets = d_targets;
    A.queue = fq;
    A.stat = d_fstat;
    A.timers = fused_timers_on ? d_fstat + 2 : nullptr;
    A.h = cfg.h;
    A.newton_tol = cfg.newton_tol;
    A.ccd_cons = cfg.ccd_conservative_factor;
    A.max_newton = cfg.max_newton_iters;
    A.max_halvings = cfg.max_line_search_halvings;
    A.fp_iters = std::max(cfg.friction_fixed_point_iters, 1);
    A.al_max_outer = cfg.al_max_outer;
    A.smem_doubles = (int)(fused_smem / sizeof(double));
    return A;
  }

  bool step_fused(const ipc_step_config& cfg) {
    if (lags_stale) {
      alloc_lags();
      lags_stale = false;
    }
    if (!fused_setup()) return false;
    // the step commits v and κ in place: keep copies for an overflow replay
    CK(cudaMemcpyAsync(v_save, W.v, sizeof(double) * W.n_dof, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(kappa_save, W.env_kappa, sizeof(double) * n_env, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(fq, 0, sizeof(int), st));
    FusedArgs A = fused_args(cfg);
    IPC_LAUNCH(K_FUSED, st, k_env_step, fused_blocks, 256, fused_smem, A);
    CK(cudaMemcpyAsync(h_status, dcd.c.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_status + 1, sweep.c.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ++stat_syncs;
    if (h_status[0] || h_status[1]) {
      CK(cudaMemcpyAsync(W.v, v_save, sizeof(double) * W.n_dof, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(W.env_kappa, kappa_save, sizeof(double) * n_env, cudaMemcpyDeviceToDevice, st));
      throw OverflowRetry();
    }
    return true;
  }

  // ---------------- sparse path (large environments) ----------------
  bool sparse = false;
  Pcg pcg{};
  int* d_counts = nullptr;
  long long* d_offs = nullptr;
  long long n_el_cap = 0, items_cap = 0;
  unsigned long long *keys = nullptr, *keys_sorted = nullptr;
  double* vals = nullptr;
  int *idx = nullptr, *perm = nullptr, *heads = nullptr;
  long long *uidx = nullptr, *seg_start = nullptr;
  unsigned* bcol = nullptr;
  double* bval = nullptr;
  int *row_cnt = nullptr, *row_first = nullptr, *bpos = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  long long lag_total = 0;
  double* g_asm = nullptr;
  int pcg_max_iters = 20000;
  double pcg_rtol = 1e-14;  // relative residual; 1e-12 left config 2 at 1.3e-6 DoF error vs the reference (splu)
  int coop_blocks = 0;
  int* d_nlive = nullptr;
  double* d_beta = nullptr;
  double* d_part1 = nullptr;
  double* d_part2 = nullptr;
  long long* h_ll = nullptr;  // pinned scalars

  void setup_sparse(const ipc_world_desc* d) {
    int nn = d->n_dof / 3;
    std::vector<int> node_env(nn), chunk_env, c0, c1, env_chunk(n_env + 1, 0);
    // env-aligned reduction chunks: small enough that the PCG spreads over
    // the SMs even for a single large env, at most 256 nodes
    int CH = std::max(32, std::min(256, ((nn + 2 * n_sm - 1) / (2 * n_sm) + 31) / 32 * 32));
    // affine bodies: 4 consecutive nodes each, preconditioned as one 12x12 block
    std::vector<int> node_aff(nn, -1), aff_node0(std::max(d->n_aff, 1), 0);
    for (int b = 0; b < d->n_aff; ++b) {
      int n0 = d->aff_dof[b] / 3;
      aff_node0[b] = n0;
      for (int q = 0; q < 4; ++q) node_aff[n0 + q] = b;
    }
    for (int e = 0; e < n_env; ++e) {
      int a = d->env_dof[e] / 3, b = d->env_dof[e + 1] / 3;
      for (int i = a; i < b; ++i) node_env[i] = e;
      env_chunk[e] = (int)chunk_env.size();
      for (int s = a; s < b;) {
        int t = std::min(b, s + CH);
        if (t < b && node_aff[t] >= 0) t = aff_node0[node_aff[t]] + 4;  // never split a body
        chunk_env.push_back(e);
        c0.push_back(s);
        c1.push_back(t);
        s = t;
      }
    }
    pcg.node_aff = pool.upload(node_aff.data(), nn);
    pcg.aff_node0 = pool.upload(aff_node0.data(), aff_node0.size());
    pcg.Minv12 = pool.alloc<double>(144 * (size_t)std::max(d->n_aff, 1));
    {
      const char* pa = getenv("IPC_PCG_AFF");
      pcg.aff_blocks = (pa && pa[0] == '0') ? 0 : 1;
      const char* pr = getenv("IPC_PCG_RTOL");
      if (pr) pcg_rtol = atof(pr);
      const char* pm = getenv("IPC_PCG_MAXIT");
      if (pm) pcg_max_iters = std::max(1, atoi(pm));
    }
    env_chunk[n_env] = (int)chunk_env.size();
    pcg.n_node = nn;
    pcg.n_chunk = (int)chunk_env.size();
    pcg.node_env = pool.upload(node_env.data(), nn);
    pcg.chunk_env = pool.upload(chunk_env.data(), chunk_env.size());
    pcg.chunk_n0 = pool.upload(c0.data(), c0.size());
    pcg.chunk_n1 = pool.upload(c1.data(), c1.size());
    pcg.env_chunk = pool.upload(env_chunk.data(), env_chunk.size());
    pcg.x = pool.alloc<double>(d->n_dof);
    pcg.r = pool.alloc<double>(d->n_dof);
    pcg.z = pool.alloc<double>(d->n_dof);
    pcg.p = pool.alloc<double>(d->n_dof);
    pcg.Ap = pool.alloc<double>(d->n_dof);
    pcg.Minv = pool.alloc<double>(9 * (size_t)nn);
    pcg.part = pool.alloc<double>(2 * (size_t)std::max(pcg.n_chunk, 1));
    pcg.env_rz = pool.alloc<double>(n_env);
    pcg.env_rz_new = pool.alloc<double>(n_env);
    pcg.env_pap = pool.alloc<double>(n_env);
    pcg.env_bb = pool.alloc<double>(n_env);
    pcg.env_rr = pool.alloc<double>(n_env);
    pcg.env_live = pool.alloc<int>(n_env);
    row_cnt = pool.alloc<int>(nn);
    row_first = pool.alloc<int>(nn);
    g_asm = pool.alloc<double>(d->n_dof);
    CK(cudaMallocHost(&h_ll, 4 * sizeof(long long)));
    d_nlive = pool.alloc<int>(3);
    CK(cudaMemset(d_nlive, 0, 3 * sizeof(int)));
    d_part2 = pool.alloc<double>(2 * (size_t)std::max(pcg.n_chunk, 1));
    d_beta = pool.alloc<double>(n_env);
    d_part1 = pool.alloc<double>(2 * (size_t)std::max(pcg.n_chunk, 1));
  }

  template <typename T>
  void grow(T*& p, long long& cap_track, long long need, long long mult = 1) {
    (void)cap_track;
    if (p) pool.free_one(p);
    p = pool.alloc<T>((size_t)(need * mult));
  }

  void ensure_cub(size_t need) {
    if (need > cub_tmp_bytes) {
      if (cub_tmp) pool.free_one(cub_tmp);
      cub_tmp = pool.alloc<char>(need);
      cub_tmp_bytes = need;
    }
  }

  // assemble the BSR Newton system of every active env and solve it with
  // block-Jacobi PCG; writes W.p, W.grad, S.pnorm, S.gnorm
  void sparse_solve(const ipc_step_config& cfg) {
    (void)cfg;
    ElemSpace sp{W.n_vert, W.n_aff, W.n_tet, dcd.pt_total, dcd.ee_total, W.n_slot, lag_total, W.n_slot};
    long long n_el = sp.n_vert + sp.n_aff + sp.n_tet + sp.n_pt + sp.n_ee + sp.n_gnd + sp.n_fr + sp.n_frg;
    if (n_el > n_el_cap) {
      if (d_counts) { pool.free_one(d_counts); pool.free_one(d_offs); }
      d_counts = pool.alloc<int>(n_el);
      d_offs = pool.alloc<long long>(n_el);
      n_el_cap = n_el;
    }
    AsmIn A{W, S, D_with(pb_dcd), dcd.c, L, W.x, W.xhat, sp};
    IPC_LAUNCH(K_ASM, st, k_asm_count, n_sm * 8, 128, 0, A, d_counts);
    size_t need = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, need, d_counts, d_offs, n_el, st));
    ensure_cub(need);
    CK(cub::DeviceScan::ExclusiveSum(cub_tmp, need, d_counts, d_offs, n_el, st));
    CK(cudaMemcpyAsync(h_ll, d_offs + n_el - 1, sizeof(long long), cudaMemcpyDeviceToHost, st));
    int last = 0;
    CK(cudaMemcpyAsync(h_count, d_counts + n_el - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    last = *h_count;
    long long n_items = h_ll[0] + last;
    if (n_items > items_cap) {
      for (void* q : {(void*)keys, (void*)keys_sorted, (void*)vals, (void*)idx, (void*)perm, (void*)heads,
                      (void*)uidx, (void*)seg_start, (void*)bcol, (void*)bval, (void*)bpos})
        if (q) pool.free_one(q);
      long long c = std::max(n_items + n_items / 2, 1LL << 16);
      keys = pool.alloc<unsigned long long>(c);
      keys_sorted = pool.alloc<unsigned long long>(c);
      vals = pool.alloc<double>(9 * c);
      idx = pool.alloc<int>(c);
      perm = pool.alloc<int>(c);
      heads = pool.alloc<int>(c);
      uidx = pool.alloc<long long>(c);
      seg_start = pool.alloc<long long>(c);
      bcol = pool.alloc<unsigned>(c);
      bval = pool.alloc<double>(9 * c);
      bpos = pool.alloc<int>(c);
      items_cap = c;
    }
    IPC_LAUNCH(K_ASM, st, k_asm_emit, n_sm * 8, 128, 0, A, d_offs, keys, vals, idx);
    need = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, need, keys, keys_sorted, idx, perm, n_items, 0, 64, st));
    ensure_cub(need);
    CK(cub::DeviceRadixSort::SortPairs(cub_tmp, need, keys, keys_sorted, idx, perm, n_items, 0, 64, st));
    IPC_LAUNCH(K_ASM, st, k_asm_heads, n_sm * 8, 256, 0, n_items, keys_sorted, heads);
    need = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, need, heads, uidx, n_items, st));
    ensure_cub(need);
    CK(cub::DeviceScan::ExclusiveSum(cub_tmp, need, heads, uidx, n_items, st));
    CK(cudaMemcpyAsync(h_ll, uidx + n_items - 1, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_count, heads + n_items - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    long long n_unique = h_ll[0] + *h_count;
    IPC_LAUNCH(K_ASM, st, k_asm_starts, n_sm * 8, 256, 0, n_items, heads, uidx, seg_start);
    CK(cudaMemsetAsync(row_cnt, 0, sizeof(int) * pcg.n_node, st));
    CK(cudaMemsetAsync(g_asm, 0, sizeof(double) * W.n_dof, st));
    IPC_LAUNCH(K_ASM, st, k_asm_reduce, n_sm * 8, 128, 0, n_items, n_unique, keys_sorted, seg_start, perm, vals,
               g_asm, bcol, bval, row_cnt, bpos);
    IPC_LAUNCH(K_ASM, st, k_bsr_rowfirst, n_sm * 8, 256, 0, n_unique, keys_sorted, seg_start, row_first);
    // PCG
    pcg.row_first = row_first;
    pcg.row_cnt = row_cnt;
    pcg.bcol = bcol;
    pcg.bval = bval;
    pcg.env_on = S.newton_active;
    double rtol2 = pcg_rtol * pcg_rtol;
    IPC_LAUNCH(K_DENSE, st, k_pcg_setup, n_sm * 8, 128, 0, pcg, g_asm);
    IPC_LAUNCH(K_DENSE, st, k_pcg_setup_z, n_sm * 8, 128, 0, pcg);
    IPC_LAUNCH(K_DENSE, st, k_pcg_partial, std::max(pcg.n_chunk, 1), 256, 0, pcg, 0);
    IPC_LAUNCH(K_DENSE, st, k_pcg_env, nblk(n_env, 128), 128, 0, pcg, n_env, 0, rtol2);
    {
      // persistent cooperative PCG: all iterations in one launch
      if (!coop_blocks) {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_coop, 256, 0));
        // one block per reduction chunk: idle blocks would only lengthen every grid barrier
        coop_blocks = std::max(1, std::min(std::min(per_sm, 4) * n_sm, pcg.n_chunk));
      }
      CK(cudaMemsetAsync(d_nlive, 0, 2 * sizeof(int), st));
      int iters = pcg_max_iters;
      void* args[] = {(void*)&pcg, (void*)&n_env, (void*)&rtol2, (void*)&iters, (void*)&d_nlive, (void*)&d_part1, (void*)&d_part2};
      prof_begin(K_PCG, st);
      CK(cudaLaunchCooperativeKernel((void*)k_pcg_coop, dim3(coop_blocks), dim3(256), args, 0, st));
      prof_end(K_PCG, st);
    }
    IPC_LAUNCH(K_DENSE, st, k_pcg_finish, n_env, 256, 0, W, S, pcg, g_asm, W.p, W.grad);
    CK(cudaGetLastError());
  }

  Derivs D_with(const PairBufs& pb) {
    Derivs d = D;
    d.pt_g = pb.pt_g; d.pt_h = pb.pt_h; d.ee_g = pb.ee_g; d.ee_h = pb.ee_h;
    d.pt_act = pb.pt_act; d.ee_act = pb.ee_act;
    d.gnd_gy = pb.gnd_gy; d.gnd_hyy = pb.gnd_hyy;
    return d;
  }
};


// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* ipc_last_error(void) { return g_err.c_str(); }

int ipc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int ipc_world_create(const ipc_world_desc* d, ipc_world** out) {
  ipc_world* w = nullptr;
  try {
    if (ipc_device_count() == 0) return set_err("no CUDA device");
    w = new ipc_world();
    Pool& P = w->pool;
    World& W = w->W;
    int ne = d->n_env;
    w->n_env = ne;
    W.n_env = ne; W.n_dof = d->n_dof; W.n_vert = d->n_vert; W.n_aff = d->n_aff; W.n_tet = d->n_tet;
    W.n_slot = d->n_slot; W.n_tri = d->n_tri; W.n_edge = d->n_edge; W.n_cbody = d->n_cbody; W.n_cons = d->n_cons;
    W.env_dof = P.upload(d->env_dof, ne + 1);
    W.env_vert = P.upload(d->env_vert, ne + 1);
    W.env_aff = P.upload(d->env_aff, ne + 1);
    W.env_tet = P.upload(d->env_tet, ne + 1);
    W.env_slot = P.upload(d->env_slot, ne + 1);
    W.env_tri = P.upload(d->env_tri, ne + 1);
    W.env_edge = P.upload(d->env_edge, ne + 1);
    W.env_cbody = P.upload(d->env_cbody, ne + 1);
    W.env_cons = P.upload(d->env_cons, ne + 1);
    W.env_pairs = P.upload(d->env_pairs, ne);
    W.env_has_ground = P.upload(d->env_has_ground, ne);
    W.env_ground_y = P.upload(d->env_ground_y, ne);
    W.env_gravity = P.upload(d->env_gravity, 3 * ne);
    W.env_dhat = P.upload(d->env_dhat, ne);
    W.env_kappa = P.upload(d->env_kappa, ne);
    W.env_kappa0 = P.upload(d->env_kappa0, ne);
    W.env_mu = P.upload(d->env_mu, ne);
    W.env_epsv = P.upload(d->env_eps_v, ne);
    // per-element env ids
    auto expand = [&](const int32_t* pre, int n) {
      std::vector<int> v(std::max(n, 1), 0);
      for (int e = 0; e < ne; ++e)
        for (int i = pre[e]; i < pre[e + 1]; ++i) v[i] = e;
      return P.upload(v.data(), v.size());
    };
    W.dof_env = expand(d->env_dof, d->n_dof);
    W.vert_env = expand(d->env_vert, d->n_vert);
    W.aff_env = expand(d->env_aff, d->n_aff);
    W.tet_env = expand(d->env_tet, d->n_tet);
    W.slot_env = expand(d->env_slot, d->n_slot);
    W.cons_env = expand(d->env_cons, d->n_cons);
    W.x = P.upload(d->x0, d->n_dof);
    W.v = P.upload(d->v0, d->n_dof);
    W.x_prev = P.alloc<double>(d->n_dof);
    W.xhat = P.alloc<double>(d->n_dof);
    W.p = P.alloc<double>(d->n_dof);
    W.xt = P.alloc<double>(d->n_dof);
    W.grad = P.alloc<double>(d->n_dof);
    W.vert_dof = P.upload(d->vert_dof, d->n_vert);
    W.vert_mass = P.upload(d->vert_mass, d->n_vert);
    W.aff_dof = P.upload(d->aff_dof, d->n_aff);
    W.aff_M = P.upload(d->aff_M, 144 * (size_t)d->n_aff);
    W.aff_acc = P.upload(d->aff_acc, 12 * (size_t)d->n_aff);
    W.aff_ortho = P.upload(d->aff_ortho, d->n_aff);
    W.tet_dof = (const int4*)P.upload(d->tet_dof, 4 * (size_t)d->n_tet);
    W.tet_Dminv = P.upload(d->tet_Dminv, 9 * (size_t)d->n_tet);
    W.tet_vol = P.upload(d->tet_vol, d->n_tet);
    W.tet_mu = P.upload(d->tet_mu, d->n_tet);
    W.tet_lam = P.upload(d->tet_lam, d->n_tet);
    W.tet_model = P.upload(d->tet_model, d->n_tet);
    W.slot_aff = P.upload(d->slot_aff, d->n_slot);
    W.slot_dof = P.upload(d->slot_dof, d->n_slot);
    W.slot_rest = P.upload(d->slot_rest, 3 * (size_t)d->n_slot);
    W.slot_cbody = P.upload(d->slot_cbody, d->n_slot);
    W.tri_v = (const int3*)P.upload(d->tri_v, 3 * (size_t)d->n_tri);
    W.tri_cbody = P.upload(d->tri_cbody, d->n_tri);
    W.edge_v = (const int2*)P.upload(d->edge_v, 2 * (size_t)d->n_edge);
    W.edge_cbody = P.upload(d->edge_cbody, d->n_edge);
    W.edge_len2 = P.upload(d->edge_len2, d->n_edge);
    W.cbody_rigid = P.upload(d->cbody_rigid, d->n_cbody);
    W.cbody_kin = P.upload(d->cbody_kin, d->n_cbody);
    W.cbody_excl = (const unsigned long long*)P.upload(d->cbody_excl, d->n_cbody);
    {
      // contiguous per-body primitive ranges (slots/tris/edges are emitted body by body)
      auto ranges = [&](const int32_t* owner, int n) {
        std::vector<int> pre(d->n_cbody + 1, 0);
        for (int i = 0; i < n; ++i) pre[owner[i] + 1]++;
        for (int b = 0; b < d->n_cbody; ++b) pre[b + 1] += pre[b];
        for (int i = 1; i < n; ++i)
          if (owner[i] < owner[i - 1]) throw std::runtime_error("primitives not grouped by body");
        return P.upload(pre.data(), pre.size());
      };
      W.cbody_slot = ranges(d->slot_cbody, d->n_slot);
      W.cbody_tri = ranges(d->tri_cbody, d->n_tri);
      W.cbody_edge = ranges(d->edge_cbody, d->n_edge);
      // chunk tables: each body's primitive range split into runs of 32
      auto chunks = [&](const int32_t* owner, int n, int* n_chunk, const int** p0, const int** cb) {
        std::vector<int> cnt(d->n_cbody + 1, 0);
        for (int i = 0; i < n; ++i) cnt[owner[i] + 1]++;
        std::vector<int> first(d->n_cbody + 1, 0);
        for (int b = 0; b < d->n_cbody; ++b) first[b + 1] = first[b] + cnt[b + 1];
        std::vector<int> starts, cbc(d->n_cbody + 1, 0);
        for (int b = 0; b < d->n_cbody; ++b) {
          cbc[b] = (int)starts.size();
          for (int s = first[b]; s < first[b + 1]; s += 32) starts.push_back(s);
        }
        cbc[d->n_cbody] = (int)starts.size();
        starts.push_back(n);
        *n_chunk = (int)starts.size() - 1;
        *p0 = P.upload(starts.data(), starts.size());
        *cb = P.upload(cbc.data(), cbc.size());
      };
      chunks(d->tri_cbody, d->n_tri, &W.n_tchunk, &W.tchunk_p0, &W.cbody_tchunk);
      chunks(d->edge_cbody, d->n_edge, &W.n_echunk, &W.echunk_p0, &W.cbody_echunk);
      W.tchunk_box = P.alloc<double>(6 * (size_t)std::max(W.n_tchunk, 1));
      W.echunk_box = P.alloc<double>(6 * (size_t)std::max(W.n_echunk, 1));
      // LBVHs for the triangles / edges of large bodies (IPC_LBVH=0: chunk walk only)
      {
        const char* lz = getenv("IPC_LBVH");
        bool on = !(lz && lz[0] == '0');
        std::vector<int> tk, tp0, tn, tnode0, tleaf0, ctb(d->n_cbody, -1), ceb(d->n_cbody, -1);
        int nodes = 0, leaves = 0;
        auto add = [&](int kind, const int32_t* owner, int nprim, std::vector<int>& dst) {
          std::vector<int> first(d->n_cbody + 1, 0);
          for (int t = 0; t < nprim; ++t) first[owner[t] + 1]++;
          for (int b = 0; b < d->n_cbody; ++b) first[b + 1] += first[b];
          for (int b = 0; b < d->n_cbody; ++b) {
            int n = first[b + 1] - first[b];
            if (!on || n < LBVH_MIN || n > LBVH_MAX) continue;
            dst[b] = (int)tk.size();
            tk.push_back(kind);
            tp0.push_back(first[b]);
            tn.push_back(n);
            tnode0.push_back(nodes);
            tleaf0.push_back(leaves);
            nodes += n - 1;
            leaves += n;
          }
        };
        add(0, d->tri_cbody, d->n_tri, ctb);
        add(1, d->edge_cbody, d->n_edge, ceb);
        W.n_tree = (int)tk.size();
        if (W.n_tree) {
          W.tree_kind = P.upload(tk.data(), tk.size());
          W.tree_p0 = P.upload(tp0.data(), tp0.size());
          W.tree_n = P.upload(tn.data(), tn.size());
          W.tree_node0 = P.upload(tnode0.data(), tnode0.size());
          W.tree_leaf0 = P.upload(tleaf0.data(), tleaf0.size());
          W.bvh_child = P.alloc<int>(2 * (size_t)nodes);
          W.bvh_parent = P.alloc<int>((size_t)nodes);
          W.bvh_lparent = P.alloc<int>((size_t)leaves);
          W.bvh_prim = P.alloc<int>((size_t)leaves);
          W.bvh_box = P.alloc<double>(6 * (size_t)nodes);
          CK(cudaFuncSetAttribute(k_lbvh_build, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(4 * LBVH_MAX * sizeof(unsigned))));
        }
        ctb.push_back(-1);  // never empty
        ceb.push_back(-1);
        W.cbody_tbvh = P.upload(ctb.data(), ctb.size());
        W.cbody_ebvh = P.upload(ceb.data(), ceb.size());
      }
      int dev = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&w->n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
    W.cons_aff = P.upload(d->cons_aff, d->n_cons);
    W.cons_kappa0 = P.upload(d->cons_kappa0, d->n_cons);
    W.cons_kappa = P.upload(d->cons_kappa0, d->n_cons);
    W.cons_mass = P.upload(d->cons_mass, d->n_cons);
    W.cons_target = P.alloc<double>(12 * (size_t)d->n_cons);
    W.cons_lam = P.alloc<double>(12 * (size_t)d->n_cons);
    W.cons_lastres = P.alloc<double>(d->n_cons);
    W.xw = P.alloc<double>(3 * (size_t)d->n_slot);
    W.xw0 = P.alloc<double>(3 * (size_t)d->n_slot);
    W.dxw = P.alloc<double>(3 * (size_t)d->n_slot);
    w->xwt = P.alloc<double>(3 * (size_t)d->n_slot);
    w->xlo = P.alloc<double>(3 * (size_t)d->n_slot);
    w->xhi = P.alloc<double>(3 * (size_t)d->n_slot);
    w->slot_force = P.alloc<double>(3 * (size_t)d->n_slot);
    w->d_status = P.alloc<int>(4);
    w->e_multi = P.alloc<double>((size_t)ipc_world::LS_M2 * ne);
    CK(cudaMallocHost(&w->h_status, 8 * sizeof(int)));
    w->d_targets = P.alloc<double>(12 * (size_t)d->n_cons);
    w->h_env_slot.assign(d->env_slot, d->env_slot + ne + 1);
    w->h_env_dof.assign(d->env_dof, d->env_dof + ne + 1);
    w->h_env_tri.assign(d->env_tri, d->env_tri + ne + 1);
    w->h_env_edge.assign(d->env_edge, d->env_edge + ne + 1);
    w->h_env_cbody.assign(d->env_cbody, d->env_cbody + ne + 1);
    for (int e = 0; e < ne; ++e) w->max_slots = std::max(w->max_slots, d->env_slot[e + 1] - d->env_slot[e]);
    {
      // CTAs per env in the broad phase: ~BROAD_ITEMS items each
      long long mx = 0;
      for (int e = 0; e < ne; ++e) {
        long long nb = d->env_cbody[e + 1] - d->env_cbody[e];
        long long rows = std::max(d->env_slot[e + 1] - d->env_slot[e], d->env_edge[e + 1] - d->env_edge[e]);
        mx = std::max(mx, rows * nb);
      }
      const char* fz = getenv("IPC_FUSED");
      if (fz) w->fused_on = fz[0] == '1';
      const char* ftz = getenv("IPC_FUSED_TIMERS");
      w->fused_timers_on = ftz && ftz[0] == '1';
      // hand-off at three waves of the per-env kernel (one CTA per SM): a
      // batched iteration costs about three per-env iterations here
      // (measured: 148 / 296 / 444 / 518 envs -> 2.58 / 2.53 / 2.47 / 2.75 ms per step)
      w->tail_envs = 3 * w->n_sm;
      const char* tz = getenv("IPC_TAIL");
      if (tz) w->tail_envs = atoi(tz);
      const char* ez = getenv("IPC_BROAD_ITEMS");
      long long per = ez ? std::max(64LL, atoll(ez)) : ipc_world::BROAD_ITEMS;
      w->bp_z = (int)std::min(64LL, std::max(1LL, (mx + per - 1) / per));
      if (w->bp_z > 1) w->bp_cnt = P.alloc<int>((size_t)ne * 2 * w->bp_z);
    }
    for (int e = 0; e < ne; ++e) {
      w->max_env_dof = std::max(w->max_env_dof, d->env_dof[e + 1] - d->env_dof[e]);
      {
        int nt = d->env_tri[e + 1] - d->env_tri[e], nE = d->env_edge[e + 1] - d->env_edge[e];
        int nbod = d->env_cbody[e + 1] - d->env_cbody[e];
        int chunks_ub = (nt + nE) / 32 + 2 * nbod + 2;
        w->max_env_prims = std::max(w->max_env_prims, d->env_slot[e + 1] - d->env_slot[e] + nt + nE + chunks_ub);
        w->max_env_groups = std::max(w->max_env_groups, d->env_vert[e + 1] - d->env_vert[e] + d->env_aff[e + 1] - d->env_aff[e]);
      }
      if (d->env_cbody[e + 1] - d->env_cbody[e] > 64)
        throw std::runtime_error("more than 64 collision bodies in one environment");
    }
    {
      // batched broad phase with the env's boxes staged in shared memory when
      // they fit comfortably (several CTAs per SM); else the global version
      size_t bsm = sizeof(double) * 6 * (size_t)w->max_env_prims;
      const char* bz = getenv("IPC_BROAD_SM");
      bool on = !(bz && bz[0] == '0');
      if (on && bsm <= 64 * 1024 && w->bp_z == 1) {
        w->broad_smem = std::max(bsm, (size_t)1024);
        CK(cudaFuncSetAttribute(k_broad_sm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w->broad_smem));
      }
    }
    const int DENSE_MAX = DENSE_MAX_N;
    w->sparse = w->max_env_dof > DENSE_MAX;
    if (!w->sparse) {
      // dense system n² + 2n, plus the slot lever arms of the parallel
      // assembly when they fit next to the kernel's static shared memory
      int optin = 0, cur = 0;
      CK(cudaGetDevice(&cur));
      CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cur));
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, k_dense_solve));
      size_t avail = (size_t)optin - fa.sharedSizeBytes;
      size_t base = (size_t)dense_smem_doubles(w->max_env_dof) * sizeof(double);
      if (base > avail) throw std::runtime_error("dense environment system exceeds shared memory");
      w->dense_smem = base;
      CK(cudaFuncSetAttribute(k_dense_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w->dense_smem));
    } else {
      w->setup_sparse(d);
    }
    // env scalar state
    EnvState& S = w->S;
    S.e0 = P.alloc<double>(ne); S.e_new = P.alloc<double>(ne); S.alpha = P.alloc<double>(ne);
    S.alpha_max = P.alloc<double>(ne); S.pnorm = P.alloc<double>(ne); S.prev_pnorm = P.alloc<double>(ne);
    S.gnorm = P.alloc<double>(ne); S.min_s_before = P.alloc<double>(ne); S.min_s = P.alloc<double>(ne);
    S.res = P.alloc<double>(ne);
    S.small_run = P.alloc<int>(ne); S.newton_active = P.alloc<int>(ne); S.ls_active = P.alloc<int>(ne);
    S.al_active = P.alloc<int>(ne); S.ls_failed = P.alloc<int>(ne); S.converged = P.alloc<int>(ne);
    S.newton_iters = P.alloc<int>(ne); S.ccd_calls = P.alloc<int>(ne); S.al_outer = P.alloc<int>(ne);
    S.err = P.alloc<int>(ne); S.any = P.alloc<int>(1);
    w->enable = P.alloc<int>(ne);
    w->ok = P.alloc<int>(ne); w->al_flag = S.al_active; w->accepted = P.alloc<int>(ne);
    w->ls_count = P.alloc<int>(ne); w->d_count = P.alloc<int>(1);
    w->env_order = P.alloc<int>(ne);
    {
      std::vector<int> iota(ne);
      for (int e = 0; e < ne; ++e) iota[e] = e;
      CK(cudaMemcpy(w->env_order, iota.data(), sizeof(int) * ne, cudaMemcpyHostToDevice));
    }
    w->env_alpha = P.alloc<double>(ne);
    CK(cudaMallocHost(&w->h_count, sizeof(int)));
    // capacities: exhaustive for small envs, bounded for large ones
    std::vector<long long> ptc(ne), eec(ne);
    for (int e = 0; e < ne; ++e) {
      long long nv = d->env_slot[e + 1] - d->env_slot[e], nt = d->env_tri[e + 1] - d->env_tri[e];
      long long nE = d->env_edge[e + 1] - d->env_edge[e];
      ptc[e] = d->env_pairs[e] ? std::min(nv * nt, std::max(4096LL, 16 * (nv + nt))) : 0;
      eec[e] = d->env_pairs[e] ? std::min(nE * nE, std::max(4096LL, 16 * nE)) : 0;
    }
    w->alloc_cands(w->dcd, ptc, eec);
    w->alloc_cands(w->sweep, ptc, eec);
    w->alloc_cands(w->ss, ptc, eec);
    w->ss.c.overflow = w->sweep.c.overflow;  // one sticky flag: the step checks dcd and sweep
    w->ss_valid = P.alloc<int>(ne);
    w->ss_rebuild = P.alloc<int>(ne);
    CK(cudaMemset(w->ss_valid, 0, sizeof(int) * ne));
    w->bb_lo = P.alloc<double>(3 * (size_t)std::max(d->n_slot, 1));
    w->bb_hi = P.alloc<double>(3 * (size_t)std::max(d->n_slot, 1));
    {
      const char* sp = getenv("IPC_SS_PAD");
      if (sp) w->ss_pad = atof(sp);
    }
    w->alloc_pairbufs(w->pb_dcd, w->dcd, true);
    w->alloc_pairbufs(w->pb_sweep, w->sweep, false);
    w->alloc_lags();
    w->body_val = P.alloc<double>(d->n_aff);
    w->D.body_g = P.alloc<double>(12 * (size_t)d->n_aff);
    w->D.body_h = P.alloc<double>(144 * (size_t)d->n_aff);
    w->tet_val = P.alloc<double>(d->n_tet);
    w->D.tet_g = P.alloc<double>(12 * (size_t)d->n_tet);
    w->D.tet_h = P.alloc<double>(PK * (size_t)d->n_tet);
    CK(cudaStreamCreateWithFlags(&w->st, cudaStreamNonBlocking));
    for (int i = 0; i < 3; ++i) CK(cudaStreamCreateWithFlags(&w->side[i], cudaStreamNonBlocking));
    for (int i = 0; i < 4; ++i) CK(cudaEventCreateWithFlags(&w->fj[i], cudaEventDisableTiming));
    if (w->fused_timers_on && !w->sparse) w->fused_setup();  // timer block for the batched solve too
    g_pdl = getenv("IPC_PDL") == nullptr || getenv("IPC_PDL")[0] != '0';
    CK(cudaDeviceSynchronize());
    *out = w;
    return 0;
  } catch (const std::exception& ex) {
    delete w;
    return set_err("%s", ex.what());
  }
}

int ipc_world_destroy(ipc_world* w) {
  if (w) {
    cudaStreamSynchronize(w->st);
    if (g_prof == &w->prof) g_prof = nullptr;
    for (auto e : w->marks) cudaEventDestroy(e);
    if (w->st) cudaStreamDestroy(w->st);
    delete w;
  }
  return 0;
}

int ipc_world_step(ipc_world* w, const ipc_step_config* cfg, const double* targets, ipc_step_report* rep) {
  return ipc_world_step_ex(w, cfg, targets, nullptr, rep);
}

static int step_impl(ipc_world* w, const ipc_step_config* cfg, const double* targets, int sched_k,
                     const uint8_t* enable, ipc_step_report* rep);

int ipc_world_step_ex(ipc_world* w, const ipc_step_config* cfg, const double* targets, const uint8_t* enable,
                      ipc_step_report* rep) {
  return step_impl(w, cfg, targets, -1, enable, rep);
}

int ipc_world_upload_schedule(ipc_world* w, const double* targets, int n_steps) {
  GUARD({
    if (w->sched) w->pool.free_one(w->sched);
    w->sched = w->pool.upload(targets, 12 * (size_t)w->W.n_cons * n_steps);
    w->sched_steps = n_steps;
  })
}

int ipc_world_step_scheduled(ipc_world* w, const ipc_step_config* cfg, int k, const uint8_t* enable,
                             ipc_step_report* rep) {
  if (k < 0 || k >= w->sched_steps) return set_err("schedule index %d out of range", k);
  return step_impl(w, cfg, nullptr, k, enable, rep);
}

static void step_core(ipc_world* w, const ipc_step_config* cfg, const double* targets, int sched_k,
                      const uint8_t* enable, ipc_step_report* rep) {
  {
    g_prof = &w->prof;
    World& W = w->W;
    EnvState& S = w->S;
    cudaStream_t st = w->st;
    int ne = w->n_env;
    double h = cfg->h;
    if (targets && W.n_cons) {
      CK(cudaMemcpyAsync(w->d_targets, targets, 12 * sizeof(double) * W.n_cons, cudaMemcpyHostToDevice, st));
      w->targets_set = true;
    } else if (sched_k >= 0 && W.n_cons) {
      CK(cudaMemcpyAsync(w->d_targets, w->sched + 12 * (size_t)W.n_cons * sched_k, 12 * sizeof(double) * W.n_cons,
                         cudaMemcpyDeviceToDevice, st));
      w->targets_set = true;
    }
    IPC_LAUNCH(K_MISC, st, k_step_begin, nblk(ne, 128), 128, 0, ne, S);
    CK(cudaMemcpyAsync(W.x_prev, W.x, sizeof(double) * W.n_dof, cudaMemcpyDeviceToDevice, st));
    w->world_pos(W.x, W.xw0);
    if (enable) {
      std::vector<int> en(ne);
      for (int e = 0; e < ne; ++e) en[e] = enable[e] ? 1 : 0;
      CK(cudaMemcpyAsync(w->enable, en.data(), 4 * ne, cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
    } else {
      IPC_LAUNCH(K_MISC, st, k_fill_int, nblk(ne, 128), 128, 0, ne, w->enable, 1);
    }
    if (!(w->use_fused() && w->step_fused(*cfg))) {
    IPC_LAUNCH(K_MISC, st, k_copy_int, nblk(ne, 128), 128, 0, ne, w->enable, w->ok);
    w->broad(w->dcd, w->pb_dcd, true, W.xw0, W.xw0, w->ok);
    // feasibility of the incoming state (ref solver.py:372-385)
    w->pairs(W.xw0, w->dcd, w->pb_dcd, 0, nullptr, K_PAIRS_V);
    int max_slots = 0;
    for (int e = 0; e < ne; ++e) max_slots = std::max(max_slots, w->h_env_slot[e + 1] - w->h_env_slot[e]);
    IPC_LAUNCH(K_GROUND, st, k_ground, dim3(nblk(max_slots, 128), ne), 128, 0, W, W.xw0, w->dcd.c, 0, w->ok, w->pb_dcd.gnd_val,
                                                             nullptr, nullptr, nullptr);
    IPC_LAUNCH(K_MISC, st, k_start_check, ne, 128, 0, W, S, w->dcd.c, w->pb_dcd.pt_val, w->pb_dcd.ee_val, w->pb_dcd.gnd_val, w->ok);
    // predictor
    IPC_LAUNCH(K_MISC, st, k_predictor, nblk(W.n_dof, 256), 256, 0, W, h);
    IPC_LAUNCH(K_MISC, st, k_predictor_forces, nblk(std::max(W.n_vert, W.n_aff), 128), 128, 0, W, h);
    // fresh AL cycle per step (ref solver.py:394-400)
    if (W.n_cons) {
      if (!w->targets_set) throw std::runtime_error("kinematic constraint targets were never set");
      IPC_LAUNCH(K_MISC, st, k_cons_reset, nblk(W.n_cons, 128), 128, 0, W, w->d_targets);
    }
    int fp_iters = std::max(cfg->friction_fixed_point_iters, 1);
    for (int fp = 0; fp < fp_iters; ++fp) {
      // lags frozen at the anchor (x_prev first, then the current iterate)
      if (w->lags_stale) {
        w->alloc_lags();
        w->lags_stale = false;
      }
      if (fp == 0) {
        IPC_LAUNCH(K_LAGS, st, k_lags, ne, BP_THREADS, 0, W, W.xw0, w->dcd.c, w->L, w->ok, w->env_order);
        IPC_LAUNCH(K_MISC, st, k_prefix, 1, 1024, 0, ne, w->L.n, w->ok, w->L.pre);
        IPC_LAUNCH(K_MISC, st, k_prefix, 1, 1024, 0, ne, w->L.g_n, w->ok, w->L.g_pre);
      } else {
        w->world_pos(W.x, W.xw);
        w->broad(w->dcd, w->pb_dcd, true, W.xw, W.xw, w->ok);
        IPC_LAUNCH(K_LAGS, st, k_lags, ne, BP_THREADS, 0, W, W.xw, w->dcd.c, w->L, w->ok, w->env_order);
        IPC_LAUNCH(K_MISC, st, k_prefix, 1, 1024, 0, ne, w->L.n, w->ok, w->L.pre);
        IPC_LAUNCH(K_MISC, st, k_prefix, 1, 1024, 0, ne, w->L.g_n, w->ok, w->L.g_pre);
      }
      IPC_LAUNCH(K_MISC, st, k_copy_int, nblk(ne, 128), 128, 0, ne, w->ok, S.al_active);
      for (int outer = 0; outer < cfg->al_max_outer; ++outer) {
        if (w->count(S.al_active) == 0) break;
        w->newton_solve(*cfg);
        IPC_LAUNCH(K_MISC, st, k_al_update, nblk(ne, 128), 128, 0, W, S, outer);
      }
      IPC_LAUNCH(K_MISC, st, k_and_not, nblk(ne, 128), 128, 0, ne, w->ok, S.ls_failed);
    }
    // post-step distance and barrier adaptation (ref solver.py:440-450)
    IPC_LAUNCH(K_MISC, st, k_copy_int, nblk(ne, 128), 128, 0, ne, w->enable, w->ok);
    IPC_LAUNCH(K_MISC, st, k_and_not, nblk(ne, 128), 128, 0, ne, w->ok, S.err);
    w->world_pos(W.x, W.xw);
    w->broad(w->dcd, w->pb_dcd, true, W.xw, W.xw, w->ok);
    IPC_LAUNCH(K_MISC, st, k_fill, nblk(ne, 128), 128, 0, ne, S.min_s, INFINITY);
    w->pairs(W.xw, w->dcd, w->pb_dcd, 0, S.min_s, K_PAIRS_V);
    IPC_LAUNCH(K_GROUND, st, k_ground, dim3(nblk(max_slots, 128), ne), 128, 0, W, W.xw, w->dcd.c, 0, w->ok, w->pb_dcd.gnd_val,
                                                             nullptr, nullptr, S.min_s);
    IPC_LAUNCH(K_MISC, st, k_kappa_adapt, nblk(ne, 128), 128, 0, W, S, w->ok);
    IPC_LAUNCH(K_MISC, st, k_finalize, nblk(W.n_dof, 256), 256, 0, W, h, w->ok);
    }
    CK(cudaGetLastError());
    if (rep) {
      w->read_reports(rep);
    } else {
      CK(cudaStreamSynchronize(st));
    }
  }
}

void ipc_world::read_reports(ipc_step_report* rep) {
  {
    {
      int ne = n_env;
      std::vector<int> it(ne), cc(ne), cv(ne), lf(ne), ao(ne), er(ne);
      std::vector<double> gn(ne), mb(ne), ma(ne), kp(ne);
      CK(cudaMemcpyAsync(it.data(), S.newton_iters, 4 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(cc.data(), S.ccd_calls, 4 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(cv.data(), S.converged, 4 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(lf.data(), S.ls_failed, 4 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(ao.data(), S.al_outer, 4 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(er.data(), S.err, 4 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(gn.data(), S.gnorm, 8 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(mb.data(), S.min_s_before, 8 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(ma.data(), S.min_s, 8 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(kp.data(), W.env_kappa, 8 * ne, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int e = 0; e < ne; ++e) {
        rep[e].newton_iters = it[e];
        rep[e].ccd_invocations = cc[e];
        rep[e].converged = cv[e];
        rep[e].line_search_failed = lf[e];
        rep[e].al_outer = ao[e];
        rep[e].error = er[e];
        rep[e].final_grad_norm = gn[e];
        rep[e].min_dist_before = std::isinf(mb[e]) ? INFINITY : std::sqrt(mb[e]);
        rep[e].min_dist_after = ma[e];
        rep[e].kappa = kp[e];
      }
    }
  }
}

static int step_impl(ipc_world* w, const ipc_step_config* cfg, const double* targets, int sched_k,
                     const uint8_t* enable, ipc_step_report* rep) {
  GUARD({
    g_prof = &w->prof;
    for (int attempt = 0;; ++attempt) {
      try {
        CK(cudaMemsetAsync(w->dcd.c.overflow, 0, sizeof(int), w->st));
        CK(cudaMemsetAsync(w->sweep.c.overflow, 0, sizeof(int), w->st));
        step_core(w, cfg, targets, sched_k, enable, rep);
        break;
      } catch (const OverflowRetry&) {
        if (attempt >= 64) throw std::runtime_error("candidate capacity overflow persists");
        // replay the step from x_prev with larger candidate capacities
        CK(cudaMemcpyAsync(w->W.x, w->W.x_prev, sizeof(double) * w->W.n_dof, cudaMemcpyDeviceToDevice, w->st));
        w->grow_overflowed();
      }
    }
  })
}

int ipc_world_run_scheduled(ipc_world* w, const ipc_step_config* cfg, int k0, int k1, ipc_step_report* rep) {
  GUARD({
    g_prof = &w->prof;
    if (!w->sched || k0 < 0 || k1 > w->sched_steps || k0 > k1)
      throw std::runtime_error("run_scheduled: steps outside the uploaded schedule");
    if (w->sparse || !w->fused_setup()) throw std::runtime_error("run_scheduled: needs a dense world");
    World& W = w->W;
    int ne = w->n_env;
    double* x0 = w->pool.alloc<double>(W.n_dof);
    CK(cudaMemcpyAsync(x0, W.x, sizeof(double) * W.n_dof, cudaMemcpyDeviceToDevice, w->st));
    for (int attempt = 0;; ++attempt) {
      if (w->lags_stale) {
        w->alloc_lags();
        w->lags_stale = false;
      }
      CK(cudaMemsetAsync(w->dcd.c.overflow, 0, sizeof(int), w->st));
      CK(cudaMemsetAsync(w->sweep.c.overflow, 0, sizeof(int), w->st));
      CK(cudaMemcpyAsync(w->v_save, W.v, sizeof(double) * W.n_dof, cudaMemcpyDeviceToDevice, w->st));
      CK(cudaMemcpyAsync(w->kappa_save, W.env_kappa, sizeof(double) * ne, cudaMemcpyDeviceToDevice, w->st));
      IPC_LAUNCH(K_MISC, w->st, k_fill_int, nblk(ne, 128), 128, 0, ne, w->enable, 1);
      CK(cudaMemsetAsync(w->fq, 0, sizeof(int), w->st));
      FusedArgs A = w->fused_args(*cfg);
      IPC_LAUNCH(K_FUSED, w->st, k_env_steps, w->fused_blocks, 256, w->fused_smem, A, w->sched, W.n_cons, k0, k1);
      CK(cudaMemcpyAsync(w->h_status, w->dcd.c.overflow, sizeof(int), cudaMemcpyDeviceToHost, w->st));
      CK(cudaMemcpyAsync(w->h_status + 1, w->sweep.c.overflow, sizeof(int), cudaMemcpyDeviceToHost, w->st));
      CK(cudaStreamSynchronize(w->st));
      if (!w->h_status[0] && !w->h_status[1]) break;
      if (attempt >= 64) throw std::runtime_error("candidate capacity overflow persists");
      // replay the whole range from its start with larger capacities
      CK(cudaMemcpyAsync(W.x, x0, sizeof(double) * W.n_dof, cudaMemcpyDeviceToDevice, w->st));
      CK(cudaMemcpyAsync(W.v, w->v_save, sizeof(double) * W.n_dof, cudaMemcpyDeviceToDevice, w->st));
      CK(cudaMemcpyAsync(W.env_kappa, w->kappa_save, sizeof(double) * ne, cudaMemcpyDeviceToDevice, w->st));
      w->grow_overflowed();
    }
    w->pool.free_one(x0);
    if (rep) w->read_reports(rep);
  })
}

int ipc_set_device(int device) {
  GUARD({ CK(cudaSetDevice(device)); })
}

int ipc_world_profile(ipc_world* w, int on, uint32_t kernel_mask) {
  GUARD({
    CK(cudaStreamSynchronize(w->st));
    w->prof.resolve();
    w->prof.on = on != 0;
    w->prof.mask = kernel_mask;
    for (int k = 0; k < NKID; ++k) { w->prof.ms[k] = 0.0; w->prof.cnt[k] = 0; }
    w->prof.launches = 0;
  })
}

int ipc_world_profile_read(ipc_world* w, double* ms, int64_t* count, int64_t* launches) {
  GUARD({
    CK(cudaStreamSynchronize(w->st));
    w->prof.resolve();
    for (int k = 0; k < NKID; ++k) {
      if (ms) ms[k] = w->prof.ms[k];
      if (count) count[k] = w->prof.cnt[k];
    }
    if (launches) *launches = w->prof.launches;
  })
}

int ipc_world_stats(ipc_world* w, int64_t* out) {
  GUARD({
    out[0] = w->stat_iters;
    out[1] = w->stat_ls_rounds;
    out[2] = w->stat_syncs;
    int pit[3] = {0, 0, 0};
    if (w->d_nlive) {
      CK(cudaStreamSynchronize(w->st));
      CK(cudaMemcpy(pit, w->d_nlive, sizeof(pit), cudaMemcpyDeviceToHost));
    }
    out[3] = pit[2];
    long long fs[2] = {0, 0};
    if (w->d_fstat) CK(cudaMemcpy(fs, w->d_fstat, sizeof(fs), cudaMemcpyDeviceToHost));
    out[4] = fs[0];
    out[5] = fs[1];
  })
}

int ipc_world_set_fused(ipc_world* w, int on) {
  GUARD({
    w->fused_on = on != 0;
    w->fused_blocks = 0;
  })
}

int ipc_world_set_fused_timers(ipc_world* w, int on) {
  GUARD({ w->fused_timers_on = on != 0; })
}

int ipc_device_clock_khz(int32_t* khz) {
  GUARD({
    int dev = 0, v = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, dev));
    *khz = v;
  })
}

int ipc_world_fused_timers(ipc_world* w, int64_t* out, int n) {
  GUARD({
    for (int k = 0; k < n; ++k) out[k] = 0;
    if (w->d_fstat) {
      CK(cudaStreamSynchronize(w->st));
      CK(cudaMemcpy(out, w->d_fstat + 2, sizeof(long long) * std::min(n, (int)FT_TOTAL), cudaMemcpyDeviceToHost));
    }
  })
}

int ipc_world_flush_l2(ipc_world* w, int64_t bytes) {
  GUARD({
    if (!w->flush_buf) w->flush_buf = w->pool.alloc<double>((size_t)bytes / 8);
    CK(cudaMemsetAsync(w->flush_buf, 0xA5, (size_t)bytes, w->st));
  })
}

int ipc_world_mark(ipc_world* w, int slot) {
  GUARD({
    while ((int)w->marks.size() <= slot) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      w->marks.push_back(e);
    }
    CK(cudaEventRecord(w->marks[slot], w->st));
  })
}

int ipc_world_elapsed(ipc_world* w, int a, int b, double* ms) {
  GUARD({
    CK(cudaEventSynchronize(w->marks[b]));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, w->marks[a], w->marks[b]));
    *ms = t;
  })
}

int ipc_world_sync(ipc_world* w) {
  GUARD({ CK(cudaStreamSynchronize(w->st)); })
}

int ipc_world_get_state(ipc_world* w, double* x, double* v) {
  GUARD({
    g_prof = &w->prof;
    if (x) CK(cudaMemcpyAsync(x, w->W.x, sizeof(double) * w->W.n_dof, cudaMemcpyDeviceToHost, w->st));
    if (v) CK(cudaMemcpyAsync(v, w->W.v, sizeof(double) * w->W.n_dof, cudaMemcpyDeviceToHost, w->st));
    CK(cudaStreamSynchronize(w->st));
  })
}

int ipc_world_set_state(ipc_world* w, const double* x, const double* v) {
  GUARD({
    g_prof = &w->prof;
    if (x) CK(cudaMemcpyAsync(w->W.x, x, sizeof(double) * w->W.n_dof, cudaMemcpyHostToDevice, w->st));
    if (v) CK(cudaMemcpyAsync(w->W.v, v, sizeof(double) * w->W.n_dof, cudaMemcpyHostToDevice, w->st));
    CK(cudaStreamSynchronize(w->st));
  })
}

int ipc_world_state_device(ipc_world* w, double** x, double** v) {
  if (x) *x = w->W.x;
  if (v) *v = w->W.v;
  return 0;
}

int ipc_world_get_kappa(ipc_world* w, double* kappa) {
  GUARD({
    g_prof = &w->prof;
    CK(cudaMemcpy(kappa, w->W.env_kappa, sizeof(double) * w->n_env, cudaMemcpyDeviceToHost));
  })
}

int ipc_world_set_kappa(ipc_world* w, const double* kappa) {
  GUARD({
    g_prof = &w->prof;
    CK(cudaMemcpy(w->W.env_kappa, kappa, sizeof(double) * w->n_env, cudaMemcpyHostToDevice));
  })
}

int ipc_world_get_constraints(ipc_world* w, double* lam, double* kappa) {
  GUARD({
    g_prof = &w->prof;
    if (lam) CK(cudaMemcpy(lam, w->W.cons_lam, sizeof(double) * 12 * w->W.n_cons, cudaMemcpyDeviceToHost));
    if (kappa) CK(cudaMemcpy(kappa, w->W.cons_kappa, sizeof(double) * w->W.n_cons, cudaMemcpyDeviceToHost));
  })
}

// DCD candidates + contact derivatives at the current state (for sensing)
static void contact_at_current(ipc_world* w) {
  World& W = w->W;
  int ne = w->n_env;
  w->world_pos(W.x, W.xw);
  w->broad(w->dcd, w->pb_dcd, true, W.xw, W.xw, nullptr);
  w->pairs(W.xw, w->dcd, w->pb_dcd, 1, nullptr, K_SENSE);
  int max_slots = 0;
  for (int e = 0; e < ne; ++e) max_slots = std::max(max_slots, w->h_env_slot[e + 1] - w->h_env_slot[e]);
  IPC_LAUNCH(K_GROUND, w->st, k_ground, dim3(nblk(max_slots, 128), ne), 128, 0, W, W.xw, w->dcd.c, 1, nullptr, w->pb_dcd.gnd_val,
                                                              w->pb_dcd.gnd_gy, w->pb_dcd.gnd_hyy, nullptr);
  IPC_LAUNCH(K_SENSE, w->st, k_slot_forces, nblk(W.n_slot, 128), 128, 0, W, w->dcd.c, w->pb_dcd.pt_g, w->pb_dcd.pt_act,
                                                        w->pb_dcd.ee_g, w->pb_dcd.ee_act, w->pb_dcd.gnd_gy, 1.0,
                                                        w->slot_force);
  CK(cudaGetLastError());
}

int ipc_world_slot_forces(ipc_world* w, double h, double* out) {
  GUARD({
    g_prof = &w->prof;
    contact_at_current(w);
    std::vector<double> f(3 * (size_t)w->W.n_slot);
    CK(cudaMemcpyAsync(f.data(), w->slot_force, sizeof(double) * f.size(), cudaMemcpyDeviceToHost, w->st));
    CK(cudaStreamSynchronize(w->st));
    double ih = 1.0 / (h * h);
    for (size_t i = 0; i < f.size(); ++i) out[i] = f[i] * ih;  // slot_force holds -g (h = 1 pass)
  })
}

int ipc_world_group_forces(ipc_world* w, double h, const uint64_t* groups, int ng, double* out) {
  GUARD({
    g_prof = &w->prof;
    contact_at_current(w);
    size_t n = (size_t)w->n_env * ng;
    unsigned long long* dg = w->pool.upload((const unsigned long long*)groups, n);
    double* dout = w->pool.alloc<double>(3 * n);
    IPC_LAUNCH(K_SENSE, w->st, k_group_forces, nblk(n, 128), 128, 0, w->W, w->slot_force, dg, ng, dout);
    CK(cudaMemcpyAsync(out, dout, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, w->st));
    CK(cudaStreamSynchronize(w->st));
    double ih = 1.0 / (h * h);
    for (size_t i = 0; i < 3 * n; ++i) out[i] *= ih;
    w->pool.free_one(dg);
    w->pool.free_one(dout);
  })
}

int ipc_world_candidates(ipc_world* w, int env, int which, int32_t* out, int64_t cap, int64_t* n) {
  GUARD({
    g_prof = &w->prof;
    World& W = w->W;
    w->world_pos(W.x, W.xw);
    w->broad(w->dcd, w->pb_dcd, true, W.xw, W.xw, nullptr);
    int cnt = 0;
    const int* src = which == 0 ? w->dcd.c.n_pt : (which == 1 ? w->dcd.c.n_ee : w->dcd.c.n_gnd);
    CK(cudaMemcpy(&cnt, src + env, sizeof(int), cudaMemcpyDeviceToHost));
    *n = cnt;
    long long m = std::min<long long>(cnt, cap);
    if (which == 0) {
      long long off = 0;
      CK(cudaMemcpy(&off, w->dcd.d_pt_off + env, sizeof(long long), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(out, w->dcd.c.pt + off, 8 * m, cudaMemcpyDeviceToHost));
    } else if (which == 1) {
      long long off = 0;
      CK(cudaMemcpy(&off, w->dcd.d_ee_off + env, sizeof(long long), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(out, w->dcd.c.ee + off, 8 * m, cudaMemcpyDeviceToHost));
    } else {
      CK(cudaMemcpy(out, w->dcd.c.gnd + w->h_env_slot[env], 4 * m, cudaMemcpyDeviceToHost));
    }
  })
}

int ipc_world_min_distance(ipc_world* w, double* out) {
  GUARD({
    g_prof = &w->prof;
    World& W = w->W;
    int ne = w->n_env;
    w->world_pos(W.x, W.xw);
    w->broad(w->dcd, w->pb_dcd, true, W.xw, W.xw, nullptr);
    double* d = w->S.min_s_before;  // scratch
    IPC_LAUNCH(K_MISC, w->st, k_fill, nblk(ne, 128), 128, 0, ne, d, INFINITY);
    w->pairs(W.xw, w->dcd, w->pb_dcd, 0, d, K_PAIRS_V);
    int max_slots = 0;
    for (int e = 0; e < ne; ++e) max_slots = std::max(max_slots, w->h_env_slot[e + 1] - w->h_env_slot[e]);
    IPC_LAUNCH(K_GROUND, w->st, k_ground, dim3(nblk(max_slots, 128), ne), 128, 0, W, W.xw, w->dcd.c, 0, nullptr, w->pb_dcd.gnd_val,
                                                                nullptr, nullptr, d);
    std::vector<double> s(ne);
    CK(cudaMemcpyAsync(s.data(), d, 8 * ne, cudaMemcpyDeviceToHost, w->st));
    CK(cudaStreamSynchronize(w->st));
    for (int e = 0; e < ne; ++e) out[e] = std::isinf(s[e]) ? INFINITY : std::sqrt(s[e]);
  })
}

int ipc_world_group_distance(ipc_world* w, const uint64_t* ga, const uint64_t* gb, double* out) {
  GUARD({
    g_prof = &w->prof;
    World& W = w->W;
    int ne = w->n_env;
    w->world_pos(W.x, W.xw);
    w->broad(w->dcd, w->pb_dcd, true, W.xw, W.xw, nullptr);
    unsigned long long* da = w->pool.upload((const unsigned long long*)ga, ne);
    unsigned long long* db = w->pool.upload((const unsigned long long*)gb, ne);
    double* dout = w->pool.alloc<double>(ne);
    IPC_LAUNCH(K_SENSE, w->st, k_group_distance, ne, 256, 0, W, w->dcd.c, W.xw, da, db, dout);
    CK(cudaMemcpyAsync(out, dout, 8 * ne, cudaMemcpyDeviceToHost, w->st));
    CK(cudaStreamSynchronize(w->st));
    w->pool.free_one(da);
    w->pool.free_one(db);
    w->pool.free_one(dout);
  })
}

int ipc_world_ground_distance(ipc_world* w, const uint64_t* g, double* out) {
  GUARD({
    g_prof = &w->prof;
    World& W = w->W;
    int ne = w->n_env;
    w->world_pos(W.x, W.xw);
    unsigned long long* dg = w->pool.upload((const unsigned long long*)g, ne);
    double* dout = w->pool.alloc<double>(ne);
    IPC_LAUNCH(K_SENSE, w->st, k_ground_distance, nblk(ne, 128), 128, 0, W, W.xw, dg, dout);
    CK(cudaMemcpyAsync(out, dout, 8 * ne, cudaMemcpyDeviceToHost, w->st));
    CK(cudaStreamSynchronize(w->st));
    w->pool.free_one(dg);
    w->pool.free_one(dout);
  })
}

}  // extern "C"

// ---------------------------------------------------------------------------
// kernel-level entry points for parity tests
// ---------------------------------------------------------------------------
namespace {
__global__ void k_t_dist(int kind, long long n, const double* st, int* region, double* s, double* g, double* h) {
  ipc_pdl_wait();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 X[4];
  for (int a = 0; a < 4; ++a) X[a] = ld3(st + 12 * i + 3 * a);
  bool par;
  int r = kind == 0 ? pt_region(X[0], X[1], X[2], X[3]) : ee_region(X[0], X[1], X[2], X[3], &par);
  double G[12], H[144];
  for (int k = 0; k < 12; ++k) G[k] = 0.0;
  for (int k = 0; k < 144; ++k) H[k] = 0.0;
  int mask;
  s[i] = dist2_derivs(kind == 0, r, X, G, H, &mask);
  region[i] = r;
  for (int k = 0; k < 12; ++k) g[12 * i + k] = G[k];
  for (int k = 0; k < 144; ++k) h[144 * i + k] = H[k];
}
__global__ void k_t_ccd(int kind, long long n, const double* px, const double* pdx, double cons, double* a) {
  ipc_pdl_wait();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 X[4], D[4];
  for (int k = 0; k < 4; ++k) {
    X[k] = ld3(px + 12 * i + 3 * k);
    D[k] = ld3(pdx + 12 * i + 3 * k);
  }
  a[i] = pair_ccd_alpha(kind, X, D, cons);
}
template <int N>
__global__ void k_t_psd(long long n, double* m) {
  ipc_pdl_wait();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) psd_project<N>(m + (long long)N * N * i, N);
}
__global__ void k_t_elastic(int model, long long n, const double* F, double mu, double lam, double* psi, double* P,
                            double* H9) {
  ipc_pdl_wait();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  M3 f;
  for (int k = 0; k < 9; ++k) f.m[k] = F[9 * i + k];
  double ps, p[9], h[81];
  if (!psi_derivs(model, f, mu, lam, &ps, p, h)) {
    psi[i] = INFINITY;
    return;
  }
  psi[i] = ps;
  for (int k = 0; k < 9; ++k) P[9 * i + k] = p[k];
  for (int k = 0; k < 81; ++k) H9[81 * i + k] = h[k];
}

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  explicit DBuf(size_t n_) : n(n_) { CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
  DBuf(const T* h, size_t n_) : DBuf(n_) {
    if (n) CK(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void get(T* h) const {
    if (n) CK(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost));
  }
  ~DBuf() { cudaFree(p); }
};
}  // namespace

extern "C" {
int ipc_dist2_derivs(int kind, int64_t n, const double* st, int32_t* region, double* s, double* g, double* h) {
  GUARD({
    DBuf<double> dst(st, 12 * n), ds(n), dg(12 * n), dh(144 * n);
    DBuf<int> dr(n);
    k_t_dist<<<nblk(n, 64), 64>>>(kind, n, dst.p, dr.p, ds.p, dg.p, dh.p);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    dr.get(region); ds.get(s); dg.get(g); dh.get(h);
  })
}
int ipc_ccd_pairs(int kind, int64_t n, const double* px, const double* pdx, double cons, double* alpha) {
  GUARD({
    DBuf<double> a(px, 12 * n), b(pdx, 12 * n), o(n);
    k_t_ccd<<<nblk(n, 64), 64>>>(kind, n, a.p, b.p, cons, o.p);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    o.get(alpha);
  })
}
int ipc_psd_project(int dim, int64_t n, double* mats) {
  GUARD({
    DBuf<double> m(mats, (size_t)dim * dim * n);
    if (dim == 6) k_t_psd<6><<<nblk(n, 64), 64>>>(n, m.p);
    else if (dim == 9) k_t_psd<9><<<nblk(n, 64), 64>>>(n, m.p);
    else if (dim == 12) k_t_psd<12><<<nblk(n, 64), 64>>>(n, m.p);
    else throw std::runtime_error("psd_project: dim must be 6, 9 or 12");
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    m.get(mats);
  })
}
int ipc_elastic_eval(int model, int64_t n, const double* F, double mu, double lam, double* psi, double* P, double* H9) {
  GUARD({
    DBuf<double> f(F, 9 * n), ps(n), p(9 * n), h(81 * n);
    k_t_elastic<<<nblk(n, 64), 64>>>(model, n, f.p, mu, lam, ps.p, p.p, h.p);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    ps.get(psi); p.get(P); h.get(H9);
  })
}
}  // extern "C"
