// Linear BVH (Karras 2012) over the triangles / edges of large collision
// bodies: the third culling level of the global broad phase (kernels.cuh
// for_item_prims), replacing the linear walk over a body's 32-primitive
// chunks with an O(log n) traversal. The reference culls through a BVH with a
// rebuild/refit cache (ref geometry/bvh.py:11 Bvh, broadphase.py:74
// BroadPhaseCache); here every broad-phase call rebuilds each tree on the
// device from the query boxes it is called with (one CTA per tree):
//
//   1. 30-bit Morton codes of the primitive box centroids in the body box;
//   2. a stable LSD radix sort of (code, primitive) in shared memory, 4-bit
//      digits, warp-level multisplit (__match_any_sync ranks, per-warp digit
//      histograms, one block scan per pass);
//   3. Karras' internal-node construction (one thread per node: direction by
//      the longest common prefix, range end by exponential + binary search,
//      split by binary search; equal codes are disambiguated by the leaf index);
//   4. bottom-up refit with per-node arrival counters in shared memory.
//
// Traversal tests node boxes with the pair margin: a node box is the union of
// its primitives' boxes, so a primitive that passes the exact prim-level test
// passes every ancestor's test — the visited set equals the chunk walk's, and
// hits are replayed in increasing primitive index, keeping the reference's
// lexicographic candidate order.
#pragma once
#include "ipc_math.cuh"
#include "world.cuh"

namespace ipc {

// query box vs a box inflated by margin, the rounding of kernels.cuh box_hit:
// monotone, so a node box containing a primitive box passes whenever the
// primitive does
__device__ __forceinline__ bool lbvh_box_hit(const double* qlo, const double* qhi, const double* plo,
                                             const double* phi, double margin) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double pmin = __dsub_rn(plo[c], margin), pmax = __dadd_rn(phi[c], margin);
    if (!(qlo[c] <= pmax && qhi[c] >= pmin)) return false;
  }
  return true;
}

constexpr int LBVH_MIN = 256;    // bodies with at least this many primitives get a tree
constexpr int LBVH_MAX = 4096;   // shared-memory sort capacity (larger bodies keep the chunk walk)
constexpr int LBVH_THREADS = 256;
constexpr int LBVH_HITS = 32;    // hits collected per traversal before falling back to the chunk walk

// primitive box (lo/hi of its slots' query boxes), the same arithmetic as prim_hit
__device__ __forceinline__ void lbvh_prim_box(const World& W, int kind, int t, const double* __restrict__ lo,
                                              const double* __restrict__ hi, double* b) {
  if (kind == 0) {
    int3 v = W.tri_v[t];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      b[c] = fmin(fmin(lo[3 * v.x + c], lo[3 * v.y + c]), lo[3 * v.z + c]);
      b[3 + c] = fmax(fmax(hi[3 * v.x + c], hi[3 * v.y + c]), hi[3 * v.z + c]);
    }
  } else {
    int2 v = W.edge_v[t];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      b[c] = fmin(lo[3 * v.x + c], lo[3 * v.y + c]);
      b[3 + c] = fmax(hi[3 * v.x + c], hi[3 * v.y + c]);
    }
  }
}

__device__ __forceinline__ unsigned lbvh_expand10(unsigned v) {  // 10 bits -> every third bit
  v = (v * 0x00010001u) & 0xFF0000FFu;
  v = (v * 0x00000101u) & 0x0F00F00Fu;
  v = (v * 0x00000011u) & 0xC30C30C3u;
  v = (v * 0x00000005u) & 0x49249249u;
  return v;
}

// longest common prefix of sorted codes i, j (index tie-break for equal codes); -1 out of range
__device__ __forceinline__ int lbvh_delta(const unsigned* code, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  unsigned a = code[i], b = code[j];
  if (a == b) return 32 + __clz((unsigned)(i ^ j));
  return __clz(a ^ b);
}

// Build tree `k` (blockIdx.x) over the query boxes [lo, hi]. Node layout of a
// tree with n leaves: internal nodes node0 .. node0+n-2 (root = node0),
// children encoded as >= 0: internal node (absolute index), < 0: ~leaf;
// leaf l (sorted position) holds primitive bvh_prim[leaf0 + l].
IPC_GLOBAL void __launch_bounds__(LBVH_THREADS) k_lbvh_build(World W, const double* __restrict__ lo,
                                                             const double* __restrict__ hi) {
  ipc_pdl_wait();
  const int k = blockIdx.x;
  const int kind = W.tree_kind[k], p0 = W.tree_p0[k], n = W.tree_n[k];
  const int node0 = W.tree_node0[k], leaf0 = W.tree_leaf0[k];
  extern __shared__ unsigned lbvh_sm[];
  unsigned* key = lbvh_sm;             // [n]
  unsigned* key2 = key + LBVH_MAX;     // [n]
  int* val = reinterpret_cast<int*>(key2 + LBVH_MAX);   // [n]
  int* val2 = val + LBVH_MAX;          // [n]
  __shared__ double sbox[6];
  __shared__ int hist[LBVH_THREADS / 32][16];
  __shared__ int dbase[LBVH_THREADS / 32][16];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = LBVH_THREADS / 32;
  // body box of the centroids
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = tid; i < n; i += LBVH_THREADS) {
    double b[6];
    lbvh_prim_box(W, kind, p0 + i, lo, hi, b);
    for (int c = 0; c < 3; ++c) {
      double ce = 0.5 * (b[c] + b[3 + c]);
      mn[c] = fmin(mn[c], ce);
      mx[c] = fmax(mx[c], ce);
    }
  }
  for (int o = 16; o > 0; o >>= 1)
    for (int c = 0; c < 3; ++c) {
      mn[c] = fmin(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
      mx[c] = fmax(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
    }
  __shared__ double wmn[NW][3], wmx[NW][3];
  if (lane == 0)
    for (int c = 0; c < 3; ++c) {
      wmn[wid][c] = mn[c];
      wmx[wid][c] = mx[c];
    }
  __syncthreads();
  if (tid < 3) {
    double a = INFINITY, b = -INFINITY;
    for (int w = 0; w < NW; ++w) {
      a = fmin(a, wmn[w][tid]);
      b = fmax(b, wmx[w][tid]);
    }
    sbox[tid] = a;
    sbox[3 + tid] = b;
  }
  __syncthreads();
  // Morton codes
  for (int i = tid; i < n; i += LBVH_THREADS) {
    double b[6];
    lbvh_prim_box(W, kind, p0 + i, lo, hi, b);
    unsigned q[3];
    for (int c = 0; c < 3; ++c) {
      double ext = sbox[3 + c] - sbox[c];
      double u = ext > 0.0 ? (0.5 * (b[c] + b[3 + c]) - sbox[c]) / ext : 0.5;
      q[c] = (unsigned)fmin(fmax(u * 1024.0, 0.0), 1023.0);
    }
    key[i] = (lbvh_expand10(q[0]) << 2) | (lbvh_expand10(q[1]) << 1) | lbvh_expand10(q[2]);
    val[i] = i;
  }
  __syncthreads();
  // stable LSD radix sort, 4-bit digits, warp-level multisplit: warp w owns
  // the contiguous element range [w*per, (w+1)*per) and walks it in 32-wide
  // chunks in order, so ranks inside a (digit, warp) bucket follow the input
  const int per = (n + NW - 1) / NW;
  for (int shift = 0; shift < 30; shift += 4) {
    if (lane < 16) hist[wid][lane] = 0;
    __syncwarp();
    int w0 = wid * per, w1 = min(n, w0 + per);
    for (int c0 = w0; c0 < w1; c0 += 32) {
      int i = c0 + lane;
      bool in = i < w1;
      unsigned d = in ? (key[i] >> shift) & 15u : 16u;
      unsigned peers = __match_any_sync(0xffffffffu, d);
      if (in && lane == __ffs(peers) - 1) hist[wid][d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    if (tid == 0) {  // exclusive scan, digit-major then warp order (stability)
      int acc = 0;
      for (int d = 0; d < 16; ++d)
        for (int w = 0; w < NW; ++w) {
          dbase[w][d] = acc;
          acc += hist[w][d];
        }
    }
    __syncthreads();
    for (int c0 = w0; c0 < w1; c0 += 32) {
      int i = c0 + lane;
      bool in = i < w1;
      unsigned kk = in ? key[i] : 0u;
      unsigned d = in ? (kk >> shift) & 15u : 16u;
      unsigned peers = __match_any_sync(0xffffffffu, d);
      int rank = __popc(peers & ((1u << lane) - 1u));
      if (in) {
        int dst = dbase[wid][d] + rank;
        key2[dst] = kk;
        val2[dst] = val[i];
      }
      __syncwarp();
      if (in && lane == __ffs(peers) - 1) dbase[wid][d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    for (int i = tid; i < n; i += LBVH_THREADS) {
      key[i] = key2[i];
      val[i] = val2[i];
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += LBVH_THREADS) W.bvh_prim[leaf0 + i] = p0 + val[i];
  // Karras internal nodes
  int* flag = val2;  // reuse: arrival counters of internal nodes
  for (int i = tid; i < n - 1; i += LBVH_THREADS) {
    int d = lbvh_delta(key, n, i, i + 1) - lbvh_delta(key, n, i, i - 1) >= 0 ? 1 : -1;
    int dmin = lbvh_delta(key, n, i, i - d);
    int lmax = 2;
    while (lbvh_delta(key, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
      if (lbvh_delta(key, n, i, i + (l + t) * d) > dmin) l += t;
    int j = i + l * d;
    int dnode = lbvh_delta(key, n, i, j);
    int s = 0;
    for (int t = (l + 1) >> 1;; t = (t + 1) >> 1) {
      if (lbvh_delta(key, n, i, i + (s + t) * d) > dnode) s += t;
      if (t == 1) break;
    }
    int split = i + s * d + min(d, 0);
    int lo_i = min(i, j), hi_i = max(i, j);
    int left = lo_i == split ? ~split : node0 + split;
    int right = hi_i == split + 1 ? ~(split + 1) : node0 + split + 1;
    W.bvh_child[2 * (node0 + i)] = left;
    W.bvh_child[2 * (node0 + i) + 1] = right;
    if (left >= 0) W.bvh_parent[left] = node0 + i; else W.bvh_lparent[leaf0 + ~left] = node0 + i;
    if (right >= 0) W.bvh_parent[right] = node0 + i; else W.bvh_lparent[leaf0 + ~right] = node0 + i;
    flag[i] = 0;
  }
  __syncthreads();
  // refit: each leaf walks up; the second child to arrive at a node unions it
  for (int l = tid; l < n; l += LBVH_THREADS) {
    if (n == 1) break;
    int node = W.bvh_lparent[leaf0 + l];
    while (true) {
      __threadfence_block();
      if (atomicAdd(&flag[node - node0], 1) == 0) break;
      double b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
      for (int s2 = 0; s2 < 2; ++s2) {
        int ch = W.bvh_child[2 * node + s2];
        double cb[6];
        if (ch >= 0) {
          for (int c = 0; c < 6; ++c) cb[c] = ((volatile double*)W.bvh_box)[6 * ch + c];
        } else {
          lbvh_prim_box(W, kind, W.bvh_prim[leaf0 + ~ch], lo, hi, cb);
        }
        for (int c = 0; c < 3; ++c) {
          b[c] = fmin(b[c], cb[c]);
          b[3 + c] = fmax(b[3 + c], cb[3 + c]);
        }
      }
      for (int c = 0; c < 6; ++c) W.bvh_box[6 * node + c] = b[c];
      if (node == node0) break;
      node = W.bvh_parent[node];
    }
  }
}

// Visit, in increasing index order, the primitives of tree k in [c0, c1) that
// pass `test` (the exact prim-level test); returns false (nothing visited)
// when more than LBVH_HITS primitives hit — the caller then walks the chunks.
template <typename Test, typename F>
__device__ __forceinline__ bool lbvh_visit(const World& W, int k, const double* qlo, const double* qhi,
                                           double margin, int c0, int c1, Test test, F f) {
  const int n = W.tree_n[k], node0 = W.tree_node0[k], leaf0 = W.tree_leaf0[k];
  int hits[LBVH_HITS];
  int nh = 0;
  int stack[64];
  int sp = 0;
  stack[sp++] = n == 1 ? ~0 : node0;
  while (sp > 0) {
    int node = stack[--sp];
    if (node < 0) {
      int t = W.bvh_prim[leaf0 + ~node];
      if (t >= c0 && t < c1 && test(t)) {
        if (nh == LBVH_HITS) return false;
        hits[nh++] = t;
      }
      continue;
    }
    const double* b = W.bvh_box + 6 * node;
    if (!lbvh_box_hit(qlo, qhi, b, b + 3, margin)) continue;
    stack[sp++] = W.bvh_child[2 * node + 1];
    stack[sp++] = W.bvh_child[2 * node];
  }
  for (int i = 1; i < nh; ++i) {  // ascending primitive order
    int v = hits[i], j = i - 1;
    while (j >= 0 && hits[j] > v) {
      hits[j + 1] = hits[j];
      --j;
    }
    hits[j + 1] = v;
  }
  for (int i = 0; i < nh; ++i) f(hits[i]);
  return true;
}

}  // namespace ipc
