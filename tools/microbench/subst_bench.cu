// Standalone microbenchmark behind DESIGN §[r2b]: the warp substitution of the
// dense env solve, plain (V0), loads hoisted (V1), and with a large live
// register array around it (V2: the compiler turns the predicated updates into
// branches and re-reads special registers; ~3x slower). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o subst_bench subst_bench.cu
// microbenchmark: warp-0 triangular substitution of the dense env solve
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ int hix(int r, int c) { return r * (r + 1) / 2 + c; }
template <int V>
__global__ void k_sub(const double* Hg, const double* dinv_g, const double* yg, double* out, int n, int reps) {
  extern __shared__ double sm[];
  double* H = sm;
  double* y = H + n * (n + 1) / 2;
  __shared__ double s_dinv[160];
  int tid = threadIdx.x;
  for (int i = tid; i < n * (n + 1) / 2; i += blockDim.x) H[i] = Hg[i];
  for (int i = tid; i < n; i += blockDim.x) { y[i] = yg[i]; s_dinv[i] = dinv_g[i]; }
  __syncthreads();
  double big[96];
#pragma unroll
  for (int i = 0; i < 96; ++i) big[i] = Hg[(i * 7 + tid) % 10] * (V == 2 ? 1.0 : 0.0);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (tid < 32) {
      const unsigned FULL = 0xffffffffu;
      int lane = tid, i1 = lane + 32;
      double y0 = lane < n ? y[lane] : 0.0, y1 = i1 < n ? y[i1] : 0.0;
      if (V == 0 || V == 2) {
        for (int k = 0; k < n; ++k) {
          double uk = __shfl_sync(FULL, k < 32 ? y0 : y1, k & 31);
          double dk = s_dinv[k];
          if (lane > k && lane < n) y0 -= (H[hix(lane, k)] * dk) * uk;
          if (i1 > k && i1 < n) y1 -= (H[hix(i1, k)] * dk) * uk;
        }
        if (lane < n) y0 *= s_dinv[lane];
        if (i1 < n) y1 *= s_dinv[i1];
        for (int k = n - 1; k >= 0; --k) {
          double xk = __shfl_sync(FULL, k < 32 ? y0 : y1, k & 31);
          if (lane < k) y0 -= (H[hix(k, lane)] * s_dinv[lane]) * xk;
          if (i1 < k) y1 -= (H[hix(k, i1)] * s_dinv[i1]) * xk;
        }
      } else {
        // V1: row k of L read by lanes ahead of the chain: the coefficient of
        // step k is loaded before the broadcast it waits on
        double dl0 = lane < n ? s_dinv[lane] : 0.0, dl1 = i1 < n ? s_dinv[i1] : 0.0;
        for (int k = 0; k < n; ++k) {
          double c0 = (lane > k && lane < n) ? H[hix(lane, k)] * s_dinv[k] : 0.0;
          double c1 = (i1 > k && i1 < n) ? H[hix(i1, k)] * s_dinv[k] : 0.0;
          double uk = __shfl_sync(FULL, k < 32 ? y0 : y1, k & 31);
          y0 -= c0 * uk;
          y1 -= c1 * uk;
        }
        y0 *= dl0;
        y1 *= dl1;
        for (int k = n - 1; k >= 0; --k) {
          double c0 = lane < k ? H[hix(k, lane)] * dl0 : 0.0;
          double c1 = i1 < k ? H[hix(k, i1)] * dl1 : 0.0;
          double xk = __shfl_sync(FULL, k < 32 ? y0 : y1, k & 31);
          y0 -= c0 * xk;
          y1 -= c1 * xk;
        }
      }
      if (lane < n) y[lane] = y0;
      if (i1 < n) y[i1] = y1;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (V == 2) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 96; ++i) acc += big[i] * big[(i + 1) % 96];
    if (acc == 12345.0) out[0] = acc;
  }
  if (tid == 0) out[blockIdx.x] = (double)(t1 - t0) / reps;
  if (tid < n) out[gridDim.x + blockIdx.x * n + tid] = y[tid];
}
int main() {
  int n = 48, E = 1024, reps = 20;
  int nl = n * (n + 1) / 2;
  double *H, *d, *y, *out;
  cudaMallocManaged(&H, nl * 8); cudaMallocManaged(&d, n * 8); cudaMallocManaged(&y, n * 8);
  cudaMallocManaged(&out, (E + E * n) * 8);
  for (int i = 0; i < nl; ++i) H[i] = 0.01 * ((i * 37) % 11);
  for (int i = 0; i < n; ++i) { d[i] = 0.5; y[i] = 1.0 + 0.01 * i; }
  size_t smem = (nl + n) * 8;
  for (int v = 0; v < 3; ++v) {
    for (int grid : {1, E}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      if (v == 0) k_sub<0><<<grid, 256, smem>>>(H, d, y, out, n, reps);
      else if (v == 1) k_sub<1><<<grid, 256, smem>>>(H, d, y, out, n, reps);
      else k_sub<2><<<grid, 256, smem>>>(H, d, y, out, n, reps);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("V%d grid %d: %.1f cycles per substitution (CTA 0), %.3f ms total, y[5]=%.17g err=%s\n", v, grid, out[0], ms, out[grid + 5], cudaGetErrorString(cudaGetLastError()));
    }
  }
}
