// fp64 roofline denominator: measured DFMA throughput of this device.
//
// MEASURED_PEAKS.json (driver-written) carries HBM and bf16 tensor peaks
// only; every kernel of the IPC step computes in fp64 on the CUDA cores, so
// the compute roofline needs the fp64 pipe's own ceiling. k_dfma_peak runs
// 8 independent DFMA chains per thread (enough ILP to cover the pipe
// latency) on a grid of 8 CTAs x 256 threads per SM; flops = 2 per DFMA.
#include <cuda_runtime.h>

#include <string>

#include "../../include/ipc_b200.h"

namespace {

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 123.456) out[0] = s;  // keeps the chains live; never true
}

}  // namespace

extern "C" int ipc_measure_fp64_peak(int iters, double* tflops) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 1;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int grid = 8 * sms, block = 256;
  k_dfma_peak<<<grid, block>>>(out, iters / 4 + 1, 0.9999999, 1e-12);  // warm-up / clock ramp
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma_peak<<<grid, block>>>(out, iters, 0.9999999, 1e-12);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return 1;
  double flops = 2.0 * 8.0 * 16.0 * (double)iters * (double)grid * (double)block;
  *tflops = flops / (best * 1e-3) / 1e12;
  return 0;
}
