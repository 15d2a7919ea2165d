// Checks the rank computation of k_env_order (solve.cuh)
// against std::sort on random keys, n = 1..1024.  nvcc -arch=sm_100a
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
__global__ void rank_order(int n, const long long* in, long long* out) {
  __shared__ long long key[4096];
  for (int i = threadIdx.x; i < n; i += blockDim.x) key[i] = in[i];
  __syncthreads();
  int lane = threadIdx.x & 31, e = blockIdx.x * 32 + (threadIdx.x >> 5);
  if (e >= n) return;
  long long k = key[e];
  unsigned cnt = 0;
  for (int j = lane; j < n; j += 32) cnt += key[j] > k;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) out[cnt] = k;
}
int main() {
  long long *din, *dout;
  cudaMalloc(&din, 32768);
  cudaMalloc(&dout, 32768);
  int bad = 0;
  for (int n : {1, 2, 3, 31, 33, 48, 100, 511, 512, 700, 1023, 1024, 3000, 4096}) {
    std::vector<long long> h(n), r(n);
    for (int i = 0; i < n; ++i) h[i] = ((long long)(rand() % 50) << 12) | (4095 - i);
    cudaMemcpy(din, h.data(), 8 * n, cudaMemcpyHostToDevice);
    rank_order<<<(n + 31) / 32, 1024>>>(n, din, dout);
    cudaMemcpy(r.data(), dout, 8 * n, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end(), [](long long a, long long b) { return a > b; });
    if (h != r) { printf("n=%d MISMATCH\n", n); ++bad; }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) rank_order<<<32, 1024>>>(1024, din, dout);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%s, %.2f us/launch\n", bad ? "FAIL" : "order_check ok", ms * 10);
  return bad;
}
