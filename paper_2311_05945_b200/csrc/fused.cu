// Translation unit of the fused per-environment step kernels (k_env_step,
// k_env_steps, k_env_newton_rest); the host engine in engine.cu launches them.
// Compiled separately so the two large units build in parallel.
#define IPC_FUSED_TU
#include <cuda_runtime.h>

#include "fused.cuh"
