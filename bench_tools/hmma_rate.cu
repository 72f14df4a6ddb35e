// Microbenchmark: legacy mma.sync m16n8k16 bf16->fp32 (SASS HMMA) on sm_100a:
// issue throughput per SM vs warps per SM, and dependent-chain latency.
// The attend consumer runs 48 HMMA per 16-row K+V tile; this bounds it.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int CHAINS>
__global__ void hmma_kernel(int iters, float* out) {
  float acc[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, b0 = a0 ^ 0x3c00u, b1 = a0 ^ 0x3f80u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1234.5f) out[0] = s;
}

template <int CHAINS>
void run(int warps_per_sm, float* out) {
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    hmma_kernel<CHAINS><<<148, warps_per_sm * 32>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double n_hmma_sm = (double)warps_per_sm * iters * CHAINS;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("chains %2d warps/SM %2d: %.2f cycles per HMMA per SM (%.2f per SMSP), %.1f TFLOP/s  %s\n", CHAINS,
         warps_per_sm, cycles / n_hmma_sm, 4 * cycles / n_hmma_sm,
         148.0 * n_hmma_sm * 4096 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  run<1>(1, out);   // latency: cycles per dependent HMMA (x1 since 1 warp)
  run<2>(1, out);
  run<8>(1, out);
  run<8>(4, out);
  run<8>(8, out);
  run<8>(16, out);
  run<16>(8, out);
  return 0;
}
