// Microbenchmark: HBM bandwidth of 16-byte cp.async gathers of 256-B rows into
// per-warp shared-memory rings, vs warps per SM and ring depth (tiles of 16
// rows x 2 arrays = 8 KB, the attend kernel's stage), against random paged rows.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>
#include <random>
#include <algorithm>

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}

template <int NSTAGE>
__global__ void ring_kernel(const int4* __restrict__ pool, const int64_t* __restrict__ rows,
                            int64_t tiles_per_warp, int* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = sm + warp * NSTAGE * 8192;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t* myrows = rows + gw * tiles_per_warp * 32;   // 32 rows (16 K + 16 V) per tile
  int acc = 0;
  auto issue = [&](int64_t t) {
    if (t < tiles_per_warp) {
      uint8_t* st = ring + (t % NSTAGE) * 8192;
#pragma unroll
      for (int g = 0; g < 8; ++g) {   // 8 instructions x 32 lanes x 16 B = 4 KB ... x2
        const int e = g * 4 + (lane >> 3);
        const int64_t r = myrows[t * 32 + e];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int ch = hf * 8 + (lane & 7);
          cp16((uint32_t)__cvta_generic_to_shared(st + e * 256 + ch * 16), pool + r * 16 + ch);
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  for (int i = 0; i < NSTAGE - 1; ++i) issue(i);
  for (int64_t t = 0; t < tiles_per_warp; ++t) {
    issue(t + NSTAGE - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NSTAGE - 1) : "memory");
    __syncwarp();
    acc ^= *reinterpret_cast<const int*>(ring + (t % NSTAGE) * 8192 + lane * 4);
    __syncwarp();
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <int NSTAGE>
void run(const int4* pool, const int64_t* rows, int64_t nrows_total, int warps_per_cta,
         int ctas_per_sm, int* out) {
  const int ctas = 148 * ctas_per_sm;
  const int64_t warps = (int64_t)ctas * warps_per_cta;
  const int64_t tiles_per_warp = nrows_total / 32 / warps;
  const size_t smem = (size_t)warps_per_cta * NSTAGE * 8192;
  cudaFuncSetAttribute(ring_kernel<NSTAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0;
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(a);
    ring_kernel<NSTAGE><<<ctas, warps_per_cta * 32, smem>>>(pool, rows, tiles_per_warp, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  const double bytes = (double)warps * tiles_per_warp * 32 * 256;
  printf("warps/SM %2d (CTAs/SM %d x %d warps), stages %d (%3zu KB smem/SM, %3d KB in flight/SM): %7.1f GB/s  %s\n",
         warps_per_cta * ctas_per_sm, ctas_per_sm, warps_per_cta, NSTAGE,
         smem * ctas_per_sm / 1024, warps_per_cta * ctas_per_sm * (NSTAGE - 1) * 8, bytes / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t pool_bytes = 8ll << 30;
  int4* pool;
  cudaMalloc(&pool, pool_bytes);
  cudaMemset(pool, 1, pool_bytes);
  int* out;
  cudaMalloc(&out, 4);
  const int64_t total_rows = pool_bytes / 256, want = 16ll << 20;
  std::vector<int64_t> rows;
  rows.reserve(want);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(0, 1);
  const int64_t npages = total_rows / 64;
  std::vector<int64_t> perm(npages);
  for (int64_t i = 0; i < npages; ++i) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), rng);
  for (int64_t pi = 0; (int64_t)rows.size() < want; ++pi)
    for (int r = 0; r < 64; ++r)
      if (U(rng) < 0.25) rows.push_back(perm[pi % npages] * 64 + r);
  rows.resize(want);
  int64_t* drows;
  cudaMalloc(&drows, want * 8);
  cudaMemcpy(drows, rows.data(), want * 8, cudaMemcpyHostToDevice);
  run<3>(pool, drows, want, 4, 2, out);    // the attend kernel today
  run<2>(pool, drows, want, 4, 2, out);
  run<4>(pool, drows, want, 3, 2, out);
  run<3>(pool, drows, want, 8, 1, out);
  run<6>(pool, drows, want, 4, 1, out);
  run<2>(pool, drows, want, 4, 3, out);
  run<2>(pool, drows, want, 8, 1, out);
  run<13>(pool, drows, want, 2, 1, out);
  run<3>(pool, drows, want, 2, 4, out);
  return 0;
}
