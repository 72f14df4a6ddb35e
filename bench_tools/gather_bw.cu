// Microbenchmark: achievable HBM read bandwidth for (a) a contiguous stream,
// (b) gathers of 256-B rows at ascending random positions (25% density) through
// a page table, as K3 does.  Each warp loads 16 B per lane (2 rows / instr)
// with ld.global.nc.v4 and many loads in flight (unrolled).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

extern "C" __global__ void stream_read(const int4* __restrict__ p, int64_t n16, int* out) {
  int acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { int4 v = __ldg(p + i); acc ^= v.x ^ v.w; }
  if (acc == 0x12345678) out[0] = acc;
}

// rows: int64 row indices (in units of 256 B rows), n_rows entries
extern "C" __global__ void gather_rows(const int4* __restrict__ pool, const int64_t* __restrict__ rows,
                                       int64_t n_rows, int* out) {
  int acc = 0;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // each warp handles 16 rows per iteration: lane l reads chunk (l & 15) of row 2*u + (l >> 4)
  for (int64_t r0 = wid * 16; r0 < n_rows; r0 += nw * 16) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = r0 + 2 * u + (lane >> 4);
      const int64_t row = r < n_rows ? rows[r] : 0;
      v[u] = __ldg(pool + row * 16 + (lane & 15));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

#include <vector>
#include <random>
#include <algorithm>
int main() {
  const int64_t pool_bytes = 8ll << 30;   // 8 GB pool
  int4* pool;
  cudaMalloc(&pool, pool_bytes);
  cudaMemset(pool, 1, pool_bytes);
  int* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int64_t n16 = (4ll << 30) / 16;
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(a);
    stream_read<<<148 * 8, 256>>>(pool, n16, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("stream read: %.1f GB/s\n", (4ll << 30) / (ms * 1e-3) / 1e9);
  const int64_t total_rows = pool_bytes / 256;
  std::mt19937_64 rng(1);
  for (double density : {0.25, 0.5, 1.0, 0.05}) {
    const int64_t want = 16ll << 20;
    std::vector<int64_t> rows;
    rows.reserve(want);
    const int64_t npages = total_rows / 64;
    std::vector<int64_t> perm(npages);
    for (int64_t i = 0; i < npages; ++i) perm[i] = i;
    std::shuffle(perm.begin(), perm.end(), rng);
    int64_t pi = 0;
    std::uniform_real_distribution<double> U(0, 1);
    while ((int64_t)rows.size() < want) {
      const int64_t page = perm[pi++ % npages];
      for (int r = 0; r < 64; ++r)
        if (U(rng) < density) rows.push_back(page * 64 + r);
    }
    rows.resize(want);
    int64_t* drows;
    cudaMalloc(&drows, want * 8);
    cudaMemcpy(drows, rows.data(), want * 8, cudaMemcpyHostToDevice);
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(a);
      gather_rows<<<148 * 8, 256>>>(pool, drows, want, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("paged gather density %.2f: %.1f GB/s rows (+%.1f GB/s index reads)\n", density,
           want * 256.0 / (ms * 1e-3) / 1e9, want * 8.0 / (ms * 1e-3) / 1e9);
    cudaFree(drows);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
