// match_heads.cu — K0: prefill similarity matching (Eq. 2-3).
//
//   T_i  = TopK(F(A_i, C))  (k largest accumulated scores over the matching
//          window, ties -> lower position)
//   S(i,j) = |T_i ∩ T'_j| / |T_i ∪ T'_j|                       (Eq. 2)
//   f(i) = argmax_j S(i, j), ties -> smallest flat SLM head j   (Eq. 3)
//
// Kernel A builds each vector's TopK as a bitset (w <= 512 -> 16 words) by
// exact rank counting; kernel B, one CTA per LLM head, scans all SLM bitsets
// with popc and compares Jaccard values as exact rationals (no float ties).
#include "common.cuh"
#include "kernels.h"

namespace skv {

namespace {
constexpr int kWords = 16;   // 512-position windows

__global__ void __launch_bounds__(256) topk_bits_kernel(const float* __restrict__ llm_F,
                                                        int32_t n_llm,
                                                        const float* __restrict__ slm_F,
                                                        int32_t w, int32_t k,
                                                        uint32_t* __restrict__ bits) {
  __shared__ float F[512];
  const int vec = blockIdx.x;
  const float* src = vec < n_llm ? llm_F + static_cast<int64_t>(vec) * w
                                 : slm_F + static_cast<int64_t>(vec - n_llm) * w;
  for (int i = threadIdx.x; i < w; i += blockDim.x) F[i] = src[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int base = (threadIdx.x & ~31); base < kWords * 32; base += blockDim.x) {
    const int v = base + lane;
    bool in = false;
    if (v < w) {
      const float fv = F[v];
      int rank = 0;
      for (int u = 0; u < w; ++u) {
        const float fu = F[u];
        rank += (fu > fv || (fu == fv && u < v)) ? 1 : 0;
      }
      in = rank < k;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0) bits[static_cast<int64_t>(vec) * kWords + base / 32] = bal;
  }
}

__global__ void __launch_bounds__(256) match_kernel(const uint32_t* __restrict__ bits,
                                                    int32_t n_llm, int32_t n_slm,
                                                    int32_t* __restrict__ head_map,
                                                    float* __restrict__ jaccard) {
  __shared__ uint32_t a[kWords];
  __shared__ int s_i[256], s_u[256], s_j[256];
  const int i = blockIdx.x;
  if (threadIdx.x < kWords) a[threadIdx.x] = bits[static_cast<int64_t>(i) * kWords + threadIdx.x];
  __syncthreads();
  int bi = -1, bu = 1, bj = 0x7fffffff;
  for (int j = threadIdx.x; j < n_slm; j += blockDim.x) {
    const uint32_t* bb = bits + static_cast<int64_t>(n_llm + j) * kWords;
    int inter = 0, uni = 0;
#pragma unroll
    for (int q = 0; q < kWords; ++q) {
      const uint32_t y = bb[q];
      inter += __popc(a[q] & y);
      uni += __popc(a[q] | y);
    }
    if (uni == 0) { inter = 1; uni = 1; }   // both empty: similarity 1
    // strictly better rational; j increases, so ties keep the smaller j
    if (static_cast<int64_t>(inter) * bu > static_cast<int64_t>(bi) * uni) {
      bi = inter; bu = uni; bj = j;
    }
  }
  s_i[threadIdx.x] = bi; s_u[threadIdx.x] = bu; s_j[threadIdx.x] = bj;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const int oi = s_i[threadIdx.x + s], ou = s_u[threadIdx.x + s], oj = s_j[threadIdx.x + s];
      const int64_t lhs = static_cast<int64_t>(oi) * s_u[threadIdx.x];
      const int64_t rhs = static_cast<int64_t>(s_i[threadIdx.x]) * ou;
      if (lhs > rhs || (lhs == rhs && oj < s_j[threadIdx.x])) {
        s_i[threadIdx.x] = oi; s_u[threadIdx.x] = ou; s_j[threadIdx.x] = oj;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    head_map[i] = s_j[0];
    jaccard[i] = static_cast<float>(static_cast<double>(s_i[0]) / static_cast<double>(s_u[0]));
  }
}
}  // namespace

cudaError_t launch_match_heads(const float* llm_F, int32_t n_llm, const float* slm_F,
                               int32_t n_slm, int32_t w, int32_t k, uint32_t* bits_ws,
                               int32_t* head_map, float* jaccard, cudaStream_t s) {
  topk_bits_kernel<<<n_llm + n_slm, 256, 0, s>>>(llm_F, n_llm, slm_F, w, k, bits_ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  match_kernel<<<n_llm, 256, 0, s>>>(bits_ws, n_llm, n_slm, head_map, jaccard);
  return cudaGetLastError();
}

}  // namespace skv
