// prefill.cu — variant f3: the prefill-side F vectors of head
// matching.  For one sequence, every layer l and q-head h (R17):
//   A[u][v] = softmax_{v <= start+u} (q_{l,u,h} · k_{l,v,kv(h)} / sqrt(d))
//   F[l*H+h][v-start] = Σ_{u in window} A[u][v],  v in [start, start+len)    (Eq. 1)
// — the column sums of the window's causal prefill attention rows over their
// full prefix; smallkv_match_heads (K0, Eq. 2-3) consumes them.
//
// CTA = (head, layer), 4 warps; each warp owns 16-query tiles of the window.
// Two passes over the key tiles of a query tile on the tensor cores
// (mma.sync m16n8k16, queries = M, keys = N): (1) per-row max and Σexp,
// (2) p = exp(s - m) / l, column-summed over the tile's rows with warp
// shuffles into per-warp shared-memory partials; the warps' partials are added
// in a fixed order (deterministic).  Q and K fragments are read straight from
// global memory (L2-resident): prefill matching is off the decode hot path.
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace skv {

namespace {
constexpr int kPfWarps = 4;

template <int D>
__global__ void __launch_bounds__(kPfWarps * 32) prefill_scores_kernel(const PrefillParams p) {
  extern __shared__ float fw[];   // [kPfWarps][len]
  const int h = blockIdx.x, l = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int G = p.heads / p.kv_heads, kvh = h / G;
  const int len = p.len;
  for (int i = threadIdx.x; i < kPfWarps * len; i += blockDim.x) fw[i] = 0.f;
  __syncthreads();
  const int32_t* bt = p.block_table + static_cast<int64_t>(p.seq) * p.max_blocks;
  const uint16_t* kpool = p.k + static_cast<int64_t>(l) * p.layer_stride;
  // element offset of key v's row in this layer's pool
  auto krow = [&](int v) -> int64_t {
    const int page = __ldg(bt + (v >> p.ps_shift));
    return ((static_cast<int64_t>(page) * p.kv_heads + kvh) * p.page_size + (v & (p.page_size - 1))) * D;
  };
  float* myf = fw + warp * len;
  for (int u0 = warp * 16; u0 < len; u0 += kPfWarps * 16) {
    // A fragments: queries u0 + gq, u0 + gq + 8 (zero past the window)
    uint32_t qa[D / 16][4];
    const int ua = u0 + gq, ub = u0 + gq + 8;
    const uint16_t* qa_row = p.q + ((static_cast<int64_t>(l) * len + ua) * p.heads + h) * D;
    const uint16_t* qb_row = p.q + ((static_cast<int64_t>(l) * len + ub) * p.heads + h) * D;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int c = 16 * kk + 2 * tq;
      qa[kk][0] = ua < len ? *reinterpret_cast<const uint32_t*>(qa_row + c) : 0u;
      qa[kk][1] = ub < len ? *reinterpret_cast<const uint32_t*>(qb_row + c) : 0u;
      qa[kk][2] = ua < len ? *reinterpret_cast<const uint32_t*>(qa_row + c + 8) : 0u;
      qa[kk][3] = ub < len ? *reinterpret_cast<const uint32_t*>(qb_row + c + 8) : 0u;
    }
    const int pa = p.start + ua, pb = p.start + ub;               // query positions
    const int kend = min(p.start + u0 + 16, p.start + len);        // keys [0, kend)
    // S tile [16 q x 8 keys] at keys n0..n0+7 (scaled, causally masked)
    auto tile = [&](int n0, float (&s)[4]) {
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      const int key = n0 + gq;                                     // this lane's B column
      const bool kv = key < kend;
      const uint16_t* kr = kpool + (kv ? krow(key) : 0);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t b0 = kv ? *reinterpret_cast<const uint32_t*>(kr + 16 * kk + 2 * tq) : 0u;
        const uint32_t b1 = kv ? *reinterpret_cast<const uint32_t*>(kr + 16 * kk + 8 + 2 * tq) : 0u;
        mma_bf16(c, qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
      }
      const int k0 = n0 + 2 * tq;
      s[0] = (k0 <= pa && ua < len) ? c[0] * p.scale : -INFINITY;
      s[1] = (k0 + 1 <= pa && ua < len) ? c[1] * p.scale : -INFINITY;
      s[2] = (k0 <= pb && ub < len) ? c[2] * p.scale : -INFINITY;
      s[3] = (k0 + 1 <= pb && ub < len) ? c[3] * p.scale : -INFINITY;
    };
    // pass 1: row max and Σexp (lane-partial over its 2 columns, then the 4 lanes of a row)
    float ma = -INFINITY, mb = -INFINITY, la = 0.f, lb = 0.f;
    for (int n0 = 0; n0 < kend; n0 += 8) {
      float s[4];
      tile(n0, s);
      const float na = fmaxf(ma, fmaxf(s[0], s[1])), nb = fmaxf(mb, fmaxf(s[2], s[3]));
      if (na > -INFINITY) {
        la = la * __expf(ma - na) + __expf(s[0] - na) + __expf(s[1] - na);
        ma = na;
      }
      if (nb > -INFINITY) {
        lb = lb * __expf(mb - nb) + __expf(s[2] - nb) + __expf(s[3] - nb);
        mb = nb;
      }
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const float m2a = __shfl_xor_sync(0xffffffffu, ma, o), l2a = __shfl_xor_sync(0xffffffffu, la, o);
      const float m2b = __shfl_xor_sync(0xffffffffu, mb, o), l2b = __shfl_xor_sync(0xffffffffu, lb, o);
      const float na = fmaxf(ma, m2a), nb = fmaxf(mb, m2b);
      la = (na > -INFINITY) ? la * __expf(ma - na) + l2a * __expf(m2a - na) : 0.f;
      lb = (nb > -INFINITY) ? lb * __expf(mb - nb) + l2b * __expf(m2b - nb) : 0.f;
      ma = na;
      mb = nb;
    }
    const float ia = la > 0.f ? 1.f / la : 0.f, ib = lb > 0.f ? 1.f / lb : 0.f;
    // pass 2: probabilities, column sums over the tile's 16 rows, window columns only
    for (int n0 = (p.start / 8) * 8; n0 < kend; n0 += 8) {
      float s[4];
      tile(n0, s);
      float c0 = (s[0] > -INFINITY ? __expf(s[0] - ma) * ia : 0.f) + (s[2] > -INFINITY ? __expf(s[2] - mb) * ib : 0.f);
      float c1 = (s[1] > -INFINITY ? __expf(s[1] - ma) * ia : 0.f) + (s[3] > -INFINITY ? __expf(s[3] - mb) * ib : 0.f);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      }
      if (gq == 0) {
        const int k0 = n0 + 2 * tq;
        if (k0 >= p.start && k0 < p.start + len) myf[k0 - p.start] += c0;
        if (k0 + 1 >= p.start && k0 + 1 < p.start + len) myf[k0 + 1 - p.start] += c1;
      }
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < len; v += blockDim.x) {
    float f = 0.f;
#pragma unroll
    for (int w = 0; w < kPfWarps; ++w) f += fw[w * len + v];
    p.F[(static_cast<int64_t>(l) * p.heads + h) * len + v] = f;
  }
}
}  // namespace

cudaError_t launch_prefill_scores(const PrefillParams& p, cudaStream_t s) {
  const size_t sm = static_cast<size_t>(kPfWarps) * p.len * sizeof(float);
  dim3 grid(p.heads, p.layers);
  if (p.head_dim == 64) {
    cudaFuncSetAttribute(prefill_scores_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    prefill_scores_kernel<64><<<grid, kPfWarps * 32, sm, s>>>(p);
  } else {
    cudaFuncSetAttribute(prefill_scores_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    prefill_scores_kernel<128><<<grid, kPfWarps * 32, sm, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace skv
