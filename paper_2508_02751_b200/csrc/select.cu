// select.cu — K2: per-row softmax statistics and the critical / marginal split.
//
// For every distinct SLM row j in image(f) and sequence b (one CTA each):
//   m' = max_v s'_v, lse' = m' + ln Σ_v exp(s'_v - m')     (A'_{f(i)} normaliser, Eq. 6)
//   recent R' = [n-R', n); positions [0, n-R') ranked by
//   (s' desc, v asc) — ranking the fp32 logits is order-equivalent to ranking
//   a' = exp(s' - lse') (R1, R3);
//   critical = rank < K' (Eq. 6 TopK), marginal = K' <= rank < K'+M' (Top(P-K), R4).
// Output: ascending compacted crit_idx / marg_idx, marg_w = a'_v, counts (K', M').
//
// Exact selection with a deterministic lower-index tie-break.  Each rank
// boundary becomes a lexicographic threshold (T, I) on (key, index), where
// key is an order-preserving uint32 of the logit (smaller key = larger score):
// position v is selected iff key_v < T or (key_v == T and v <= I).
//   Fast path: one pass builds a 256-bin histogram that is LINEAR in the logit
//   value over [min, max] of the ranked positions (monotone, so bins are
//   ordered like scores; per-warp private shared-memory histograms), a suffix
//   scan finds each boundary's bin, one pass collects that bin's (key, index)
//   pairs, and the boundary is the pair of exact rank among them (rank
//   counting on <= kCandCap candidates).
//   Fallback (a boundary bin holds more than kCandCap positions, e.g. massive
//   ties): a 4-pass 8-bit MSB radix select finds T exactly and a ballot pass
//   locates I.
// Both lists are then emitted in ascending order by one writing pass with
// per-warp ballot prefix sums (per-warp counts come from the per-warp
// histograms and the boundary candidates; the fallback adds a counting pass).
// Dispatch (launch_select): rows of up to kRegMaxLen tokens without f1's
// running sums take the register split (select_reg.cuh: 256 x 16, 512 x 16 or
// 512 x 24 positions, five barriers, rare rows to the to-do launch); longer
// rows the long split (select_long.cuh).  The generic split below serves f1.
// Row storage by length: up to kThreads*kRegRow (4096) tokens the row lives in
// registers (16 consecutive positions per thread, bins packed 4 per register,
// SIMD byte compares for the candidate and emission passes, output offsets
// from one block-wide scan); up to kSmemCap tokens it is staged in shared
// memory; longer rows are re-read from global memory (L2-resident across the
// passes).  All reductions use a fixed order.
#include <float.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

#include "select_long.cuh"
#include "select_row.cuh"
#include "select_reg.cuh"

namespace skv {

namespace {
#ifndef SKV_SMEM_CAP
#define SKV_SMEM_CAP 8192
#endif
#ifndef SKV_REG_MAX_LEN
#define SKV_REG_MAX_LEN 12288
#endif
constexpr int kRegMaxLen = SKV_REG_MAX_LEN;   // rows the register split holds (f1: the splits below)
constexpr int kSmemCap = SKV_SMEM_CAP;   // rows staged in shared memory (5 B per token); longer rows read L2 directly
                                 // (measured faster from 16K tokens up: more CTAs per SM)

// grid (B, max_rows): the CTAs of a row are consecutive and the rows past the
// launch's image (idle CTAs) come last.
// Launched with programmatic dependent launch: K1's logits / statistics are
// read only after the previous grid has completed.  The plan kernel that
// follows may be scheduled during this grid's tail; it waits for completion
// before reading anything (and an attend launched right after select runs
// without its overlap flag, include/smallkv.h)
template <bool kInSmem, bool kLogBins, int kRegE>
__global__ void __launch_bounds__(kThreads, kRegE > 0 ? SKV_SELECT_REG_MINB : (kInSmem ? 5 : 4)) select_kernel(const SelectParams p) {
  griddep_launch_dependents();
  griddep_wait();
  const int r = p.layer_off[p.layer_begin] + static_cast<int>(blockIdx.y);
  if (r >= p.layer_off[p.layer_end]) return;
  if constexpr (!kInSmem && kRegE == 0)
    select_row_long<kLogBins>(p, p.rows[r], blockIdx.x);   // rows longer than kSmemCap
  else
    select_row<kInSmem, kLogBins, kRegE>(p, p.rows[r], blockIdx.x);
}

// Rows longer than kSmemCap: the long split (select_long.cuh), kT threads per CTA.
template <bool kLogBins, int kT>
__global__ void __launch_bounds__(kT, kT >= 1024 ? 1 : (kT >= 512 ? 2 : 4)) select_long_kernel(const SelectParams p) {
  griddep_launch_dependents();
  griddep_wait();
  const int r = p.layer_off[p.layer_begin] + static_cast<int>(blockIdx.y);
  if (r >= p.layer_off[p.layer_end]) return;
  select_row_long<kLogBins, kT>(p, p.rows[r], blockIdx.x);
}

#ifndef SKV_SELECT_REGK_MINB
#define SKV_SELECT_REGK_MINB 5
#endif
// Rows of <= 4096 tokens without f1's running sums: the register split
// (select_reg.cuh); the rows it hands over are finished by the to-do launch.
template <bool kLogBins, int kT, int kE>
__global__ void __launch_bounds__(kT, kT == 256 ? SKV_SELECT_REGK_MINB : 2) select_reg_kernel(const SelectParams p) {
  griddep_launch_dependents();
  griddep_wait();
  const int r = p.layer_off[p.layer_begin] + static_cast<int>(blockIdx.y);
  if (r >= p.layer_off[p.layer_end]) return;
  select_row_reg<kLogBins, kT, kE>(p, p.rows[r], blockIdx.x);
}

// ---------------------------------------------------------------------------
// Variant f2 (R16): group score rows and per-head marginal weights.
constexpr int kGroupThreads = 256;

// (m', lse') of SLM row j for sequence b from K1's per-chunk statistics
__device__ __forceinline__ float2 row_lse(const GroupParams& p, int j, int b) {
  const int n = p.seq_lens[b];
  const int nch = (n + p.chunk_tokens - 1) / p.chunk_tokens;
  const float4* st = p.stats + (static_cast<int64_t>(j) * p.batch + b) * p.n_chunks;
  float m = -FLT_MAX, sum = 0.f;
  for (int c = 0; c < nch; ++c) lse_combine(m, sum, st[c].x, st[c].y);
  return make_float2(m, m + logf(sum));
}

// CTA = (layer*H_kv + g, b): F_g[v] = Σ_h exp(s'_{f(l,h)}[v] - lse'_{f(l,h)}) in head
// order, plus (max, 1, min, max over the ranked range) for the split.
__global__ void __launch_bounds__(kGroupThreads) group_score_kernel(const GroupParams p) {
  __shared__ int s_j[8];
  __shared__ float s_lse[8];
  __shared__ float s_mult[8];   // multiplicity of each distinct row (0 for repeats)
  __shared__ float s_red[2][kGroupThreads / 32];
  const int gl = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int l = gl / p.H_kv, g = gl % p.H_kv, G = p.H / p.H_kv;
  if (b == 0 && tid == 0) {
    p.rows[gl] = gl;
    if (gl == 0) {
      p.layer_off[0] = 0;
      p.layer_off[1] = p.L * p.H_kv;
    }
  }
  if (tid < G) {
    const int j = p.head_map[l * p.H + g * G + tid];
    const float2 ml = row_lse(p, j, b);
    s_j[tid] = j;
    s_lse[tid] = ml.y;
    p.slm_lse[(static_cast<int64_t>(j) * p.batch + b) * 2] = ml.x;
    p.slm_lse[(static_cast<int64_t>(j) * p.batch + b) * 2 + 1] = ml.y;
  }
  __syncthreads();
  if (tid < G) {
    // heads sharing a row contribute the same a' row: read it once, weight it by
    // the number of heads (F_g = Σ_h a'_{f(h)} = Σ_distinct j mult_j · a'_j)
    int first = tid;
    for (int h = 0; h < tid; ++h)
      if (s_j[h] == s_j[tid]) {
        first = h;
        break;
      }
    float m = 0.f;
    if (first == tid)
      for (int h = tid; h < G; ++h) m += s_j[h] == s_j[tid] ? 1.f : 0.f;
    s_mult[tid] = m;
  }
  __syncthreads();
  const int n = p.seq_lens[b];
  const int N = n - iclamp(p.n_recent[b], 0, n);
  float* out = p.score + (static_cast<int64_t>(gl) * p.batch + b) * p.row_stride;
  // distinct rows only (first occurrence order), each with its multiplicity
  int nd = 0;
  const float* rowp[8];
  float dm[8], dl[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    rowp[h] = nullptr;
    dm[h] = 0.f;
    dl[h] = 0.f;
  }
  for (int h = 0; h < G; ++h) {
    if (s_mult[h] == 0.f) continue;
#pragma unroll
    for (int d = 0; d < 8; ++d)
      if (d == nd) {
        rowp[d] = p.logits + (static_cast<int64_t>(s_j[h]) * p.batch + b) * p.row_stride;
        dm[d] = s_mult[h];
        dl[d] = s_lse[h];
      }
    ++nd;
  }
  float lo = FLT_MAX, hi = -FLT_MAX;
  // 4 consecutive positions per thread per step, U steps per round: each
  // distinct row's U 16-byte loads are in flight together
  constexpr int U = 4;
  const bool al = (p.row_stride & 3) == 0;
  for (int r0 = 4 * tid; r0 < n; r0 += U * 4 * kGroupThreads) {
    float f[U][4];
#pragma unroll
    for (int it = 0; it < U; ++it) f[it][0] = f[it][1] = f[it][2] = f[it][3] = 0.f;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      if (d >= nd) break;
      float x[U][4];
#pragma unroll
      for (int it = 0; it < U; ++it) {
        const int v0 = r0 + it * 4 * kGroupThreads;
        if (al && v0 + 3 < n) {
          const float4 f4 = __ldg(reinterpret_cast<const float4*>(rowp[d] + v0));
          x[it][0] = f4.x;
          x[it][1] = f4.y;
          x[it][2] = f4.z;
          x[it][3] = f4.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) x[it][u] = v0 + u < n ? __ldg(rowp[d] + v0 + u) : 0.f;
        }
      }
#pragma unroll
      for (int it = 0; it < U; ++it)
#pragma unroll
        for (int u = 0; u < 4; ++u) f[it][u] += dm[d] * __expf(x[it][u] - dl[d]);
    }
#pragma unroll
    for (int it = 0; it < U; ++it) {
      const int v0 = r0 + it * 4 * kGroupThreads;
      if (v0 >= n) break;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + u < N) {
          lo = fminf(lo, f[it][u]);
          hi = fmaxf(hi, f[it][u]);
        }
      if (al && v0 + 3 < n) {
        *reinterpret_cast<float4*>(out + v0) = make_float4(f[it][0], f[it][1], f[it][2], f[it][3]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v0 + u < n) out[v0 + u] = f[it][u];
      }
    }
  }
  lo = -warp_max(-lo);
  hi = warp_max(hi);
  if ((tid & 31) == 0) {
    s_red[0][tid >> 5] = lo;
    s_red[1][tid >> 5] = hi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kGroupThreads / 32; ++w) {
      lo = fminf(lo, s_red[0][w]);
      hi = fmaxf(hi, s_red[1][w]);
    }
    p.gstats[static_cast<int64_t>(gl) * p.batch + b] = make_float4(hi, 1.f, lo, hi);
  }
}

// CTA = (layer*H_kv + g, b): marg_w8[m][h] = a'_{f(l,h)}[marg_idx[m]] (Eq. 6), 0 for h >= G.
__global__ void __launch_bounds__(kGroupThreads) group_weights_kernel(const GroupParams p) {
  __shared__ int s_j[8];
  __shared__ float s_lse[8];
  const int gl = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int l = gl / p.H_kv, g = gl % p.H_kv, G = p.H / p.H_kv;
  if (tid < G) {
    const int j = p.head_map[l * p.H + g * G + tid];
    s_j[tid] = j;
    s_lse[tid] = p.slm_lse[(static_cast<int64_t>(j) * p.batch + b) * 2 + 1];
  }
  __syncthreads();
  const int64_t gb = static_cast<int64_t>(gl) * p.batch + b;
  const int Mc = p.counts[gb * 2 + 1];
  // one marginal entry per thread: its position, then all G rows' logits at once
  for (int m = tid; m < Mc; m += kGroupThreads) {
    const int k = p.marg_idx[gb * p.max_marg + m];
    float x[8];
#pragma unroll
    for (int h = 0; h < 8; ++h)
      x[h] = h < G ? __ldg(p.logits + (static_cast<int64_t>(s_j[h]) * p.batch + b) * p.row_stride + k) : 0.f;
    float4* dst = reinterpret_cast<float4*>(p.marg_w8 + (gb * p.max_marg + m) * 8);
    float w[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) w[h] = h < G ? __expf(x[h] - s_lse[h]) : 0.f;
    dst[0] = make_float4(w[0], w[1], w[2], w[3]);
    dst[1] = make_float4(w[4], w[5], w[6], w[7]);
  }
}
}  // namespace

// overlap_previous: launch with programmatic dependent launch so this grid may
// run alongside the immediately preceding kernel (the next chunk's K1).  The
// caller guarantees that this grid's inputs were complete before that kernel
// started (they come from an earlier launch on the stream).
// tuning knob: SMALLKV_SELECT_REG=generic keeps short rows on select_row's register variant
static bool reg_generic() {
  static const bool g = [] {
    const char* e = getenv("SMALLKV_SELECT_REG");
    return e && e[0] == 'g';
  }();
  return g;
}

cudaError_t launch_select(const SelectParams& p, int32_t max_rows, int32_t max_seq_len,
                          bool overlap_previous, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.batch, max_rows);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = overlap_previous ? 1 : 0;
  cudaError_t e;
  if (max_seq_len <= kRegMaxLen && !p.acc && !reg_generic()) {
    // dynamic shared memory (512-thread rows): the row as loaded, 4 B per position
    auto reg = [&](auto kern, int threads, int per) -> cudaError_t {
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = threads > 256 ? static_cast<size_t>(threads) * per * 4 : 0;
      if (cfg.dynamicSmemBytes) {
        const cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(cfg.dynamicSmemBytes));
        if (r != cudaSuccess) return r;
      }
      return cudaLaunchKernelEx(&cfg, kern, p);
    };
    if (max_seq_len <= 4096)
      e = reg(p.log_bins ? select_reg_kernel<true, 256, 16> : select_reg_kernel<false, 256, 16>, 256, 16);
    else if (max_seq_len <= 8192)
      e = reg(p.log_bins ? select_reg_kernel<true, 512, 16> : select_reg_kernel<false, 512, 16>, 512, 16);
    else
      e = reg(p.log_bins ? select_reg_kernel<true, 512, 24> : select_reg_kernel<false, 512, 24>, 512, 24);
    if (e != cudaSuccess) return e;
    return launch_select_todo(p, s);
  } else if (max_seq_len <= kThreads * kRegRow) {
    e = cudaLaunchKernelEx(&cfg, p.log_bins ? select_kernel<false, true, kRegRow> : select_kernel<false, false, kRegRow>, p);
  } else if (max_seq_len <= kSmemCap) {
    cfg.dynamicSmemBytes = static_cast<size_t>(max_seq_len) * 5 + 16;
    auto k = p.log_bins ? select_kernel<true, true, 0> : select_kernel<true, false, 0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(cfg.dynamicSmemBytes));
    e = cudaLaunchKernelEx(&cfg, k, p);
  } else {
    static const int long_cta = [] {
      const char* v = getenv("SMALLKV_LONG_CTA");   // tuning knob: 256, 512 or 1024
      // 256: measured fastest at configs 3 and 4 (1024 threads, one CTA per
      // SM, reads the row from DRAM once — 4.0 -> 1.46 GB at config 4 — but
      // the CTA's serial phases then idle the SM: 1.13 vs 0.97 ms)
      const int t = v ? atoi(v) : 256;
      return (t == 512 || t == 1024) ? t : 256;
    }();
    cfg.blockDim = dim3(long_cta);
    if (long_cta == 256)
      e = cudaLaunchKernelEx(&cfg, p.log_bins ? select_long_kernel<true, 256> : select_long_kernel<false, 256>, p);
    else if (long_cta == 512)
      e = cudaLaunchKernelEx(&cfg, p.log_bins ? select_long_kernel<true, 512> : select_long_kernel<false, 512>, p);
    else
      e = cudaLaunchKernelEx(&cfg, p.log_bins ? select_long_kernel<true, 1024> : select_long_kernel<false, 1024>, p);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_group_score(const GroupParams& p, cudaStream_t s) {
  group_score_kernel<<<dim3(p.L * p.H_kv, p.batch), kGroupThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_group_weights(const GroupParams& p, cudaStream_t s) {
  group_weights_kernel<<<dim3(p.L * p.H_kv, p.batch), kGroupThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace skv
