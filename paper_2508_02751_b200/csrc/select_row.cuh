// select_row.cuh — K2's per-row split (one 256-thread CTA per row), shared by
// the standalone split (select.cu) and the fused score + split kernel
// (score_select.cu).  Device code only; nothing here is shared with oracle/.
//
// For one SLM row j and sequence b:
//   m' = max_v s'_v, lse' = m' + ln Σ_v exp(s'_v - m')     (A'_{f(i)} normaliser, Eq. 6)
//   recent R' = [n-R', n); positions [0, n-R') ranked by (s' desc, v asc);
//   critical = rank < K' (Eq. 6 TopK), marginal = K' <= rank < K'+M' (Top(P-K), R4).
// The algorithm is described at the top of select.cu.
#pragma once

#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace skv {
namespace {
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 256;
constexpr int kCandCap = 1024;
constexpr int kRegRow = 16;     // rows up to kThreads * 16 tokens are held in registers

__device__ __forceinline__ int iclamp(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }
// 0xff in byte k iff k < r (r positions left in a 4-position word; r <= 0: none)
__device__ __forceinline__ uint32_t valid_bytes(int r) {
  return r >= 4 ? 0xffffffffu : (r <= 0 ? 0u : (1u << (8 * r)) - 1u);
}
// byte mask (0x00 / 0xff per byte) -> 4-bit mask
__device__ __forceinline__ uint32_t bytes_to_bits(uint32_t x) { return ((x & 0x08040201u) * 0x01010101u) >> 24; }

// deterministic combine of per-thread (max, Σexp) pairs
__device__ __forceinline__ void lse_combine(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  s = s * __expf(m - mm) + s2 * __expf(m2 - mm);
  m = mm;
}

// kRegE > 0 (rows of <= kThreads * kRegE tokens): each thread holds positions
// [kRegE*tid, kRegE*tid + kRegE) of the row in registers for the histogram,
// candidate and emission passes (no staging, no per-warp segments: output
// offsets come from one block-wide scan); the rare refinement / radix paths
// re-read the row from global memory (L2).
#ifndef SKV_SELECT_REG_MINB
#define SKV_SELECT_REG_MINB 5
#endif
template <bool kInSmem, bool kLogBins, int kRegE>
__device__ __forceinline__ void select_row(const SelectParams& p, const int j, const int b) {
  constexpr bool kRegs = kRegE > 0;
  static_assert(!(kRegs && kInSmem), "register rows read the rare paths from global memory");
  extern __shared__ __align__(16) float vals[];   // [n] row, then (kInSmem) [n] bin bytes (+16)
  __shared__ uint32_t hist[kWarps][kBins];
  __shared__ unsigned long long cand[2][kCandCap];
  __shared__ float red[4][kWarps];
  __shared__ int wcnt[kWarps][2];
  __shared__ int wsel[kWarps][2];
  __shared__ int s_have_counts;
  __shared__ int s_bin[2], s_above[2], s_nc[2], s_fallback;
  __shared__ int s_refine[2], s_sub[2];
  __shared__ uint32_t s_tk[2];
  __shared__ int s_ti[2];
  __shared__ uint32_t s_pref[2];
  __shared__ int s_rem[2];

  const int n = p.seq_lens[b];
  const int64_t rb = static_cast<int64_t>(j) * p.batch + b;
  const float* row = p.logits + rb * p.row_stride;
  const int Rc = iclamp(p.n_recent[b], 0, n);
  const int Kc = min(iclamp(p.k_crit[b], 0, n - Rc), p.max_crit);
  const int Mc = min(iclamp(p.k_marg[b], 0, n - Rc - Kc), p.max_marg);
  const int N = n - Rc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lt = lanemask_lt();
  // the ranking score: the logit (R1) or, for variant f1, the running column
  // sum acc (Eq. 1) updated below
  float* accrow = p.acc ? p.acc + rb * p.row_stride : nullptr;
  const float* score = accrow ? accrow : row;
  auto VAL = [&](int i) -> float { return kInSmem ? vals[i] : score[i]; };
  // positions i..i+3 (i a multiple of 4): shared memory, or global memory with
  // one 16-byte load when the row is 16-byte aligned (long rows)
  const bool g_al = (p.row_stride & 3) == 0;
  auto LOAD4 = [&](int i) -> float4 {
    if (kInSmem) return *reinterpret_cast<const float4*>(vals + i);
    // (plain loads, not the read-only path: the f1 scores were written by this kernel)
    if (g_al) return *reinterpret_cast<const float4*>(score + i);
    return make_float4(score[i], score[i + 1], score[i + 2], score[i + 3]);
  };

  float x[kRegs ? kRegE : 1];
  uint32_t pbin[kRegs ? kRegE / 4 : 1];
  const int i0 = kRegs ? kRegE * tid : 0;
  if (kRegs && !accrow) {
#pragma unroll
    for (int q = 0; q < (kRegs ? kRegE / 4 : 0); ++q) {
      const int i = i0 + 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g_al && i + 3 < n) {
        v = *reinterpret_cast<const float4*>(row + i);
      } else {
        if (i < n) v.x = row[i];
        if (i + 1 < n) v.y = row[i + 1];
        if (i + 2 < n) v.z = row[i + 2];
        if (i + 3 < n) v.w = row[i + 3];
      }
      x[4 * q] = v.x;
      x[4 * q + 1] = v.y;
      x[4 * q + 2] = v.z;
      x[4 * q + 3] = v.w;
    }
  }
  // ---- pass 1: stage the row; (max, Σexp) over [0, n) and the ranked range
  // [min, max] over [0, N) are merged from K1's per-chunk statistics (fixed order)
  if (kInSmem && !accrow) {
    // all copies in flight at once (one memory round trip for the row)
    if ((p.row_stride & 3) == 0) {
      const int n4 = n >> 2;
      for (int i = tid; i < n4; i += kThreads) cp_async16(smem_u32(vals + 4 * i), row + 4 * i, true);
      for (int i = 4 * n4 + tid; i < n; i += kThreads) cp_async4(smem_u32(vals + i), row + i);
    } else {
      for (int i = tid; i < n; i += kThreads) cp_async4(smem_u32(vals + i), row + i);
    }
    cp_async_commit();
  }
  if (warp == 0) {
    const int nch = (n + p.chunk_tokens - 1) / p.chunk_tokens;
    const float4* st = p.stats + rb * p.n_chunks;
    float m2 = -FLT_MAX, s2 = 0.f, l2 = FLT_MAX, h2 = -FLT_MAX;
    for (int c = lane; c < nch; c += 32) {
      const float4 v = st[c];
      lse_combine(m2, s2, v.x, v.y);
      l2 = fminf(l2, v.z);
      h2 = fmaxf(h2, v.w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lse_combine(m2, s2, __shfl_xor_sync(0xffffffffu, m2, o), __shfl_xor_sync(0xffffffffu, s2, o));
      l2 = fminf(l2, __shfl_xor_sync(0xffffffffu, l2, o));
      h2 = fmaxf(h2, __shfl_xor_sync(0xffffffffu, h2, o));
    }
    if (lane == 0) {
      red[0][0] = m2;
      red[1][0] = s2;
      red[2][0] = l2;
      red[3][0] = h2;
      p.lse[rb * 2] = m2;
      p.lse[rb * 2 + 1] = m2 + logf(s2);
      p.counts[rb * 2] = Kc;
      p.counts[rb * 2 + 1] = Mc;
    }
  }
  if (kInSmem && !accrow) cp_async_wait<0>();
  __syncthreads();
  const float lse = red[0][0] + logf(red[1][0]);
  float vlo = red[2][0], vhi = red[3][0];
  if (accrow) {
    // f1: acc[v] += a'_v for v < n (in place), rank on acc; range over [0, N)
    float lo = FLT_MAX, hi = -FLT_MAX;
    if (kRegs) {
#pragma unroll
      for (int e = 0; e < (kRegs ? kRegE : 0); ++e) {
        const int i = i0 + e;
        if (i < n) {
          const float v = accrow[i] + __expf(row[i] - lse);
          accrow[i] = v;
          x[e] = v;
          if (i < N) {
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
          }
        }
      }
    }
    for (int i = kRegs ? n : tid; i < n; i += kThreads) {
      const float v = accrow[i] + __expf(row[i] - lse);
      accrow[i] = v;
      if (kInSmem) vals[i] = v;
      if (i < N) {
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
      }
    }
    lo = -warp_max(-lo);
    hi = warp_max(hi);
    __syncthreads();
    if (lane == 0) {
      red[2][warp] = lo;
      red[3][warp] = hi;
    }
    __syncthreads();
    vlo = FLT_MAX;
    vhi = -FLT_MAX;
    for (int w = 0; w < kWarps; ++w) {
      vlo = fminf(vlo, red[2][w]);
      vhi = fmaxf(vhi, red[3][w]);
    }
  }
  const int rA = Kc, rB = Kc + Mc;
  if (rB == 0) return;

  // per-warp contiguous segments of [0, N) (index order = output order)
  // (multiples of 128 positions: the shared-memory passes give each lane 4
  // consecutive positions per step)
  const int seg = ((N + kWarps * 128 - 1) / (kWarps * 128)) * 128;
  const int s0 = warp * seg, s1 = min(N, s0 + seg);

  // ---- boundaries as lexicographic thresholds (T, I)
  // Histogram coordinate: the score itself, or (variant f2's group scores —
  // sums of probabilities, heavily skewed towards 0) its logarithm.  Either is
  // monotone, so bins stay ordered like scores; exactness comes from the keys.
  // (log coordinate: the bit pattern of a positive float, a monotone piecewise-
  // linear log2 — integer conversion instead of a full-precision logf)
  auto bv = [&](float v) {
    return kLogBins ? static_cast<float>(__float_as_uint(fmaxf(v, 1e-30f))) : v;
  };
  const float blo = bv(vlo);
  const float scale = 255.99f / (bv(vhi) - blo);
  const bool all_equal = !(vhi > vlo);
  if (tid == 0) {
    s_fallback = (!all_equal && !isfinite(scale)) ? 1 : 0;
    s_have_counts = 0;
    s_refine[0] = s_refine[1] = 0;
  }
  __syncthreads();
  if (all_equal) {
    // every ranked score ties: the lowest indices win
    if (tid < 2) {
      const int rr = tid == 0 ? rA : rB;
      s_tk[tid] = rr > 0 ? desc_key(vlo) : 0u;
      s_ti[tid] = rr - 1;
    }
  } else if (!s_fallback) {
    for (int i = tid; i < kWarps * kBins; i += kThreads) (&hist[0][0])[i] = 0u;
    __syncthreads();
    uint8_t* sbin = reinterpret_cast<uint8_t*>(vals + n);
    if (kRegs) {
#pragma unroll
      for (int q = 0; q < (kRegs ? kRegE / 4 : 0); ++q) {
        uint32_t packed = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int bin = iclamp(static_cast<int>((bv(x[4 * q + k]) - blo) * scale), 0, kBins - 1);
          packed |= static_cast<uint32_t>(bin) << (8 * k);
          if (i0 + 4 * q + k < N) atomicAdd(&hist[warp][bin], 1u);
        }
        pbin[q] = packed;
      }
    } else if (kInSmem) {
      // 4 consecutive positions per lane: one 16-B load, one 4-B bin store
      for (int base = s0 + 4 * lane; base < s1; base += 128) {
        const float4 v4 = *reinterpret_cast<const float4*>(vals + base);
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
        uint32_t packed = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int bin = iclamp(static_cast<int>((bv(vv[k]) - blo) * scale), 0, kBins - 1);
          packed |= static_cast<uint32_t>(bin & 255) << (8 * k);
          if (base + k < s1) atomicAdd(&hist[warp][bin], 1u);
        }
        *reinterpret_cast<uint32_t*>(sbin + base) = packed;
      }
    } else {
      // long rows, read from global memory (L2): 4 positions per lane, 2 x 16 B in flight
      for (int base = s0 + 4 * lane; base < s1; base += 256) {
        float4 v4[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) v4[q] = base + 128 * q < s1 ? LOAD4(base + 128 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float vv[4] = {v4[q].x, v4[q].y, v4[q].z, v4[q].w};
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (base + 128 * q + k < s1)
              atomicAdd(&hist[warp][iclamp(static_cast<int>((bv(vv[k]) - blo) * scale), 0, kBins - 1)], 1u);
        }
      }
    }
    __syncthreads();
    if (warp < 2 && (warp == 0 ? rA > 0 : true)) {
      // bins from the top: lane covers bins 255-8*lane .. 248-8*lane
      const int rr = warp == 0 ? rA : rB;
      int c[8], tot = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int bin = kBins - 1 - (lane * 8 + q);
        int v = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) v += static_cast<int>(hist[w][bin]);
        c[q] = v;
        tot += v;
      }
      int incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int above = incl - tot;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (above < rr && rr <= above + c[q]) {
          s_bin[warp] = kBins - 1 - (lane * 8 + q);
          s_above[warp] = above;
          s_nc[warp] = c[q];
          s_refine[warp] = c[q] > kCandCap ? 1 : 0;   // refine inside the bin (long rows)
        }
        above += c[q];
      }
    }
    __syncthreads();
    // Second level for an overfull boundary bin (long rows): 256 value-linear
    // sub-bins inside it; the boundary becomes (bin, sub-bin) and only that
    // sub-bin's positions are candidates.  (Per-warp output counts are then
    // recounted before the emission.)  Still overfull: radix fallback.
    const bool refine = s_refine[0] | s_refine[1];
    auto sub_of = [&](int t, float v) {
      return iclamp(static_cast<int>((bv(v) - (blo + static_cast<float>(s_bin[t]) / scale)) * (scale * 256.f)),
                    0, kBins - 1);
    };
    auto bin_of = [&](float v) { return iclamp(static_cast<int>((bv(v) - blo) * scale), 0, kBins - 1); };
    if (refine && !s_fallback) {
      for (int i = tid; i < 2 * kBins; i += kThreads) (&hist[0][0])[i] = 0u;
      __syncthreads();
      for (int i4 = 4 * tid; i4 < N; i4 += 4 * kThreads) {
        const float4 v4 = LOAD4(i4);
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (i4 + k >= N) break;
          const int bin = bin_of(vv[k]);
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (s_refine[t] && bin == s_bin[t]) atomicAdd(&hist[t][sub_of(t, vv[k])], 1u);
        }
      }
      __syncthreads();
      if (warp < 2 && s_refine[warp]) {
        const int rem = (warp == 0 ? rA : rB) - s_above[warp];
        int c[8], tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          c[q] = static_cast<int>(hist[warp][kBins - 1 - (lane * 8 + q)]);
          tot += c[q];
        }
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        int above = incl - tot;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (above < rem && rem <= above + c[q]) {
            s_sub[warp] = kBins - 1 - (lane * 8 + q);
            s_above[warp] += above;
            s_nc[warp] = c[q];
            if (c[q] > kCandCap) s_fallback = 1;
          }
          above += c[q];
        }
      }
      __syncthreads();
    }
    if (!s_fallback) {
      const int binA = rA > 0 ? s_bin[0] : -1, binB = s_bin[1];
      const bool shared = binA == binB && !refine;
      __shared__ int s_cnt[2];
      if (tid < 2) s_cnt[tid] = 0;
      __syncthreads();
      const uint8_t* sbin = reinterpret_cast<const uint8_t*>(vals + n);
      auto take = [&](int i, int bin, float v) {
        const unsigned long long kv =
            (static_cast<unsigned long long>(desc_key(v)) << 32) | static_cast<uint32_t>(i);
        if (bin == binA && (!s_refine[0] || sub_of(0, v) == s_sub[0]))
          cand[0][atomicAdd(&s_cnt[0], 1)] = kv;
        if (bin == binB && !shared && (!s_refine[1] || sub_of(1, v) == s_sub[1]))
          cand[1][atomicAdd(&s_cnt[1], 1)] = kv;
      };
      if (kRegs) {
        // SIMD byte compares of the packed bins, 4 positions per instruction
        const uint32_t pa = binA >= 0 ? static_cast<uint32_t>(binA) * 0x01010101u : 0u;
        const uint32_t pb = static_cast<uint32_t>(binB) * 0x01010101u;
#pragma unroll
        for (int q = 0; q < (kRegs ? kRegE / 4 : 0); ++q) {
          uint32_t hit = __vcmpeq4(pbin[q], pb);
          if (binA >= 0) hit |= __vcmpeq4(pbin[q], pa);
          hit = bytes_to_bits(hit & valid_bytes(N - (i0 + 4 * q)));
          if (hit) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if ((hit >> k) & 1u)
                take(i0 + 4 * q + k, static_cast<int>((pbin[q] >> (8 * k)) & 0xffu), x[4 * q + k]);
          }
        }
      } else if (kInSmem) {
        // 4 bin bytes per load; SIMD byte compares skip words without a boundary bin
        const uint32_t pa = binA >= 0 ? static_cast<uint32_t>(binA) * 0x01010101u : 0u;
        const uint32_t pb = static_cast<uint32_t>(binB) * 0x01010101u;
        for (int i4 = 4 * tid; i4 < N; i4 += 4 * kThreads) {
          const uint32_t w = *reinterpret_cast<const uint32_t*>(sbin + i4);
          uint32_t hit = __vcmpeq4(w, pb);
          if (binA >= 0) hit |= __vcmpeq4(w, pa);
          if (hit == 0u) continue;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (((hit >> (8 * k)) & 0xffu) && i4 + k < N) take(i4 + k, static_cast<int>((w >> (8 * k)) & 0xffu), VAL(i4 + k));
        }
      } else {
        for (int i4 = 4 * tid; i4 < N; i4 += 4 * kThreads) {
          const float4 v4 = LOAD4(i4);
          const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (i4 + k >= N) break;
            const int bin = iclamp(static_cast<int>((bv(vv[k]) - blo) * scale), 0, kBins - 1);
            if (bin == binA || bin == binB) take(i4 + k, bin, vv[k]);
          }
        }
      }
      __syncthreads();
      // the pair of exact rank (rem - 1) among a bin's candidates (all distinct)
      for (int t = 0; t < 2; ++t) {
        const int rr = t == 0 ? rA : rB;
        if (rr == 0) continue;
        const int li = (t == 1 && shared) ? 0 : t;
        const int nc = s_cnt[li];
        const int want = rr - s_above[t] - 1;
        for (int c = tid; c < nc; c += kThreads) {
          const unsigned long long v = cand[li][c];
          int rank = 0;
          for (int d = 0; d < nc; ++d) rank += cand[li][d] < v ? 1 : 0;
          if (rank == want) {
            s_tk[t] = static_cast<uint32_t>(v >> 32);
            s_ti[t] = static_cast<int>(v & 0xffffffffu);
          }
        }
      }
      if (tid == 0 && rA == 0) {
        s_tk[0] = 0u;
        s_ti[0] = -1;
      }
      // per-warp output counts straight from the per-warp histograms plus the
      // selected candidates of each warp's segment (no counting pass)
      if (tid < 2 * kWarps) (&wsel[0][0])[tid] = 0;
      __syncthreads();
      for (int t = 0; t < (kRegs ? 0 : 2); ++t) {
        const int rr = t == 0 ? rA : rB;
        if (rr == 0) continue;
        const int li = (t == 1 && shared) ? 0 : t;
        const unsigned long long thr =
            (static_cast<unsigned long long>(s_tk[t]) << 32) | static_cast<uint32_t>(s_ti[t]);
        for (int c = tid; c < s_cnt[li]; c += kThreads) {
          const unsigned long long v = cand[li][c];
          if (v <= thr) atomicAdd(&wsel[static_cast<int>(v & 0xffffffffu) / seg][t], 1);
        }
      }
      if (!refine && !kRegs) {   // (after a refinement the per-warp histograms are gone: recount)
        int ab[2] = {0, 0};
        for (int t = 0; t < 2; ++t) {
          const int bt_ = (t == 0 && rA == 0) ? kBins : s_bin[t];
          int a = 0;
          for (int bin = bt_ + 1 + lane; bin < kBins; bin += 32) a += static_cast<int>(hist[warp][bin]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          ab[t] = a;
        }
        __syncthreads();
        if (lane == 0) {
          const int cw = ab[0] + wsel[warp][0];
          wcnt[warp][0] = cw;
          wcnt[warp][1] = ab[1] + wsel[warp][1] - cw;
        }
        if (tid == 0) s_have_counts = 1;
      }
    }
  }
  __syncthreads();
  if (s_fallback) {
    // ---- 4-pass 8-bit MSB radix select of the exact keys, then the tie index
    uint32_t(*rh)[256] = reinterpret_cast<uint32_t(*)[256]>(&hist[0][0]);
    uint32_t pref0 = 0, pref1 = 0;
    int rem0 = rA, rem1 = rB;
    const bool act0 = rA > 0;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      const uint32_t hmask = pass == 0 ? 0u : (0xffffffffu << (shift + 8));
      const bool same = act0 && pref0 == pref1;
      for (int i = tid; i < 512; i += kThreads) rh[i >> 8][i & 255] = 0;
      __syncthreads();
      for (int base = warp * 32; base < N; base += kThreads) {
        const int i = base + lane;
        const bool valid = i < N;
        const uint32_t k = valid ? desc_key(VAL(i)) : 0u;
        const uint32_t dig = (k >> shift) & 255u;
        const bool in0 = valid && act0 && (k & hmask) == pref0;
        const bool in1 = valid && !same && (k & hmask) == pref1;
        const uint32_t g0 = __match_any_sync(0xffffffffu, in0 ? dig : 0x100u);
        if (in0 && lane == __ffs(g0) - 1) atomicAdd(&rh[0][dig], __popc(g0));
        const uint32_t g1 = __match_any_sync(0xffffffffu, in1 ? dig : 0x100u);
        if (in1 && lane == __ffs(g1) - 1) atomicAdd(&rh[1][dig], __popc(g1));
      }
      __syncthreads();
      if (warp < 2 && (warp == 0 ? act0 : true)) {
        const uint32_t* h = (warp == 1 && same) ? rh[0] : rh[warp];
        const int rem = warp == 0 ? rem0 : rem1;
        int c[8], tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          c[q] = static_cast<int>(h[lane * 8 + q]);
          tot += c[q];
        }
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        int before = incl - tot;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (before < rem && rem <= before + c[q]) {
            s_pref[warp] = (warp == 0 ? pref0 : pref1) | (static_cast<uint32_t>(lane * 8 + q) << shift);
            s_rem[warp] = rem - before;
          }
          before += c[q];
        }
      }
      __syncthreads();
      if (act0) {
        pref0 = s_pref[0];
        rem0 = s_rem[0];
      }
      pref1 = s_pref[1];
      rem1 = s_rem[1];
      __syncthreads();
    }
    // index of the take-th (1-based) position whose key equals T, per target
    for (int t = 0; t < 2; ++t) {
      const int rr = t == 0 ? rA : rB;
      if (rr == 0) {
        if (tid == 0) {
          s_tk[0] = 0u;
          s_ti[0] = -1;
        }
        continue;
      }
      const uint32_t T = t == 0 ? pref0 : pref1;
      const int take = t == 0 ? rem0 : rem1;
      int eq = 0;
      for (int base = s0; base < s1; base += 32) {
        const int i = base + lane;
        eq += __popc(__ballot_sync(0xffffffffu, i < s1 && desc_key(VAL(i)) == T));
      }
      if (lane == 0) wcnt[warp][0] = eq;
      __syncthreads();
      int before = 0;
      for (int w = 0; w < warp; ++w) before += wcnt[w][0];
      if (before < take && take <= before + eq) {
        for (int base = s0; base < s1; base += 32) {
          const int i = base + lane;
          const uint32_t bal = __ballot_sync(0xffffffffu, i < s1 && desc_key(VAL(i)) == T);
          const int k = take - before;   // 1-based within this warp's remaining ties
          if (k >= 1 && k <= __popc(bal)) {
            if (lane == 0) {
              uint32_t m = bal;
              for (int q = 1; q < k; ++q) m &= m - 1;
              s_tk[t] = T;
              s_ti[t] = base + __ffs(m) - 1;
            }
            break;
          }
          before += __popc(bal);
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();

  // ---- emission: (count per warp segment if not known,) write ascending lists.
  // Thresholds compared as floats: key < T  <=>  x > key_to_float(T) (with -0 == +0).
  const float XA = key_to_float(s_tk[0]), XB = key_to_float(s_tk[1]);
  const int IA = s_ti[0], IB = s_ti[1];
  // per-lane classification of positions i..i+3 (shared-memory path)
  auto classify4 = [&](int i, uint32_t& cm, uint32_t& mm, float (&xs)[4]) {
    const float4 v4 = i < s1 ? LOAD4(i) : make_float4(0.f, 0.f, 0.f, 0.f);
    xs[0] = v4.x;
    xs[1] = v4.y;
    xs[2] = v4.z;
    xs[3] = v4.w;
    cm = 0u;
    mm = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ik = i + k;
      const bool valid = ik < s1;
      const bool isC = valid && (xs[k] > XA || (xs[k] == XA && ik <= IA));
      const bool inB = valid && (xs[k] > XB || (xs[k] == XB && ik <= IB));
      cm |= static_cast<uint32_t>(isC) << k;
      mm |= static_cast<uint32_t>(inB && !isC) << k;
    }
  };
  int32_t* crit = p.crit_idx + rb * p.max_crit;
  int32_t* marg = p.marg_idx + rb * p.max_marg;
  float* mw = p.marg_w + rb * p.max_marg;
  if constexpr (kRegs) {
    // register rows: per-thread masks, one block-wide exclusive scan of the
    // packed (critical | marginal << 16) counts, then each thread writes its
    // positions in ascending order
    // Positions in bins strictly above / below a boundary bin are decided by
    // their bin (bins are monotone in the score and each threshold lies in its
    // boundary bin); boundary-bin positions, and rows without bins (all ties,
    // radix fallback), compare exactly.
    const bool use_bins = !all_equal && !s_fallback;
    const uint32_t ea = rA > 0 && use_bins ? static_cast<uint32_t>(s_bin[0]) * 0x01010101u : 0u;
    const uint32_t eb = use_bins ? static_cast<uint32_t>(s_bin[1]) * 0x01010101u : 0u;
    uint32_t cm = 0u, bsel = 0u;
#pragma unroll
    for (int q = 0; q < kRegE / 4; ++q) {
      const uint32_t vm = valid_bytes(N - (i0 + 4 * q));
      uint32_t c4 = 0u, b4 = 0u, ex = bytes_to_bits(vm);
      if (use_bins) {
        if (rA > 0) c4 = bytes_to_bits(__vcmpgtu4(pbin[q], ea) & vm);
        b4 = bytes_to_bits(__vcmpgtu4(pbin[q], eb) & vm);
        ex = bytes_to_bits(((rA > 0 ? __vcmpeq4(pbin[q], ea) : 0u) | __vcmpeq4(pbin[q], eb)) & vm);
      }
      if (ex) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if ((ex >> k) & 1u) {
            const int i = i0 + 4 * q + k;
            const float v = x[4 * q + k];
            const uint32_t isC = ((v > XA) | ((v == XA) & (i <= IA))) ? 1u : 0u;
            const uint32_t inB = ((v > XB) | ((v == XB) & (i <= IB))) ? 1u : 0u;
            c4 = (c4 & ~(1u << k)) | (isC << k);
            b4 = (b4 & ~(1u << k)) | (inB << k);
          }
        }
      }
      cm |= c4 << (4 * q);
      bsel |= b4 << (4 * q);
    }
    const uint32_t mm = bsel & ~cm;
    const int own = __popc(cm) | (__popc(mm) << 16);
    int incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wcnt[warp][0] = incl;
    __syncthreads();
    int ex = incl - own;
    for (int w = 0; w < warp; ++w) ex += wcnt[w][0];
    int ac = ex & 0xffff, am = ex >> 16;
    // ascending set bits; a' re-read from the logits row (L1 / L2 hit: this
    // thread loaded it; for f1 the logit is not the ranking value anyway)
    for (uint32_t m = cm; m; m &= m - 1u) crit[ac++] = i0 + __ffs(m) - 1;
    for (uint32_t m = mm; m; m &= m - 1u) {
      const int i = i0 + __ffs(m) - 1;
      marg[am] = i;
      mw[am] = __expf(row[i] - lse);   // a' of the current step (Eq. 6)
      ++am;
    }
    return;
  }
  if (!s_have_counts) {
    int cc = 0, cb = 0;
    for (int base = s0 + 4 * lane; base < s1; base += 128) {
      uint32_t cm, mm;
      float xs[4];
      classify4(base, cm, mm, xs);
      cc += __popc(cm);
      cb += __popc(mm);
    }
    cc = warp_sum_i(cc);
    cb = warp_sum_i(cb);
    if (lane == 0) {
      wcnt[warp][0] = cc;
      wcnt[warp][1] = cb;
    }
    __syncthreads();
  }
  int oc = 0, om = 0;
  for (int w = 0; w < warp; ++w) {
    oc += wcnt[w][0];
    om += wcnt[w][1];
  }
  // 128 positions per warp step: per-lane masks, one packed warp scan
  for (int base0 = s0; base0 < s1; base0 += 128) {
    const int base = base0 + 4 * lane;
    uint32_t cm, mm;
    float xs[4];
    classify4(base, cm, mm, xs);
    const int own = __popc(cm) | (__popc(mm) << 16);
    int incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int ac = oc + ((incl - own) & 0xffff), am = om + ((incl - own) >> 16);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if ((cm >> k) & 1u) crit[ac++] = base + k;
      if ((mm >> k) & 1u) {
        marg[am] = base + k;
        mw[am] = __expf((accrow ? row[base + k] : xs[k]) - lse);   // a' of the current step (Eq. 6)
        ++am;
      }
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    oc += tot & 0xffff;
    om += tot >> 16;
  }
}

}  // namespace
}  // namespace skv
