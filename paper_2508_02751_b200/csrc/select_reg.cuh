// select_reg.cuh — K2's split of SHORT rows (n <= 12288 tokens: the 4K and 8K
// contexts) with the row held in registers: one CTA per (SLM row, sequence),
// kRegE consecutive positions per thread (256 x 16 up to 4096 tokens, 512 x 16
// up to 8192, 512 x 24 up to 12288).
//
// Same result as select_row (select_row.cuh; Eq. 4, Eq. 6
// P:141-152, R1-R5, R10; f2's log-coordinate bins, R16): exact lexicographic
// ranking by (order-preserving key, index), ascending lists, marg_w = a' of
// the current step.  Built for the fewest block barriers (five), because at
// 4K tokens a row is ~1 us of work and the barriers, not the arithmetic, set
// its latency:
//   1. zero the per-warp histograms, load the row, merge K1's chunk
//      statistics (lse', ranked range [lo, hi])                    | barrier
//   2. 256 bins linear in the score (monotone), packed 4 per register  | barrier
//   3. warps 0 / 1: suffix scan -> each boundary's bin and the count above it
//                                                                     | barrier
//   4. the boundary bins' (key, index) pairs -> shared lists          | barrier
//   5. each thread classifies its positions: by bin above / below a boundary
//      bin, by exact rank among that bin's pairs inside it (no threshold
//      broadcast); one block-wide scan of the packed counts      | barrier
//   6. each thread writes its positions (ascending) at its offsets.
// Rows this path does not take — f1's running sums (they are updated in
// place, select_row), all-equal or non-finite score ranges, a boundary bin
// with more than kRegCap positions — go to the to-do list that the long split
// (select_long.cuh) finishes in the launch right after (usually empty).
#pragma once

#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace skv {
namespace {
constexpr int kRegBins = 256;
constexpr int kRankDirect = 48;   // boundary lists up to this long: ranks counted per position

__device__ __forceinline__ int rclamp(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }
// 0xff in byte k iff k < r (r positions left in a 4-position word; r <= 0: none)
__device__ __forceinline__ uint32_t rvalid_bytes(int r) {
  return r >= 4 ? 0xffffffffu : (r <= 0 ? 0u : (1u << (8 * r)) - 1u);
}
// byte mask (0x00 / 0xff per byte) -> 4-bit mask
__device__ __forceinline__ uint32_t rbytes_to_bits(uint32_t x) { return ((x & 0x08040201u) * 0x01010101u) >> 24; }
// The want-th smallest (0-based) of n distinct u64 in shared memory, by one
// warp: MSB-first 8-bit radix select (h: a 256-word shared histogram of the
// warp's own).  All lanes return it.
__device__ __forceinline__ unsigned long long warp_select_u64(const unsigned long long* lst, int n, int want,
                                                              uint32_t* h, int lane) {
  unsigned long long prefix = 0ull, mask = 0ull;
  int rem = want;
  for (int shift = 56; shift >= 0; shift -= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) h[lane * 8 + q] = 0u;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const unsigned long long v = lst[i];
      if ((v & mask) == prefix) atomicAdd(&h[static_cast<int>((v >> shift) & 255ull)], 1u);
    }
    __syncwarp();
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
    int run = incl - tot, dig = -1, below = 0, cnt = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (rem >= run && rem < run + c[q]) {
        dig = lane * 8 + q;
        below = run;
        cnt = c[q];
      }
      run += c[q];
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, dig >= 0)) - 1;
    dig = __shfl_sync(0xffffffffu, dig, src);
    below = __shfl_sync(0xffffffffu, below, src);
    cnt = __shfl_sync(0xffffffffu, cnt, src);
    prefix |= static_cast<unsigned long long>(dig) << shift;
    mask |= 255ull << shift;
    rem -= below;
    __syncwarp();
    if (cnt == 1) break;   // one value left with this prefix
  }
  if (mask == ~0ull) return prefix;
  unsigned long long found = 0ull;
  bool hit = false;
  for (int i = lane; i < n; i += 32) {
    const unsigned long long v = lst[i];
    if ((v & mask) == prefix) {
      found = v;
      hit = true;
    }
  }
  const int src = __ffs(__ballot_sync(0xffffffffu, hit)) - 1;
  return __shfl_sync(0xffffffffu, found, src < 0 ? 0 : src);
}

__device__ __forceinline__ void rlse_combine(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  s = s * __expf(m - mm) + s2 * __expf(m2 - mm);
  m = mm;
}

// kRegThreads threads x kRegE positions per thread (rows up to their product)
template <bool kLogBins, int kRegThreads, int kRegE>
__device__ __forceinline__ void select_row_reg(const SelectParams& p, const int j, const int b) {
  constexpr int kRegWarps = kRegThreads / 32;
  constexpr int kRegCap = kRegThreads * kRegE / 16;   // boundary-bin pairs held per boundary
  constexpr bool kSmemRow = kRegThreads > 256;          // the row kept in (dynamic) shared memory
  static_assert(kRegE % 4 == 0 && kRegE <= 32, "16-bit packed counts, 32-bit masks");
  __shared__ __align__(16) uint32_t hist[kRegWarps][kRegBins];
  __shared__ unsigned long long cand[2][kRegCap];
  __shared__ float red[4];
  __shared__ int s_cnt[2], s_bin[2], s_above[2], s_nc[2];
  __shared__ int wtot[kRegWarps];
  extern __shared__ __align__(16) float s_row[];   // [kRegThreads * kRegE] the row as loaded (kSmemRow)

  const int n = p.seq_lens[b];
  const int64_t rb = static_cast<int64_t>(j) * p.batch + b;
  const float* row = p.logits + rb * p.row_stride;
  const int Rc = rclamp(p.n_recent[b], 0, n);
  const int Kc = min(rclamp(p.k_crit[b], 0, n - Rc), p.max_crit);
  const int Mc = min(rclamp(p.k_marg[b], 0, n - Rc - Kc), p.max_marg);
  const int N = n - Rc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = kRegE * tid;

  // ---- 1. histograms zeroed, the row in registers, the row statistics
  {
    uint4* h4 = reinterpret_cast<uint4*>(&hist[0][0]);
#pragma unroll
    for (int i = tid; i < kRegWarps * kRegBins / 4; i += kRegThreads) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (tid < 2) s_cnt[tid] = 0;
  float x[kRegE];
  const bool al = (p.row_stride & 3) == 0;
#pragma unroll
  for (int q = 0; q < kRegE / 4; ++q) {
    const int i = i0 + 4 * q;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (al && i + 3 < n) {
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
    // (512-thread rows: a copy in shared memory for the positions read back
    // later — boundary-bin pairs, marginal weights — instead of an L2 round
    // trip each; measured +2.7% at config 5, -0.5% at config 2's 256 threads)
    if (kSmemRow) *reinterpret_cast<float4*>(s_row + i) = v;
  }
  if (warp == 0) {
    // (max, Σexp) over [0, n) and [min, max] over [0, N) from K1's per-chunk
    // statistics, merged in a fixed order
    const int nch = (n + p.chunk_tokens - 1) / p.chunk_tokens;
    const float4* st = p.stats + rb * p.n_chunks;
    float m2 = -FLT_MAX, s2 = 0.f, l2 = FLT_MAX, h2 = -FLT_MAX;
    for (int c = lane; c < nch; c += 32) {
      const float4 v = st[c];
      rlse_combine(m2, s2, v.x, v.y);
      l2 = fminf(l2, v.z);
      h2 = fmaxf(h2, v.w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      rlse_combine(m2, s2, __shfl_xor_sync(0xffffffffu, m2, o), __shfl_xor_sync(0xffffffffu, s2, o));
      l2 = fminf(l2, __shfl_xor_sync(0xffffffffu, l2, o));
      h2 = fmaxf(h2, __shfl_xor_sync(0xffffffffu, h2, o));
    }
    if (lane == 0) {
      red[0] = m2;
      red[1] = s2;
      red[2] = l2;
      red[3] = h2;
      p.lse[rb * 2] = m2;
      p.lse[rb * 2 + 1] = m2 + logf(s2);
      p.counts[rb * 2] = Kc;
      p.counts[rb * 2 + 1] = Mc;
    }
  }
  __syncthreads();
  const int rA = Kc, rB = Kc + Mc;
  if (rB == 0) return;
  const float lse = red[0] + logf(red[1]);
  const float vlo = red[2], vhi = red[3];
  // histogram coordinate: the score, or (f2's group scores, sums of
  // probabilities skewed towards 0) the bit pattern of the positive float, a
  // monotone piecewise-linear log2
  auto bv = [](float v) { return kLogBins ? static_cast<float>(__float_as_uint(fmaxf(v, 1e-30f))) : v; };
  const float blo = bv(vlo);
  const float scale = 255.99f / (bv(vhi) - blo);
  if (!(vhi > vlo) || !isfinite(scale)) {
    // all ranked scores tie, or the range overflows: the long split's exact paths
    if (tid == 0) p.todo[atomicAdd(p.todo_count, 1)] = static_cast<int32_t>(rb);
    return;
  }

  // ---- 2. histogram (positions >= N are the recent window: not ranked)
  uint32_t pbin[kRegE / 4];
#pragma unroll
  for (int q = 0; q < kRegE / 4; ++q) {
    uint32_t packed = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int bin = rclamp(static_cast<int>((bv(x[4 * q + k]) - blo) * scale), 0, kRegBins - 1);
      packed |= static_cast<uint32_t>(bin) << (8 * k);
      if (i0 + 4 * q + k < N) atomicAdd(&hist[warp][bin], 1u);
    }
    pbin[q] = packed;
  }
  __syncthreads();

  // ---- 3. boundary bins (warp 0: rank rA, warp 1: rank rB), from the top
  if (warp < 2 && (warp == 0 ? rA > 0 : true)) {
    const int rr = warp == 0 ? rA : rB;
    int c[8], tot = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int bin = kRegBins - 1 - (lane * 8 + q);
      int v = 0;
#pragma unroll
      for (int w = 0; w < kRegWarps; ++w) v += static_cast<int>(hist[w][bin]);
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
        s_bin[warp] = kRegBins - 1 - (lane * 8 + q);
        s_above[warp] = above;
        s_nc[warp] = c[q];
      }
      above += c[q];
    }
  }
  __syncthreads();
  const int binA = rA > 0 ? s_bin[0] : -1, binB = s_bin[1];
  const bool shared = binA == binB;   // one pair list serves both boundaries
  if ((rA > 0 && s_nc[0] > kRegCap) || s_nc[1] > kRegCap) {
    if (tid == 0) p.todo[atomicAdd(p.todo_count, 1)] = static_cast<int32_t>(rb);
    return;
  }
  const int aboveA = s_above[0], aboveB = s_above[1];

  // ---- 4. the boundary bins' (key, index) pairs
  const uint32_t ea = binA >= 0 ? static_cast<uint32_t>(binA) * 0x01010101u : 0u;
  const uint32_t eb = static_cast<uint32_t>(binB) * 0x01010101u;
  uint32_t exm = 0u;   // bit e: position i0 + e is ranked and in a boundary bin
#pragma unroll
  for (int q = 0; q < kRegE / 4; ++q) {
    uint32_t hit = __vcmpeq4(pbin[q], eb);
    if (binA >= 0) hit |= __vcmpeq4(pbin[q], ea);
    exm |= rbytes_to_bits(hit & rvalid_bytes(N - (i0 + 4 * q))) << (4 * q);
  }
  // (the few boundary positions re-read their score from shared memory and
  // recompute its bin: the scores need not stay live in registers past the
  // histogram)
  for (uint32_t m = exm; m; m &= m - 1u) {
    const int i = i0 + __ffs(m) - 1;
    const float v = kSmemRow ? s_row[i] : __ldg(row + i);
    const int bin = rclamp(static_cast<int>((bv(v) - blo) * scale), 0, kRegBins - 1);
    const int t = bin == binA ? 0 : 1;
    cand[t][atomicAdd(&s_cnt[t], 1)] = (static_cast<unsigned long long>(desc_key(v)) << 32) | static_cast<uint32_t>(i);
  }
  __syncthreads();
  const int nA = binA >= 0 ? s_cnt[0] : 0, nB = s_cnt[1];
  // Long boundary lists (8K-token rows: ~100+ pairs): each boundary's threshold
  // pair by a one-warp radix select, O(n), broadcast after one more barrier.
  // Short ones: every boundary position counts its own rank, O(n) per
  // position, no barrier.
  // (256-thread rows, <= 4096 tokens: measured faster without it — config 2
  // 63 vs 66 us — so compiled out there)
  const bool radix = kRegThreads > 256 && (nA > kRankDirect || nB > kRankDirect);   // (uniform)
  __shared__ unsigned long long s_thr[2];
  if (radix) {
    if (warp < 2 && (warp == 1 || binA >= 0)) {
      const int t = warp;
      const unsigned long long* lst = (t == 1 && shared) ? cand[0] : cand[t];
      const int n = t == 0 || shared ? nA : nB;
      const int want = (t == 0 ? rA - aboveA : rB - aboveB) - 1;
      const unsigned long long thr = warp_select_u64(lst, n, want, &hist[t][0], lane);
      if (lane == 0) s_thr[t] = thr;
    }
    __syncthreads();
  }

  // ---- 5. classification.  Bins strictly above a boundary bin are inside it
  // (bins are monotone in the score), bins below outside; a boundary-bin
  // position is inside iff (count above its bin) + (its rank among the bin's
  // pairs) < the boundary rank.
  uint32_t cm = 0u, bsel = 0u;
#pragma unroll
  for (int q = 0; q < kRegE / 4; ++q) {
    const uint32_t vm = rvalid_bytes(N - (i0 + 4 * q));
    const uint32_t c4 = rA > 0 ? rbytes_to_bits(__vcmpgtu4(pbin[q], ea) & vm) : 0u;
    const uint32_t b4 = rbytes_to_bits(__vcmpgtu4(pbin[q], eb) & vm);
    cm |= c4 << (4 * q);
    bsel |= b4 << (4 * q);
  }
  if (exm && radix) {
    for (uint32_t m = exm; m; m &= m - 1u) {
      const int e = __ffs(m) - 1;
      const int i = i0 + e;
      const float v = kSmemRow ? s_row[i] : __ldg(row + i);
      const int bin = rclamp(static_cast<int>((bv(v) - blo) * scale), 0, kRegBins - 1);
      const unsigned long long kv = (static_cast<unsigned long long>(desc_key(v)) << 32) | static_cast<uint32_t>(i);
      if (bin == binA) {
        if (kv <= s_thr[0]) cm |= 1u << e;
        if (!shared || kv <= s_thr[1]) bsel |= 1u << e;
      } else if (kv <= s_thr[1]) {
        bsel |= 1u << e;
      }
    }
  } else if (exm) {
    for (uint32_t m = exm; m; m &= m - 1u) {
      const int e = __ffs(m) - 1;
      const int i = i0 + e;
      const float v = kSmemRow ? s_row[i] : __ldg(row + i);
      const int bin = rclamp(static_cast<int>((bv(v) - blo) * scale), 0, kRegBins - 1);
      const unsigned long long kv = (static_cast<unsigned long long>(desc_key(v)) << 32) | static_cast<uint32_t>(i);
      const int t = bin == binA ? 0 : 1;
      const unsigned long long* lst = cand[t];
      const int nc = t == 0 ? nA : nB;
      int rank = 0;
      for (int d = 0; d < nc; ++d) rank += lst[d] < kv ? 1 : 0;
      if (t == 0) {
        if (aboveA + rank < rA) cm |= 1u << e;
        // binB < binA unless shared; then the same list ranks boundary B
        if (!shared || aboveB + rank < rB) bsel |= 1u << e;
      } else if (aboveB + rank < rB) {
        bsel |= 1u << e;
      }
    }
  }
  const uint32_t mm = bsel & ~cm;
  const int own = __popc(cm) | (__popc(mm) << 16);
  int incl = own;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  int ex = incl - own;
#pragma unroll
  for (int w = 0; w < kRegWarps - 1; ++w) ex += w < warp ? wtot[w] : 0;

  // ---- 6. ascending lists at this thread's offsets
  int32_t* crit = p.crit_idx + rb * p.max_crit;
  int32_t* marg = p.marg_idx + rb * p.max_marg;
  float* mw = p.marg_w + rb * p.max_marg;
  int ac = ex & 0xffff, am = ex >> 16;
  for (uint32_t m = cm; m; m &= m - 1u) crit[ac++] = i0 + __ffs(m) - 1;
  for (uint32_t m = mm; m; m &= m - 1u) {
    const int i = i0 + __ffs(m) - 1;
    marg[am] = i;
    mw[am] = __expf((kSmemRow ? s_row[i] : __ldg(row + i)) - lse);   // a' of the current step (Eq. 6)
    ++am;
  }
}

}  // namespace
}  // namespace skv
