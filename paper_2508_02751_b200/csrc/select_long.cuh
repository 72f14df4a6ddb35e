// select_long.cuh — K2's split of LONG rows (n > kSmemCap, e.g. 32K / 128K
// contexts): one 256-thread CTA per (SLM row, sequence), the row read from
// global memory (L2 / HBM) in every pass with 8 independent 16-byte loads in
// flight per thread (32 KB per CTA), so the ~3 passes over a 512 KB row run
// at memory speed instead of at the latency of 2 loads per thread.
//
// Same result as select_row (select_row.cuh; Eq. 4, Eq. 6
// P:141-152, R1-R5, R10; variant f1's running sums, Eq. 1; variant
// f2's log-coordinate bins, R16): exact lexicographic thresholds (T, I) on
// (order-preserving key, index) per rank boundary, ascending lists, marg_w =
// a' of the current step.
//   1. (max, Σexp) from K1's chunk statistics -> lse'; ranked range [lo, hi]
//      (f1: acc += a' first, range of the updated sums);
//   2. one CTA-wide histogram of 2048 bins linear in the score (monotone) —
//      at 128K tokens a boundary bin holds ~200 positions, so the sub-bin
//      level of select_row is rarely needed; a boundary bin with more than
//      kCap positions is refined with 2048 sub-bins, and a still-overfull one
//      (massive exact ties) takes the exact 4-pass 8-bit radix select;
//   3. one pass collects the boundary bins' (key, index) pairs and counts,
//      per warp segment, the positions above them (the output offsets), the
//      pair of exact rank is the threshold;
//   4. one pass writes both ascending lists per warp segment.
#pragma once

#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace skv {
namespace {

constexpr int kLongThreads = 256;
constexpr int kLongWarps = kLongThreads / 32;
constexpr int kLongBins = 2048;
constexpr int kLongCap = 1024;
#ifndef SKV_LONG_U
#define SKV_LONG_U 4
#endif
constexpr int kLongU = SKV_LONG_U;   // 16-byte loads in flight per thread and pass

__device__ __forceinline__ int lclamp(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

// The smallest float f (value order, -inf .. +inf) with pred(f) true, for a
// predicate monotone in f (false below some f, true from it on); NaN when no
// float satisfies it.  One warp, a 32-way search over the order-preserving
// float keys: 7 ballot rounds.  All lanes return it.
template <typename Pred>
__device__ __forceinline__ float warp_first_float(Pred pred, int lane) {
  auto from_key = [](uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); };
  constexpr uint32_t kNegInf = 0x007fffffu, kPosInf = 0xff800000u;   // keys of -inf, +inf
  if (!__any_sync(0xffffffffu, lane == 0 && pred(from_key(kPosInf)))) return __int_as_float(0x7fc00000);
  long long L = static_cast<long long>(kNegInf) - 1, H = kPosInf;   // pred(L) false, pred(H) true
  while (H - L > 1) {
    const long long step = (H - L + 31) / 32;
    const long long k = min(L + step * (lane + 1), H);
    const uint32_t bal = __ballot_sync(0xffffffffu, pred(from_key(static_cast<uint32_t>(k))));
    const int f = __ffs(bal) - 1;   // lane 31 holds H: some lane is true
    const long long nH = min(L + step * (f + 1), H);
    L = f == 0 ? L : L + step * f;
    H = nH;
  }
  return from_key(static_cast<uint32_t>(H));
}

// U float4 loads of positions base + stride*u (+0..3) of src: unguarded when
// the last one is fully inside [0, lim) (and the row is 16-byte aligned)
template <int U>
__device__ __forceinline__ void long_loadU(const float* src, int base, int stride, int lim, bool al,
                                           float4 (&v)[U]) {
  if (al && base + stride * (U - 1) + 3 < lim) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(reinterpret_cast<const float4*>(src + base + stride * u));
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + stride * u;
      v[u].x = i < lim ? src[i] : 0.f;
      v[u].y = i + 1 < lim ? src[i + 1] : 0.f;
      v[u].z = i + 2 < lim ? src[i + 2] : 0.f;
      v[u].w = i + 3 < lim ? src[i + 3] : 0.f;
    }
  }
}

// One warp writes the ascending lists of its segment [s0, s1) of the ranked
// range (s0 a multiple of 4): position i is critical iff (score, i) <= (XA, IA)
// lexicographically (score > XA, or == XA and i <= IA), in the inclusive set
// iff <= (XB, IB), marginal iff inclusive and not critical.  oc / om: the
// warp's first slots in crit / marg.  score = the ranking value (logits, or
// f1's sums: then `row` holds the logits, whose a' is marg_w).
// Each lane takes 16 consecutive positions per step (four 16-byte loads, L1
// allocating: the halves of a sector two loads apart are one L1 line), so one
// packed warp scan serves 512 positions and the lists are written per set bit.
__device__ __forceinline__ void long_emit(const float* score, const float* row, int s0, int s1, int lane,
                                          float XA, int IA, float XB, int IB, float lse, bool al,
                                          int32_t* crit, int32_t* marg, float* mw, int oc, int om) {
  for (int base = s0; base < s1; base += 512) {
    const int p0 = base + 16 * lane;
    float v[16];
    if (al && p0 + 15 < s1) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 t = *reinterpret_cast<const float4*>(score + p0 + 4 * u);
        v[4 * u] = t.x;
        v[4 * u + 1] = t.y;
        v[4 * u + 2] = t.z;
        v[4 * u + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = p0 + e < s1 ? score[p0 + e] : 0.f;
    }
    // (score, i) <= (X, I): for a whole step with i <= I that is score >= X,
    // with i > I score > X; only the one step holding I compares both
    // Whole steps take the sign of a difference: v >= X iff v - X has a clear
    // sign bit (IEEE without flush-to-zero: distinct floats never subtract to
    // zero, equal ones give +0; inf - inf is the canonical, positive NaN), and
    // v > X iff X - v has it set; one FADD and one funnel shift per position.
    auto sel16 = [&](float X, int I) {
      uint32_t r = 0u;
      if (X != X) return 0u;   // no target (NaN threshold): nothing selected
      if (p0 + 15 <= I) {
        uint32_t sg = 0u;
#pragma unroll
        for (int e = 15; e >= 0; --e) sg = __funnelshift_l(__float_as_uint(v[e] - X), sg, 1);
        r = ~sg & 0xffffu;
      } else if (p0 > I) {
        uint32_t sg = 0u;
#pragma unroll
        for (int e = 15; e >= 0; --e) sg = __funnelshift_l(__float_as_uint(X - v[e]), sg, 1);
        r = sg & 0xffffu;
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          r |= static_cast<uint32_t>(v[e] > X || (v[e] == X && p0 + e <= I)) << e;
      }
      return r;
    };
    const uint32_t vmask = s1 - p0 >= 16 ? 0xffffu : (s1 > p0 ? (1u << (s1 - p0)) - 1u : 0u);
    const uint32_t cm = sel16(XA, IA) & vmask;   // (NaN XA when there is no target A: none)
    const uint32_t bm = sel16(XB, IB) & vmask;
    const uint32_t mm = bm & ~cm;
    const int own = __popc(cm) | (__popc(mm) << 16);
    int incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int ac = oc + ((incl - own) & 0xffff), am = om + ((incl - own) >> 16);
    for (uint32_t m = cm; m; m &= m - 1u) crit[ac++] = p0 + __ffs(m) - 1;
    // per set bit (a 16-way predicated loop costs every lane ~100 instructions
    // per step); the value comes back from L1 — this lane loaded it just now
    // (f1: the logit, not the running sum: a' of the current step, Eq. 6)
    const float* wsrc = row ? row : score;
    for (uint32_t m = mm; m; m &= m - 1u) {
      const int i = p0 + __ffs(m) - 1;
      marg[am] = i;
      mw[am] = __expf(wsrc[i] - lse);
      ++am;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    oc += tot & 0xffff;
    om += tot >> 16;
  }
}

// kT threads per CTA: 256 (several CTAs per SM) or 1024 (one per SM: only
// 148 rows live, so at 128K tokens passes 2 and 3 find the row in L2)
template <bool kLogBins, int kT = kLongThreads>
__device__ __forceinline__ void select_row_long(const SelectParams& p, const int j, const int b) {
  constexpr int kW = kT / 32;
  __shared__ uint32_t hist[kLongBins];
  __shared__ unsigned long long cand[2][kLongCap];
  __shared__ float red[4][kW];
  __shared__ int wab[kW][2];
  __shared__ int wsel[kW][2];
  __shared__ int s_i[16];            // [0,1] cell count, [2,3] bin, [4,5] above, [6,7] cand count
  __shared__ uint32_t s_u[4];        // [0,1] radix prefix, [2,3] threshold key
  __shared__ int s_ti[2], s_rem[2];
  __shared__ float s_thr[2][2];      // target t's cell [lo, hi) in score order

  const int n = p.seq_lens[b];
  const int64_t rb = static_cast<int64_t>(j) * p.batch + b;
  const float* row = p.logits + rb * p.row_stride;
  const int Rc = lclamp(p.n_recent[b], 0, n);
  const int Kc = min(lclamp(p.k_crit[b], 0, n - Rc), p.max_crit);
  const int Mc = min(lclamp(p.k_marg[b], 0, n - Rc - Kc), p.max_marg);
  const int N = n - Rc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* accrow = p.acc ? p.acc + rb * p.row_stride : nullptr;
  const float* score = accrow ? accrow : row;
  const bool al = (p.row_stride & 3) == 0;
  // kLongU float4 loads of positions base + stride*u (+0..3): unguarded when the
  // last one is fully inside [0, lim)
  auto loadU = [&](const float* src, int base, int stride, int lim, float4 (&v)[kLongU]) {
    if (al && base + stride * (kLongU - 1) + 3 < lim) {
#pragma unroll
      for (int u = 0; u < kLongU; ++u) v[u] = __ldcg(reinterpret_cast<const float4*>(src + base + stride * u));
    } else {
#pragma unroll
      for (int u = 0; u < kLongU; ++u) {
        const int i = base + stride * u;
        v[u].x = i < lim ? src[i] : 0.f;
        v[u].y = i + 1 < lim ? src[i + 1] : 0.f;
        v[u].z = i + 2 < lim ? src[i + 2] : 0.f;
        v[u].w = i + 3 < lim ? src[i + 3] : 0.f;
      }
    }
  };
  // positions i..i+3 (i a multiple of 4, i < lim); lanes past lim read zeros
  auto load4 = [&](const float* src, int i, int lim) -> float4 {
    if (i >= lim) return make_float4(0.f, 0.f, 0.f, 0.f);
    if (al && i + 3 < lim) return __ldcg(reinterpret_cast<const float4*>(src + i));
    float4 v;
    v.x = src[i];
    v.y = i + 1 < lim ? src[i + 1] : 0.f;
    v.z = i + 2 < lim ? src[i + 2] : 0.f;
    v.w = i + 3 < lim ? src[i + 3] : 0.f;
    return v;
  };

  // ---- 1. statistics: (max, Σexp) over [0, n) and the ranked range from K1's chunks
  if (warp == 0) {
    const int nch = (n + p.chunk_tokens - 1) / p.chunk_tokens;
    const float4* st = p.stats + rb * p.n_chunks;
    float m2 = -FLT_MAX, s2 = 0.f, l2 = FLT_MAX, h2 = -FLT_MAX;
    for (int c = lane; c < nch; c += 32) {
      const float4 v = st[c];
      const float mm = fmaxf(m2, v.x);
      s2 = s2 * __expf(m2 - mm) + v.y * __expf(v.x - mm);
      m2 = mm;
      l2 = fminf(l2, v.z);
      h2 = fmaxf(h2, v.w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, m2, o), so = __shfl_xor_sync(0xffffffffu, s2, o);
      const float mm = fmaxf(m2, mo);
      s2 = s2 * __expf(m2 - mm) + so * __expf(mo - mm);
      m2 = mm;
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
  __syncthreads();
  const float lse = red[0][0] + logf(red[1][0]);
  float vlo = red[2][0], vhi = red[3][0];
  if (accrow) {
    // f1: acc[v] += a'_v for v < n (in place), rank on acc; range over [0, N)
    float lo = FLT_MAX, hi = -FLT_MAX;
    for (int base = 4 * tid; base < n; base += 4 * kT * kLongU) {
      float4 a[kLongU], s[kLongU];
#pragma unroll
      for (int u = 0; u < kLongU; ++u) {
        a[u] = load4(accrow, base + 4 * kT * u, n);
        s[u] = load4(row, base + 4 * kT * u, n);
      }
#pragma unroll
      for (int u = 0; u < kLongU; ++u) {
        const int i = base + 4 * kT * u;
        float av[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
        const float sv[4] = {s[u].x, s[u].y, s[u].z, s[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (i + k >= n) continue;
          av[k] += __expf(sv[k] - lse);
          accrow[i + k] = av[k];
          if (i + k < N) {
            lo = fminf(lo, av[k]);
            hi = fmaxf(hi, av[k]);
          }
        }
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
    for (int w = 0; w < kW; ++w) {
      vlo = fminf(vlo, red[2][w]);
      vhi = fmaxf(vhi, red[3][w]);
    }
    __threadfence_block();
  }
  const int rA = Kc, rB = Kc + Mc;
  if (rB == 0) return;

  // per-warp contiguous segments of [0, N) (index order = output order),
  // multiples of 128 positions (4 consecutive per lane per step)
  const int seg = ((N + kW * 128 - 1) / (kW * 128)) * 128;
  const int s0 = min(N, warp * seg), s1 = min(N, s0 + seg);

  auto bv = [&](float v) {
    return kLogBins ? static_cast<float>(__float_as_uint(fmaxf(v, 1e-30f))) : v;
  };
  const float blo = bv(vlo);
  const float scale1 = (static_cast<float>(kLongBins) - 0.01f) / (bv(vhi) - blo);
  const bool all_equal = !(vhi > vlo);
  const bool bad_range = !all_equal && !isfinite(scale1);
  // bin = min(trunc_u32(fma(v, scale, off)), top): one FFMA, a saturating
  // conversion (negatives and NaN -> 0) and a min.  Only monotonicity in the
  // score matters (the thresholds are then found exactly), not where the bin
  // edges fall.
  const float off1 = -blo * scale1;
  auto bin1 = [&](float v) {
    return static_cast<int>(min(__float2uint_rz(fmaf(bv(v), scale1, off1)), static_cast<unsigned>(kLongBins - 1)));
  };
  // level-2 sub-bins inside boundary bin B of target t
  float lo2[2] = {0.f, 0.f}, sc2[2] = {0.f, 0.f};
  int b1[2] = {-1, -1}, b2[2] = {-1, -1};
  bool lv2[2] = {false, false};
  auto bin2 = [&](float v, int t) {
    return static_cast<int>(min(__float2uint_rz(fmaf(bv(v), sc2[t], -lo2[t] * sc2[t])),
                                static_cast<unsigned>(kLongBins - 1)));
  };
  // target t's cell: -1 below (worse), 0 inside, +1 above (better)
  auto where = [&](float v, int t) -> int {
    const int x = bin1(v);
    if (x != b1[t]) return x > b1[t] ? 1 : -1;
    if (!lv2[t]) return 0;
    const int y = bin2(v, t);
    return y == b2[t] ? 0 : (y > b2[t] ? 1 : -1);
  };
  int above_g[2] = {0, 0};
  bool fallback = bad_range;
  uint32_t TK[2] = {0u, 0u};
  int TI[2] = {-1, -1};

  // histogram of the positions in [0, N) that lie in cell t_src (t_src < 0:
  // all) under bin function `fn`, then the boundary bin of each target in
  // `tmask` from the top: s_i[t] count in the bin, s_i[2+t] bin, s_i[4+t] above
  auto level = [&](int t_src, auto fn, uint32_t tmask, const int* want) {
    for (int i = tid; i < kLongBins; i += kT) hist[i] = 0u;
    __syncthreads();
    const int bsrc = t_src >= 0 ? b1[t_src] : -1;
    const uint32_t hist_s = smem_u32(hist);
    int base = 4 * tid;
    if (bsrc < 0) {
      // level 1, whole chunks: no bound or cell test per position
      for (; base + 4 * kT * (kLongU - 1) + 3 < N; base += 4 * kT * kLongU) {
        float4 v4[kLongU];
        loadU(score, base, 4 * kT, N, v4);
#pragma unroll
        for (int u = 0; u < kLongU; ++u) {
          const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
          for (int k = 0; k < 4; ++k)
            asm volatile("red.shared.add.u32 [%0], 1;\n" ::"r"(hist_s + 4u * static_cast<uint32_t>(fn(vv[k]))) : "memory");
        }
      }
    }
    for (; base < N; base += 4 * kT * kLongU) {
      float4 v4[kLongU];
      loadU(score, base, 4 * kT, N, v4);
#pragma unroll
      for (int u = 0; u < kLongU; ++u) {
        const int i = base + 4 * kT * u;
        const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // level 2: only positions inside the level-1 boundary bin
          const bool take = i + k < N && (bsrc < 0 || bin1(vv[k]) == bsrc);
          // shared-window reduction (the lambda sees `hist` through a generic
          // reference; the explicit .shared address avoids a generic atomic)
          if (take) asm volatile("red.shared.add.u32 [%0], 1;\n" ::"r"(hist_s + 4u * static_cast<uint32_t>(fn(vv[k]))) : "memory");
        }
      }
    }
    __syncthreads();
    if (warp < 2 && ((tmask >> warp) & 1u)) {
      const int t = warp, rr = want[t];
      constexpr int PER = kLongBins / 32;
      int tot = 0;
      for (int q = 0; q < PER; ++q) tot += static_cast<int>(hist[kLongBins - 1 - (lane * PER + q)]);
      int incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int ab = incl - tot;
      if (ab < rr && rr <= incl) {
        for (int q = 0; q < PER; ++q) {
          const int bi = kLongBins - 1 - (lane * PER + q);
          const int c = static_cast<int>(hist[bi]);
          if (ab < rr && rr <= ab + c) {
            s_i[t] = c;
            s_i[2 + t] = bi;
            s_i[4 + t] = ab;
          }
          ab += c;
        }
      }
    }
    __syncthreads();
  };

  if (!all_equal && !fallback) {
    const int want1[2] = {rA, rB};
    level(-1, bin1, rA > 0 ? 3u : 2u, want1);
    int cnt[2] = {0, 0};
    for (int t = 0; t < 2; ++t) {
      if (t == 0 && rA == 0) continue;
      b1[t] = s_i[2 + t];
      above_g[t] = s_i[4 + t];
      cnt[t] = s_i[t];
    }
    __syncthreads();
    for (int t = 0; t < 2; ++t) {
      if ((t == 0 && rA == 0) || cnt[t] <= kLongCap) continue;
      // level 2: sub-bins linear inside the boundary bin (outlier-stretched ranges)
      lv2[t] = true;
      lo2[t] = blo + static_cast<float>(b1[t]) / scale1;
      sc2[t] = scale1 * static_cast<float>(kLongBins);
      const int want2[2] = {rA - above_g[0], rB - above_g[1]};
      const int tt = t;
      level(t, [&](float v) { return bin2(v, tt); }, 1u << t, want2);
      b2[t] = s_i[2 + t];
      above_g[t] += s_i[4 + t];
      cnt[t] = s_i[t];
      __syncthreads();
      if (cnt[t] > kLongCap) fallback = true;
    }
  }

  if (fallback) {
    // ---- massive exact ties: 4-pass 8-bit MSB radix select of the keys, then the tie index
    uint32_t(*rh)[256] = reinterpret_cast<uint32_t(*)[256]>(&hist[0]);
    uint32_t pref[2] = {0u, 0u};
    int rem[2] = {rA, rB};
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      const uint32_t hmask = pass == 0 ? 0u : (0xffffffffu << (shift + 8));
      for (int i = tid; i < 512; i += kT) rh[i >> 8][i & 255] = 0;
      __syncthreads();
      for (int base = warp * 32; base < N; base += kT) {
        const int i = base + lane;
        const bool valid = i < N;
        const uint32_t k = valid ? desc_key(score[i]) : 0u;
        const uint32_t dig = (k >> shift) & 255u;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const bool in = valid && (t == 1 || rA > 0) && (k & hmask) == pref[t];
          const uint32_t grp = __match_any_sync(0xffffffffu, in ? dig : 0x100u);
          if (in && lane == __ffs(grp) - 1) atomicAdd(&rh[t][dig], __popc(grp));
        }
      }
      __syncthreads();
      if (warp < 2 && (warp == 1 || rA > 0)) {
        const int t = warp;
        int c[8], tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          c[q] = static_cast<int>(rh[t][lane * 8 + q]);
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
          if (before < rem[t] && rem[t] <= before + c[q]) {
            s_u[t] = pref[t] | (static_cast<uint32_t>(lane * 8 + q) << shift);
            s_rem[t] = rem[t] - before;
          }
          before += c[q];
        }
      }
      __syncthreads();
      for (int t = 0; t < 2; ++t) {
        if (t == 0 && rA == 0) continue;
        pref[t] = s_u[t];
        rem[t] = s_rem[t];
      }
      __syncthreads();
    }
    // the rem-th (1-based) position in index order whose key equals T
    for (int t = 0; t < 2; ++t) {
      if (t == 0 && rA == 0) continue;
      const uint32_t T = pref[t];
      int eq = 0;
      for (int base = s0; base < s1; base += 32) {
        const int i = base + lane;
        eq += __popc(__ballot_sync(0xffffffffu, i < s1 && desc_key(score[i]) == T));
      }
      if (lane == 0) wab[warp][0] = eq;
      __syncthreads();
      int before = 0;
      for (int w = 0; w < warp; ++w) before += wab[w][0];
      if (before < rem[t] && rem[t] <= before + eq) {
        for (int base = s0; base < s1; base += 32) {
          const int i = base + lane;
          const uint32_t bal = __ballot_sync(0xffffffffu, i < s1 && desc_key(score[i]) == T);
          const int k = rem[t] - before;
          if (k >= 1 && k <= __popc(bal)) {
            if (lane == 0) {
              uint32_t m = bal;
              for (int q = 1; q < k; ++q) m &= m - 1;
              s_ti[t] = base + __ffs(m) - 1;
            }
            break;
          }
          before += __popc(bal);
        }
      }
      __syncthreads();
      TK[t] = T;
      TI[t] = s_ti[t];
    }
  } else if (!all_equal) {
    // ---- candidates of the boundary cells, per-warp counts above them
    // `where` is monotone in the score, so target t's cell is one interval
    // [lo_t, hi_t) of floats and "above" is v >= hi_t: warp t finds both
    // bounds exactly by a 32-way search over the order-preserving float keys
    // (7 rounds each); a bound no float reaches is NaN (every compare false).
    if (warp < 2) {
      const int t = warp;
      if (lane == 0) s_i[6 + t] = 0;
      float bnd[2] = {__int_as_float(0x7fc00000), __int_as_float(0x7fc00000)};
      if (t == 1 || rA > 0) {
        // smallest float with where(f, t) >= e (e = 0: cell or above; 1: above)
#pragma unroll 1
        for (int e = 0; e < 2; ++e) bnd[e] = warp_first_float([&](float f) { return where(f, t) >= e; }, lane);
      }
      if (lane == 0) {
        s_thr[t][0] = bnd[0];
        s_thr[t][1] = bnd[1];
      }
    }
    __syncthreads();
    int ab[2] = {0, 0};
    const float lo0 = s_thr[0][0], hi0 = s_thr[0][1], lo1 = s_thr[1][0], hi1 = s_thr[1][1];
    auto cand_one = [&](float v, int i) {
      const bool a0 = v >= hi0, a1 = v >= hi1;
      ab[0] += a0 ? 1 : 0;
      ab[1] += a1 ? 1 : 0;
      const bool in0 = v >= lo0 && !a0, in1 = v >= lo1 && !a1;
      if (in0 || in1) {   // rare: a boundary cell
        const unsigned long long key = (static_cast<unsigned long long>(desc_key(v)) << 32) | static_cast<uint32_t>(i);
        if (in0) cand[0][atomicAdd(&s_i[6], 1)] = key;
        if (in1) cand[1][atomicAdd(&s_i[7], 1)] = key;
      }
    };
    int base0 = s0;
    static_assert(kLongU * 4 <= 32, "one mask bit per position of a chunk");
    for (; base0 + 128 * kLongU <= s1; base0 += 128 * kLongU) {   // whole chunks
      float4 v4[kLongU];
      loadU(score, base0 + 4 * lane, 128, s1, v4);
      // per position: four compares and three predicated bit sets (above A,
      // above B, boundary cell); the counts are two popcounts per chunk and
      // the rare boundary positions are inserted after the chunk
      uint32_t m0 = 0u, m1 = 0u, mr = 0u;
#pragma unroll
      for (int u = 0; u < kLongU; ++u) {
        const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float v = vv[k];
          const bool a0 = v >= hi0, a1 = v >= hi1;
          const uint32_t bit = 1u << (4 * u + k);
          if (a0) m0 |= bit;
          if (a1) m1 |= bit;
          if ((v >= lo0 && !a0) || (v >= lo1 && !a1)) mr |= bit;
        }
      }
      ab[0] += __popc(m0);
      ab[1] += __popc(m1);
      while (mr) {
        const int e = __ffs(mr) - 1;
        mr &= mr - 1u;
        float v = 0.f;   // the value back out of this lane's registers
#pragma unroll
        for (int u = 0; u < kLongU; ++u) {
          const float w = (e & 3) == 0 ? v4[u].x : (e & 3) == 1 ? v4[u].y : (e & 3) == 2 ? v4[u].z : v4[u].w;
          v = (e >> 2) == u ? w : v;
        }
        const int i = base0 + 128 * (e >> 2) + 4 * lane + (e & 3);
        const bool in0 = v >= lo0 && !(v >= hi0), in1 = v >= lo1 && !(v >= hi1);
        const unsigned long long key = (static_cast<unsigned long long>(desc_key(v)) << 32) | static_cast<uint32_t>(i);
        if (in0) cand[0][atomicAdd(&s_i[6], 1)] = key;
        if (in1) cand[1][atomicAdd(&s_i[7], 1)] = key;
      }
    }
    for (; base0 < s1; base0 += 128 * kLongU) {
      float4 v4[kLongU];
      loadU(score, base0 + 4 * lane, 128, s1, v4);
#pragma unroll
      for (int u = 0; u < kLongU; ++u) {
        const int i = base0 + 128 * u + 4 * lane;
        const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (i + k < s1) cand_one(vv[k], i + k);
      }
    }
    ab[0] = warp_sum_i(ab[0]);
    ab[1] = warp_sum_i(ab[1]);
    if (lane == 0) {
      wab[warp][0] = ab[0];
      wab[warp][1] = ab[1];
    }
    __syncthreads();
    // the pair of exact rank (want - 1) among a cell's candidates (all distinct)
    for (int t = 0; t < 2; ++t) {
      if (t == 0 && rA == 0) continue;
      const int nc = s_i[6 + t];
      const int want = (t == 0 ? rA : rB) - above_g[t] - 1;
      for (int c = tid; c < nc; c += kT) {
        const unsigned long long v = cand[t][c];
        int rank = 0;
        for (int d = 0; d < nc; ++d) rank += cand[t][d] < v ? 1 : 0;
        if (rank == want) {
          s_u[2 + t] = static_cast<uint32_t>(v >> 32);
          s_ti[t] = static_cast<int>(v & 0xffffffffu);
        }
      }
    }
    __syncthreads();
    for (int t = 0; t < 2; ++t) {
      if (t == 0 && rA == 0) continue;
      TK[t] = s_u[2 + t];
      TI[t] = s_ti[t];
    }
  }

  // ---- per-warp output offsets
  int cbase = 0, mbase = 0;
  if (all_equal) {
    cbase = min(s0, rA);
    mbase = min(max(s0, rA), rB) - rA;
  } else if (fallback) {
    // (rare) count each warp segment's selections with the exact thresholds
    const float XA = rA > 0 ? key_to_float(TK[0]) : __int_as_float(0x7fc00000), XB = key_to_float(TK[1]);
    int cc = 0, cb = 0;
    for (int i = s0 + lane; i < s1; i += 32) {
      const float v = score[i];
      const bool isC = v > XA || (v == XA && i <= TI[0]);
      const bool inB = v > XB || (v == XB && i <= TI[1]);
      cc += isC ? 1 : 0;
      cb += inB ? 1 : 0;
    }
    cc = warp_sum_i(cc);
    cb = warp_sum_i(cb);
    if (lane == 0) {
      wab[warp][0] = cc;
      wab[warp][1] = cb;
      wsel[warp][0] = wsel[warp][1] = 0;
    }
    __syncthreads();
    for (int w = 0; w < warp; ++w) {
      cbase += wab[w][0];
      mbase += wab[w][1] - wab[w][0];
    }
  } else {
    if (tid < 2 * kW) (&wsel[0][0])[tid] = 0;
    __syncthreads();
    for (int t = 0; t < 2; ++t) {
      if (t == 0 && rA == 0) continue;
      const unsigned long long thr = (static_cast<unsigned long long>(TK[t]) << 32) | static_cast<uint32_t>(TI[t]);
      const int nc = s_i[6 + t];
      for (int c = tid; c < nc; c += kT) {
        const unsigned long long v = cand[t][c];
        if (v <= thr) atomicAdd(&wsel[static_cast<int>(v & 0xffffffffu) / seg][t], 1);
      }
    }
    __syncthreads();
    int ia = 0, ib = 0;
    for (int w = 0; w < warp; ++w) {
      ia += wab[w][0] + wsel[w][0];
      ib += wab[w][1] + wsel[w][1];
    }
    cbase = rA > 0 ? ia : 0;
    mbase = ib - cbase;
  }

  // ---- emission: this warp's segment
  const float XA = rA > 0 ? (all_equal ? vlo : key_to_float(TK[0])) : __int_as_float(0x7fc00000);
  const float XB = all_equal ? vlo : key_to_float(TK[1]);
  const int IA = all_equal ? rA - 1 : TI[0], IB = all_equal ? rB - 1 : TI[1];
  long_emit(score, accrow ? row : nullptr, s0, s1, lane, XA, IA, XB, IB, lse, al,
            p.crit_idx + rb * p.max_crit, p.marg_idx + rb * p.max_marg, p.marg_w + rb * p.max_marg,
            cbase, mbase);
}

}  // namespace
}  // namespace skv
