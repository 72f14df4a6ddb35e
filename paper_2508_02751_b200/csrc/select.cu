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
// Exact selection with a deterministic lower-index tie-break: the two rank
// boundaries are found by a 4-pass MSB radix select (8-bit digits) over
// order-preserving uint32 keys, with warp-aggregated shared-memory histograms
// (match_any); ties at a boundary are resolved by index through per-warp
// ballot prefix counts, then both lists are emitted in ascending order in one
// pass.  Rows up to kSmemCap tokens are held in shared memory; longer rows are
// re-read from global memory (they stay L2-resident across the passes).
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace skv {

namespace {
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kSmemCap = 40960;  // tokens held in shared memory (160 KB)

__device__ __forceinline__ int iclamp(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

template <bool kInSmem>
__global__ void __launch_bounds__(kThreads) select_kernel(const SelectParams p) {
  extern __shared__ uint32_t keys[];
  __shared__ uint32_t hist[2][256];
  __shared__ float red[kWarps];
  __shared__ int wcnt[kWarps][4];
  __shared__ int woff[kWarps][4];
  __shared__ uint32_t s_pref[2];
  __shared__ int s_rem[2];

  const int r = blockIdx.x;
  if (r >= *p.n_rows) return;
  const int j = p.rows[r];
  const int b = blockIdx.y;
  const int n = p.seq_lens[b];
  const int64_t rb = static_cast<int64_t>(j) * p.batch + b;
  const float* row = p.logits + rb * p.row_stride;
  const int Rc = iclamp(p.n_recent[b], 0, n);
  const int Kc = min(iclamp(p.k_crit[b], 0, n - Rc), p.max_crit);
  const int Mc = min(iclamp(p.k_marg[b], 0, n - Rc - Kc), p.max_marg);
  const int N = n - Rc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- 1. row max (and stage the row in shared memory)
  float mx = -FLT_MAX;
  for (int i = tid; i < n; i += kThreads) {
    const float x = row[i];
    if (kInSmem) keys[i] = __float_as_uint(x);
    mx = fmaxf(mx, x);
  }
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (warp == 0) {
    float v = lane < kWarps ? red[lane] : -FLT_MAX;
    v = warp_max(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const float m = red[0];
  __syncthreads();
  // ---- 2. Σ exp(s - m) in a fixed order (deterministic)
  float se = 0.f;
  for (int i = tid; i < n; i += kThreads) {
    const float x = kInSmem ? __uint_as_float(keys[i]) : row[i];
    se += expf(x - m);
  }
  se = warp_sum(se);
  if (lane == 0) red[warp] = se;
  __syncthreads();
  if (warp == 0) {
    float v = lane < kWarps ? red[lane] : 0.f;
    v = warp_sum(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const float lse = m + logf(red[0]);
  if (tid == 0) {
    p.lse[rb * 2] = m;
    p.lse[rb * 2 + 1] = lse;
    p.counts[rb * 2] = Kc;
    p.counts[rb * 2 + 1] = Mc;
  }
  if (kInSmem) {
    for (int i = tid; i < N; i += kThreads) keys[i] = desc_key(__uint_as_float(keys[i]));
    __syncthreads();
  }
  auto KEY = [&](int i) -> uint32_t { return kInSmem ? keys[i] : desc_key(row[i]); };

  // ---- 3. radix select of the rank boundaries rA = K', rB = K'+M'
  const int rA = Kc, rB = Kc + Mc;
  uint32_t pref0 = 0, pref1 = 0;
  int rem0 = rA, rem1 = rB;
  const bool act0 = rA > 0, act1 = rB > 0;
  if (act1) {
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      const uint32_t hmask = pass == 0 ? 0u : (0xffffffffu << (shift + 8));
      const bool same = act0 && pref0 == pref1;
      hist[tid >> 8][tid & 255] = 0;
      __syncthreads();
      for (int base = warp * 32; base < N; base += kThreads) {
        const int i = base + lane;
        const bool valid = i < N;
        const uint32_t k = valid ? KEY(i) : 0u;
        const uint32_t dig = (k >> shift) & 255u;
        const bool in0 = valid && act0 && (k & hmask) == pref0;
        const bool in1 = valid && !same && (k & hmask) == pref1;
        const uint32_t g0 = __match_any_sync(0xffffffffu, in0 ? dig : 0x100u);
        if (in0 && lane == __ffs(g0) - 1) atomicAdd(&hist[0][dig], __popc(g0));
        const uint32_t g1 = __match_any_sync(0xffffffffu, in1 ? dig : 0x100u);
        if (in1 && lane == __ffs(g1) - 1) atomicAdd(&hist[1][dig], __popc(g1));
      }
      __syncthreads();
      if (warp < 2 && (warp == 0 ? act0 : act1)) {
        const uint32_t* h = (warp == 1 && same) ? hist[0] : hist[warp];
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
        int found = -1, newrem = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (found < 0 && before < rem && rem <= before + c[q]) {
            found = lane * 8 + q;
            newrem = rem - before;
          }
          before += c[q];
        }
        if (found >= 0) {
          s_pref[warp] = (warp == 0 ? pref0 : pref1) | (static_cast<uint32_t>(found) << shift);
          s_rem[warp] = newrem;
        }
      }
      __syncthreads();
      if (act0) { pref0 = s_pref[0]; rem0 = s_rem[0]; }
      pref1 = s_pref[1];
      rem1 = s_rem[1];
      __syncthreads();
    }
  }
  // thresholds and how many elements equal to them are taken (by lowest index)
  const uint32_t TA = act0 ? pref0 : 0u, TB = act1 ? pref1 : 0u;
  const int takeA = act0 ? rem0 : 0, takeB = act1 ? rem1 : 0;

  // ---- 4. per-warp segment counts
  const int seg = ((N + kThreads - 1) / kThreads) * 32;
  const int s0 = warp * seg, s1 = min(N, s0 + seg);
  int ltA = 0, eqA = 0, ltB = 0, eqB = 0;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + lane;
    const bool valid = i < s1;
    const uint32_t k = valid ? KEY(i) : 0xffffffffu;
    ltA += __popc(__ballot_sync(0xffffffffu, valid && act0 && k < TA));
    eqA += __popc(__ballot_sync(0xffffffffu, valid && act0 && k == TA));
    ltB += __popc(__ballot_sync(0xffffffffu, valid && act1 && k < TB));
    eqB += __popc(__ballot_sync(0xffffffffu, valid && act1 && k == TB));
  }
  if (lane == 0) {
    wcnt[warp][0] = ltA; wcnt[warp][1] = eqA; wcnt[warp][2] = ltB; wcnt[warp][3] = eqB;
  }
  __syncthreads();
  if (tid == 0) {
    int tA = 0, tB = 0, oc = 0, om = 0;
    for (int w = 0; w < kWarps; ++w) {
      woff[w][0] = tA; woff[w][1] = tB; woff[w][2] = oc; woff[w][3] = om;
      const int cw = wcnt[w][0] + iclamp(takeA - tA, 0, wcnt[w][1]);
      const int bw = wcnt[w][2] + iclamp(takeB - tB, 0, wcnt[w][3]);
      tA += wcnt[w][1];
      tB += wcnt[w][3];
      oc += cw;
      om += bw - cw;
    }
  }
  __syncthreads();

  // ---- 5. emit ascending lists
  int tieA = woff[warp][0], tieB = woff[warp][1], oc = woff[warp][2], om = woff[warp][3];
  int32_t* crit = p.crit_idx + rb * p.max_crit;
  int32_t* marg = p.marg_idx + rb * p.max_marg;
  float* mw = p.marg_w + rb * p.max_marg;
  const uint32_t lt = lanemask_lt();
  for (int base = s0; base < s1; base += 32) {
    const int i = base + lane;
    const bool valid = i < s1;
    const uint32_t k = valid ? KEY(i) : 0xffffffffu;
    const bool eA = valid && act0 && k == TA;
    const bool eB = valid && act1 && k == TB;
    const uint32_t bA = __ballot_sync(0xffffffffu, eA);
    const uint32_t bB = __ballot_sync(0xffffffffu, eB);
    const bool isC = valid && act0 && (k < TA || (eA && tieA + __popc(bA & lt) < takeA));
    const bool inB = valid && act1 && (k < TB || (eB && tieB + __popc(bB & lt) < takeB));
    const bool isM = inB && !isC;
    const uint32_t bc = __ballot_sync(0xffffffffu, isC);
    const uint32_t bm = __ballot_sync(0xffffffffu, isM);
    if (isC) crit[oc + __popc(bc & lt)] = i;
    if (isM) {
      const int o = om + __popc(bm & lt);
      marg[o] = i;
      mw[o] = expf(key_to_float(k) - lse);
    }
    tieA += __popc(bA);
    tieB += __popc(bB);
    oc += __popc(bc);
    om += __popc(bm);
  }
}
}  // namespace

cudaError_t launch_select(const SelectParams& p, int32_t max_rows, int32_t max_seq_len,
                          cudaStream_t s) {
  dim3 grid(max_rows, p.batch);
  if (max_seq_len <= kSmemCap) {
    const size_t sm = static_cast<size_t>(max_seq_len) * 4;
    if (sm > 48 * 1024)
      cudaFuncSetAttribute(select_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sm));
    select_kernel<true><<<grid, kThreads, sm, s>>>(p);
  } else {
    select_kernel<false><<<grid, kThreads, 0, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace skv
