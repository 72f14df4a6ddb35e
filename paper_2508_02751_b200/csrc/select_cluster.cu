// select_cluster.cu — K2 for LONG rows (32K / 128K contexts): the split of one
// (SLM row, sequence) by a thread-block cluster of C CTAs, each owning a
// contiguous segment of the ranked range, cooperating through distributed
// shared memory ("a thread-block cluster per long row").
//
// Same result as select_row / select_row_long (Eq. 4, Eq. 6
// P:141-152, R1-R5, R10; f2's log-coordinate bins, R16): exact
// lexicographic thresholds (T, I) on (order-preserving key, index), ascending
// lists, marg_w = a' of the current step.  Per row:
//   1. every CTA merges K1's chunk statistics (identical, fixed order) ->
//      lse', ranked range; CTA 0 writes (m', lse') and the counts;
//   2. each CTA histograms its segment (2048 bins linear in the score);
//      cluster barrier; CTA c sums bin slice c over the cluster (DSMEM);
//      barrier; each CTA finds the boundary bins from the slice totals and
//      the owning slice (the same answer everywhere);
//   3. each CTA collects its segment's boundary-bin (key, index) pairs and
//      per-warp counts above them; barrier; every CTA copies the cluster's
//      candidates, ranks its own, and the owner of each exact rank broadcasts
//      the threshold into every CTA's shared memory; barrier;
//   4. output offsets: lower CTAs' above-counts and candidates at or above
//      the thresholds (from the gathered lists), then the warps'; each warp
//      writes its sub-segment's ascending lists.
// A boundary bin holding more than kCCap positions (outlier-stretched ranges,
// massive exact ties) sends the row to a to-do list that the single-CTA long
// split (select_long.cuh: sub-bins, exact radix select) finishes right after.
#include <float.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "select_long.cuh"

namespace skv {

namespace {
constexpr int kCT = 256;
constexpr int kCW = kCT / 32;
constexpr int kCBins = 2048;
constexpr int kCCap = 1024;
constexpr int kCU = 4;
constexpr int kTodoCtas = 64;

struct ClusterShared {       // read / written across the cluster (same offsets everywhere)
  uint32_t slice_tot;        // this CTA's reduced histogram slice, summed
  int ncand[2];              // own boundary-bin candidates per target
  int above[2];              // own positions above the boundary bins per target
  int pad[3];
  unsigned long long thr[2];   // (T << 32 | I) written by the owner of each exact rank
};

template <bool kLogBins>
__global__ void __launch_bounds__(kCT, 3) select_cluster_kernel(const SelectParams p) {
  __shared__ uint32_t hist[kCBins];
  __shared__ __align__(16) uint32_t red[kCBins / 2];
  __shared__ unsigned long long cown[2][kCCap];
  __shared__ unsigned long long call[2][kCCap];
  __shared__ __align__(16) ClusterShared cs;
  __shared__ float sred[4];
  __shared__ int s_i[8];
  __shared__ int wab[kCW][2], wsel[kCW][2], s_pre[kCW][2];
  __shared__ float s_bnd[2][2];   // target t's boundary bin as a float interval [lo, hi)
  __shared__ int s_cnt[2][16], s_abv[2][16], s_off[2][17];

  griddep_launch_dependents();
  griddep_wait();
  const int C = static_cast<int>(gridDim.x), c = blockIdx.x;   // cluster (C, 1, 1): rank = blockIdx.x
  const int r = p.layer_off[p.layer_begin] + static_cast<int>(blockIdx.y);
  if (r >= p.layer_off[p.layer_end]) return;                    // uniform over the cluster
  const int j = p.rows[r], b = blockIdx.z;
  const int n = p.seq_lens[b];
  const int64_t rb = static_cast<int64_t>(j) * p.batch + b;
  const float* row = p.logits + rb * p.row_stride;
  const int Rc = lclamp(p.n_recent[b], 0, n);
  const int Kc = min(lclamp(p.k_crit[b], 0, n - Rc), p.max_crit);
  const int Mc = min(lclamp(p.k_marg[b], 0, n - Rc - Kc), p.max_marg);
  const int N = n - Rc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool al = (p.row_stride & 3) == 0;

  // ---- 1. statistics (every CTA, select_row_long's merge order)
  if (warp == 0) {
    const int nch = (n + p.chunk_tokens - 1) / p.chunk_tokens;
    const float4* st = p.stats + rb * p.n_chunks;
    float m2 = -FLT_MAX, s2 = 0.f, l2 = FLT_MAX, h2 = -FLT_MAX;
    for (int q = lane; q < nch; q += 32) {
      const float4 v = st[q];
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
      sred[0] = m2;
      sred[1] = s2;
      sred[2] = l2;
      sred[3] = h2;
      if (c == 0) {
        p.lse[rb * 2] = m2;
        p.lse[rb * 2 + 1] = m2 + logf(s2);
        p.counts[rb * 2] = Kc;
        p.counts[rb * 2 + 1] = Mc;
      }
    }
  }
  __syncthreads();
  const float lse = sred[0] + logf(sred[1]);
  const float vlo = sred[2], vhi = sred[3];
  const int rA = Kc, rB = Kc + Mc;
  if (rB == 0) return;

  // this CTA's segment of [0, N) (multiples of 1024 positions) and its warps' sub-segments
  const int S = ((N + C - 1) / C + 1023) & ~1023;
  const int g0 = min(N, c * S), g1 = min(N, g0 + S);
  const int wseg = S / kCW;   // a multiple of 128
  const int s0 = min(g1, g0 + warp * wseg), s1 = min(g1, s0 + wseg);

  auto bv = [&](float v) {
    return kLogBins ? static_cast<float>(__float_as_uint(fmaxf(v, 1e-30f))) : v;
  };
  const float blo = bv(vlo);
  const float scale1 = (static_cast<float>(kCBins) - 0.01f) / (bv(vhi) - blo);
  const bool all_equal = !(vhi > vlo);
  constexpr float kTop = static_cast<float>(kCBins) - 0.5f;
  auto bin1 = [&](float v) { return static_cast<int>(fminf(fmaxf((bv(v) - blo) * scale1, 0.f), kTop)); };
  auto to_do = [&]() {   // the single-CTA long split finishes this row
    if (c == 0 && tid == 0) p.todo[atomicAdd(p.todo_count, 1)] = static_cast<int32_t>(rb);
  };
  int32_t* crit = p.crit_idx + rb * p.max_crit;
  int32_t* marg = p.marg_idx + rb * p.max_marg;
  float* mw = p.marg_w + rb * p.max_marg;

  if (all_equal) {
    // every ranked score ties: the lowest indices win (R3), no cooperation needed
    long_emit(row, nullptr, s0, s1, lane, rA > 0 ? vlo : __int_as_float(0x7fc00000), rA - 1, vlo, rB - 1,
              lse, al, crit, marg, mw, min(s0, rA), min(max(s0, rA), rB) - rA);
    return;
  }
  if (!isfinite(scale1)) {
    to_do();
    return;
  }

  // ---- 2. histogram of the segment, reduced over the cluster in slices
  const uint32_t hist_s = smem_u32(hist), red_s = smem_u32(red);
  for (int i = tid; i < kCBins; i += kCT) hist[i] = 0u;
  __syncthreads();
  for (int base = g0 + 4 * tid; base < g1; base += 4 * kCT * kCU) {
    float4 v4[kCU];
    long_loadU<kCU>(row, base, 4 * kCT, g1, al, v4);
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
      const int i = base + 4 * kCT * u;
      const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i + k < g1)
          asm volatile("red.shared.add.u32 [%0], 1;\n" ::"r"(hist_s + 4u * static_cast<uint32_t>(bin1(vv[k])))
                       : "memory");
    }
  }
  __syncthreads();
  cluster_sync();   // (A) every CTA's histogram complete
  const int NS = kCBins / C;   // bins per slice (C a power of two <= 16)
  {
    uint32_t tot = 0;
    for (int i4 = tid; i4 < NS / 4; i4 += kCT) {
      uint4 sum = make_uint4(0u, 0u, 0u, 0u);
      for (int q = 0; q < C; ++q) {
        const uint4 v = ld_dsmem_u32x4(hist_s + 16u * static_cast<uint32_t>(c * NS / 4 + i4), q);
        sum.x += v.x;
        sum.y += v.y;
        sum.z += v.z;
        sum.w += v.w;
      }
      reinterpret_cast<uint4*>(red)[i4] = sum;
      tot += sum.x + sum.y + sum.z + sum.w;
    }
    tot = static_cast<uint32_t>(warp_sum_i(static_cast<int>(tot)));
    if (lane == 0) wab[warp][0] = static_cast<int>(tot);
    __syncthreads();
    if (tid == 0) {
      uint32_t t2 = 0;
      for (int w = 0; w < kCW; ++w) t2 += static_cast<uint32_t>(wab[w][0]);
      cs.slice_tot = t2;
    }
  }
  cluster_sync();   // (B) reduced slices and their totals visible
  if (warp < 2 && (warp == 1 || rA > 0)) {
    const int t = warp, want = t == 0 ? rA : rB;
    // slice totals of all CTAs at once (lane q), suffix sums from the top slice
    const int stq = lane < C ? static_cast<int>(ld_dsmem_u32(smem_u32(&cs.slice_tot), lane)) : 0;
    int suf = stq;   // sum of slices q.. C-1 for lane q
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_down_sync(0xffffffffu, suf, o);
      if (lane + o < 32) suf += y;
    }
    // owner: the slice q with suffix(q+1) < want <= suffix(q)
    const int above_q = suf - stq;
    const uint32_t hit = __ballot_sync(0xffffffffu, lane < C && above_q < want && want <= suf);
    const int owner = hit ? __ffs(hit) - 1 : 0;
    const int acc = __shfl_sync(0xffffffffu, above_q, owner);
    // the owner's slice from its top: lane covers NS/32 consecutive bins (>= 4)
    const int per = NS / 32;
    int cnt[16];
    int tsum = 0;
    for (int k4 = 0; k4 < per; k4 += 4) {
      const int lo = NS - (lane * per + k4) - 4;   // bins lo..lo+3, taken from the top
      const uint4 v = ld_dsmem_u32x4(red_s + 4u * static_cast<uint32_t>(lo), owner);
      cnt[k4] = static_cast<int>(v.w);
      cnt[k4 + 1] = static_cast<int>(v.z);
      cnt[k4 + 2] = static_cast<int>(v.y);
      cnt[k4 + 3] = static_cast<int>(v.x);
      tsum += cnt[k4] + cnt[k4 + 1] + cnt[k4 + 2] + cnt[k4 + 3];
    }
    int incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int ab = acc + incl - tsum;
    for (int k = 0; k < per; ++k) {
      if (ab < want && want <= ab + cnt[k]) {
        s_i[t] = cnt[k];
        s_i[2 + t] = owner * NS + NS - 1 - (lane * per + k);
        s_i[4 + t] = ab;
      }
      ab += cnt[k];
    }
  }
  __syncthreads();
  int b1[2] = {kCBins, kCBins}, above_g[2] = {0, 0};
  bool over = false;
  for (int t = 0; t < 2; ++t) {
    if (t == 0 && rA == 0) continue;
    b1[t] = s_i[2 + t];
    above_g[t] = s_i[4 + t];
    over |= s_i[t] > kCCap;
  }
  if (over) {   // uniform: every CTA found the same bins and counts
    to_do();
    cluster_sync();   // no CTA exits while another still reads its slices
    return;
  }

  // ---- 3. candidates of the boundary bins, per-warp counts above them.
  // bin1 is monotone in the score, so target t's bin is one float interval
  // [lo, hi): warp t finds both bounds exactly (select_long.cuh), and a
  // position is then decided by compares (b1 = kCBins: no target, NaN bounds).
  if (warp < 2) {
    const int t = warp, bt = b1[t];
    float lo = __int_as_float(0x7fc00000), hi = lo;
    if (bt < kCBins) {
      lo = warp_first_float([&](float f) { return bin1(f) >= bt; }, lane);
      hi = warp_first_float([&](float f) { return bin1(f) > bt; }, lane);
    }
    if (lane == 0) {
      s_bnd[t][0] = lo;
      s_bnd[t][1] = hi;
      cs.ncand[t] = 0;
    }
  }
  __syncthreads();
  {
    int ab[2] = {0, 0};
    const float lo0 = s_bnd[0][0], hi0 = s_bnd[0][1], lo1 = s_bnd[1][0], hi1 = s_bnd[1][1];
    auto insert = [&](float v, int i) {
      const bool in0 = v >= lo0 && !(v >= hi0), in1 = v >= lo1 && !(v >= hi1);
      const unsigned long long kv = (static_cast<unsigned long long>(desc_key(v)) << 32) | static_cast<uint32_t>(i);
      if (in0) cown[0][atomicAdd(&cs.ncand[0], 1)] = kv;
      if (in1) cown[1][atomicAdd(&cs.ncand[1], 1)] = kv;
    };
    int base0 = s0;
    for (; base0 + 128 * kCU <= s1; base0 += 128 * kCU) {   // whole chunks: masks, as in select_long.cuh
      float4 v4[kCU];
      long_loadU<kCU>(row, base0 + 4 * lane, 128, s1, al, v4);
      uint32_t m0 = 0u, m1 = 0u, mr = 0u;
#pragma unroll
      for (int u = 0; u < kCU; ++u) {
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
        float v = 0.f;
#pragma unroll
        for (int u = 0; u < kCU; ++u) {
          const float w = (e & 3) == 0 ? v4[u].x : (e & 3) == 1 ? v4[u].y : (e & 3) == 2 ? v4[u].z : v4[u].w;
          v = (e >> 2) == u ? w : v;
        }
        insert(v, base0 + 128 * (e >> 2) + 4 * lane + (e & 3));
      }
    }
    for (; base0 < s1; base0 += 128 * kCU) {
      float4 v4[kCU];
      long_loadU<kCU>(row, base0 + 4 * lane, 128, s1, al, v4);
#pragma unroll
      for (int u = 0; u < kCU; ++u) {
        const int i = base0 + 128 * u + 4 * lane;
        const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (i + k >= s1) continue;
          ab[0] += vv[k] >= hi0 ? 1 : 0;
          ab[1] += vv[k] >= hi1 ? 1 : 0;
          insert(vv[k], i + k);
        }
      }
    }
    ab[0] = warp_sum_i(ab[0]);
    ab[1] = warp_sum_i(ab[1]);
    if (lane == 0) {
      wab[warp][0] = ab[0];
      wab[warp][1] = ab[1];
    }
  }
  __syncthreads();
  if (tid < 2) {
    int a = 0;
    for (int w = 0; w < kCW; ++w) a += wab[w][tid];
    cs.above[tid] = a;
  }
  cluster_sync();   // (C) candidates and above-counts of every CTA visible
  // gather the cluster's candidates (rank order) and the lower CTAs' above-counts
  // every CTA's candidate counts and above-counts at once (warp t, lane q)
  if (warp < 2 && lane < C) {
    s_cnt[warp][lane] = static_cast<int>(ld_dsmem_u32(smem_u32(&cs.ncand[warp]), lane));
    s_abv[warp][lane] = static_cast<int>(ld_dsmem_u32(smem_u32(&cs.above[warp]), lane));
  }
  __syncthreads();
  int nc[2] = {0, 0}, below_above[2] = {0, 0};
  for (int t = 0; t < 2; ++t) {
    for (int q = 0; q < C; ++q) {
      s_off[t][q] = nc[t];
      nc[t] += s_cnt[t][q];
      if (q < c) below_above[t] += s_abv[t][q];
    }
    s_off[t][C] = nc[t];
  }
  if (rA == 0) nc[0] = 0;
  // copy the cluster's candidates in rank order: (q, i) flattened over the threads
  for (int t = 0; t < 2; ++t) {
    if (t == 0 && rA == 0) continue;
    const uint32_t src = smem_u32(&cown[t][0]);
    for (int x = tid; x < nc[t]; x += kCT) {
      int q = 0;
      while (x >= s_off[t][q + 1]) ++q;
      call[t][x] = ld_dsmem_u64(src + 8u * static_cast<uint32_t>(x - s_off[t][q]), q);
    }
  }
  __syncthreads();
  // rank own candidates; the owner of each exact rank broadcasts (T, I)
  for (int t = 0; t < 2; ++t) {
    if (t == 0 && rA == 0) continue;
    const int want0 = (t == 0 ? rA : rB) - above_g[t] - 1;
    const int own = cs.ncand[t];
    for (int i = tid; i < own; i += kCT) {
      const unsigned long long v = cown[t][i];
      int rank = 0;
      for (int d = 0; d < nc[t]; ++d) rank += call[t][d] < v ? 1 : 0;
      if (rank == want0)
        for (int q = 0; q < C; ++q) st_dsmem_u64(smem_u32(&cs.thr[t]), q, v);
    }
  }
  cluster_sync();   // (D) thresholds in every CTA (no remote access after this)
  const unsigned long long thrA = rA > 0 ? cs.thr[0] : 0ull, thrB = cs.thr[1];

  // ---- 4. output offsets: lower CTAs (above-counts + their candidates at or
  // above the thresholds), then this CTA's warps; emission
  if (tid < 2 * kCW) (&wsel[0][0])[tid] = 0;
  __syncthreads();
  int lowc[2] = {0, 0};
  for (int t = 0; t < 2; ++t) {
    if (t == 0 && rA == 0) continue;
    const unsigned long long thr = t == 0 ? thrA : thrB;
    for (int d = tid; d < nc[t]; d += kCT) {
      const unsigned long long v = call[t][d];
      if (v > thr) continue;
      const int i = static_cast<int>(v & 0xffffffffu);
      if (i < g0) ++lowc[t];
      else if (i < g1) atomicAdd(&wsel[(i - g0) / wseg][t], 1);
    }
  }
  lowc[0] = warp_sum_i(lowc[0]);
  lowc[1] = warp_sum_i(lowc[1]);
  if (lane == 0) {
    s_pre[warp][0] = lowc[0];
    s_pre[warp][1] = lowc[1];
  }
  __syncthreads();
  int ia = below_above[0], ib = below_above[1];
  for (int w = 0; w < kCW; ++w) {
    ia += s_pre[w][0];
    ib += s_pre[w][1];
  }
  for (int w = 0; w < warp; ++w) {
    ia += wab[w][0] + wsel[w][0];
    ib += wab[w][1] + wsel[w][1];
  }
  if (rA == 0) ia = 0;
  const float XA = rA > 0 ? key_to_float(static_cast<uint32_t>(thrA >> 32)) : __int_as_float(0x7fc00000);
  const int IA = rA > 0 ? static_cast<int>(thrA & 0xffffffffu) : -1;
  const float XB = key_to_float(static_cast<uint32_t>(thrB >> 32));
  const int IB = static_cast<int>(thrB & 0xffffffffu);
  long_emit(row, nullptr, s0, s1, lane, XA, IA, XB, IB, lse, al, crit, marg, mw, ia, ib - ia);
}

// To-do mode: rows the cluster split handed over, one 256-thread CTA each in turn.
template <bool kLogBins>
__global__ void __launch_bounds__(kLongThreads, 4) select_todo_kernel(const SelectParams p) {
  griddep_launch_dependents();
  griddep_wait();
  const int cnt = *p.todo_count;
  for (int i = blockIdx.x; i < cnt; i += gridDim.x) {
    const int rbi = p.todo[i];
    select_row_long<kLogBins>(p, rbi / p.batch, rbi % p.batch);
    __syncthreads();
  }
  // the last CTA (every CTA has read the count by then) empties the list for
  // the next split launch of the same call (SLM-layer chunks)
  if (threadIdx.x == 0 && atomicAdd(p.todo_count + 1, 1) == static_cast<int>(gridDim.x) - 1) {
    p.todo_count[0] = 0;
    p.todo_count[1] = 0;
  }
}
}  // namespace

cudaError_t launch_select_cluster(const SelectParams& p, int32_t max_rows, int32_t cluster,
                                  cudaStream_t s) {
  static const int forced = [] {
    const char* e = getenv("SMALLKV_SPLIT_CLUSTER");   // tuning knob: 2, 4, 8 or 16
    return e ? atoi(e) : 0;
  }();
  const int C = (forced == 2 || forced == 4 || forced == 8 || forced == 16) ? forced : cluster;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, max_rows, p.batch);
  cfg.blockDim = dim3(kCT);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  auto k = p.log_bins ? select_cluster_kernel<true> : select_cluster_kernel<false>;
  if (C > 8) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, p);
  if (e != cudaSuccess) return e;
  // the rows it handed over (usually none)
  return launch_select_todo(p, s);
}

cudaError_t launch_select_todo(const SelectParams& p, cudaStream_t s) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t c2 = {};
  c2.gridDim = dim3(kTodoCtas);
  c2.blockDim = dim3(kLongThreads);
  c2.stream = s;
  c2.attrs = attr;
  c2.numAttrs = 1;
  const cudaError_t e =
      cudaLaunchKernelEx(&c2, p.log_bins ? select_todo_kernel<true> : select_todo_kernel<false>, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace skv
