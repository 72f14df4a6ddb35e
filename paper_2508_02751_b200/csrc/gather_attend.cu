// gather_attend.cu — K3 (+ fused K4): SmallKV's compensated decode attention.
//
// Alg. 1 l.11-14, App. D SmallKV_attention_forward:
//   O_c = softmax over the critical ∪ recent tokens (R2: FlashAttention over
//         the selected K/V),
//   O_m = Σ_{k ∈ marginal} A'_{f(i)}[k] · V[k]   (Eq. 6 second branch),
//   O   = O_c + O_m                                (no renormalisation, R13).
//
// B200 design.  Work unit = LLM kv-group g of sequence b.  Its q-heads map to
// one or more DISTINCT SLM rows r (D6); the group's "virtual list" is
//     [ recent R' (every head critical) | crit(r_0) | marg(r_0) | crit(r_1) | ... ]
// with a 16-bit head mask per entry (bits 0..7: critical for head h, bits
// 8..15: marginal for head h).  For a group-coherent map (one row) this is
// exactly the group's union, so every K/V row is read from HBM once; for a
// non-coherent map a position chosen by two rows is read twice.
// The list is split over the gridDim.x CTAs of a cluster in byte-balanced
// shares; the plan kernel (K3a) pre-stages each share's first batch (pool row
// offsets, head masks, marginal weights), then every warp streams its own
// 8 KB tiles — 16 K+V rows (recent / critical) or 32 V rows (marginal) — with
// cp.async (4 rows x 128 B per instruction, XOR-swizzled, zero-filled tails)
// through a private 3-stage ring
// and runs on the tensor cores (mma.sync m16n8k16) in the transposed
// orientation, so no MMA row is spent on absent heads (a kv-group has G <= 8
// q-heads, the MMA's M is 16):
//   S^T[16 tok x 8 heads]  = K_tile[16 x d] · Q_group^T      (8 MMAs for d=128)
//   O_c^T[d x 8 heads]    += V_tile^T · P^T                  (softmax weights p)
//   O_m^T[d x 8 heads]    += V_tile^T · A'^T                 (marginal weights a')
// P^T leaves the QK accumulators in (token, head) order; movmatrix transposes
// its bf16 pairs into the B-operand layout.  Weights are split into bf16
// hi + lo parts (two MMAs) to keep ~2^-17 relative precision.  The online
// softmax is lazy: a head's base is raised (with the O rescale) only when a
// score exceeds it by more than 8 (log2 units) — one warp vote per tile in the
// common case.  Warps merge in shared memory in a fixed order; the CTAs of a
// group merge through distributed shared memory in rank order (K4 fused):
// bit-reproducible.
#include <float.h>
#include <limits.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace skv {

#ifdef SKV_TRACE
__device__ long long* g_trace = nullptr;
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// record of CTA `cta` of layer `skv_tl`: kTraceSlots int64 (tools/attend_trace.py):
// 0-8 globaltimer ns at the SKV_T points, 10 entries of the share, 11 SM id,
// 12 ns thread 0 spent in CTA-synchronous batch staging, 13 batches
constexpr int kTraceSlots = 16;
#define SKV_TS(i, v)                                                                     \
  if (g_trace && threadIdx.x == 0) {                                                     \
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;      \
    g_trace[(static_cast<int64_t>(skv_tl) * 4096 + cta) * kTraceSlots + (i)] = (v);      \
  }
#define SKV_T(i) SKV_TS(i, gtimer())
#else
#define SKV_T(i)
#define SKV_TS(i, v)
#endif

namespace {
constexpr int kTile = 16;      // rows (tokens) per warp tile
#ifndef SKV_ATTEND_WARPS
#define SKV_ATTEND_WARPS 8
#endif
#ifndef SKV_ATTEND_STAGES
#define SKV_ATTEND_STAGES 3
#endif
constexpr int kWarps = SKV_ATTEND_WARPS;      // one CTA per SM (8 warps x 3-stage rings = 192 KB)
constexpr int kThreads = kWarps * 32;
constexpr int kBatch = 1024;   // entries whose positions/pages/weights are staged at once
constexpr int kAsyncStageMinLen = 8192;   // contexts above this stage their batches asynchronously

template <int D>
constexpr int stages_for() { return SKV_ATTEND_STAGES; }
template <int D>
constexpr int stage_bytes() { return 2 * kTile * D * 2; }

// [row offset][mask][weight]: kBatch each (batch buffer 0) | stages (kWarps x
// NSTAGE) | batch buffer 1 (the next batch is staged while this one streams) |
// page-table scratch of the batch being staged
template <int D>
constexpr size_t smem_bytes() {
  return 2 * static_cast<size_t>(kBatch) * 12 + static_cast<size_t>(kBatch) * 4 +
         static_cast<size_t>(kWarps) * stages_for<D>() * stage_bytes<D>();
}

// Lazy online softmax: the running max used as the exponent base is only
// raised when a new score exceeds it by more than this (log2 units), so the
// O rescale is skipped for almost every tile; exp2 arguments stay <= 8.
constexpr float kRescaleSlack = 8.f;

// Layout of one (layer, sequence, kv-group) virtual list:
//   [ recent Rc | crit(r_0) | marg(r_0) | crit(r_1) | marg(r_1) | ... ]
struct GroupLayout {
  int T, nrows, Rc, n;
  int rj[8], rK[8], rM[8];
  uint32_t rhm[8];
};
constexpr int kHdrBytes = 256;
static_assert(sizeof(GroupLayout) <= kHdrBytes && sizeof(GroupLayout) % 16 == 0, "plan header");

// Plan record of one (layer, sequence, kv-group): header + for each cluster
// rank the first kBatch staged entries (row offset, head mask, marginal weight).
// Tile table of one batch: word 0 = the tile count, then one packed word per
// tile; kTileTableBytes per cluster rank in the plan record (first batch).
constexpr int kMaxTiles = kBatch / kTile + 2 * 8 + 2;
constexpr int kTileTableBytes = 384;
static_assert((kMaxTiles + 1) * 4 <= kTileTableBytes && kTileTableBytes % 16 == 0, "tile table");
__host__ __device__ constexpr int64_t plan_record_bytes(int nc) {
  return kHdrBytes + static_cast<int64_t>(nc) * (kTileTableBytes + kBatch * 12);
}
// record layout: [header][tile tables: nc x kTileTableBytes][slots: nc x kBatch x 12]
__host__ __device__ constexpr int64_t plan_slot_offset(int nc, int c) {
  return kHdrBytes + static_cast<int64_t>(nc) * kTileTableBytes + static_cast<int64_t>(c) * kBatch * 12;
}

// All threads: distinct SLM rows of the group's heads (first occurrence order)
// and the list sizes.  K' and M' follow from the sequence's budgets with the
// clamp of R5 (the same values smallkv_select writes to `counts`), so one round
// of independent loads suffices.
__device__ void build_layout(const AttendParams& p, int layer, int b, int g, GroupLayout& L) {
  __shared__ int s_j[8];
  const int G = p.heads / p.kv_heads;
  const int tid = threadIdx.x;
  if (tid < G) s_j[tid] = p.head_map[layer * p.heads + g * G + tid];
  if (tid == 32) {
    const int n = p.seq_lens[b];
    const int Rc = min(max(p.n_recent[b], 0), n);
    const int Kc = min(min(max(p.k_crit[b], 0), n - Rc), p.max_crit);
    const int Mc = min(min(max(p.k_marg[b], 0), n - Rc - Kc), p.max_marg);
    L.n = n;
    L.Rc = Rc;
    L.rK[0] = Kc;   // temporarily: the per-row sizes
    L.rM[0] = Mc;
  }
  __syncthreads();
  if (tid == 0 && p.group_sel) {
    // variant f2: one shared selection row per (layer, kv-group), all heads
    L.rj[0] = layer * p.kv_heads + g;
    L.rhm[0] = (1u << G) - 1u;
    L.nrows = 1;
    L.T = L.Rc + L.rK[0] + L.rM[0];
  } else if (tid == 0) {
    const int Kc = L.rK[0], Mc = L.rM[0];
    int nr = 0;
    for (int h = 0; h < G; ++h) {
      int k = 0;
      while (k < nr && L.rj[k] != s_j[h]) ++k;
      if (k == nr) {
        L.rj[nr] = s_j[h];
        L.rhm[nr] = 0u;
        ++nr;
      }
      L.rhm[k] |= 1u << h;
    }
    for (int k = 0; k < nr; ++k) {
      L.rK[k] = Kc;
      L.rM[k] = Mc;
    }
    L.nrows = nr;
    L.T = L.Rc + nr * (Kc + Mc);
  }
  __syncthreads();
}

// First entry of cluster rank c's share of the group's list.  Shares are
// balanced by BYTES, not entries: a critical/recent entry reads K and V (weight
// 2), a marginal one only V (weight 1); rank c starts at the first entry whose
// cumulative weight reaches floor(W * c / NC).
__device__ __forceinline__ int split_begin(const GroupLayout& L, int c, int NC) {
  int64_t W = 2 * static_cast<int64_t>(L.Rc);
  for (int k = 0; k < L.nrows; ++k) W += 2 * static_cast<int64_t>(L.rK[k]) + L.rM[k];
  const int64_t target = (W * c) / NC;
  int64_t w = 0;
  int x = 0;
  auto seg = [&](int len, int weight, int& out) -> bool {
    const int64_t sw = static_cast<int64_t>(len) * weight;
    if (w + sw >= target) {
      out = x + static_cast<int>((target - w + weight - 1) / weight);
      return true;
    }
    w += sw;
    x += len;
    return false;
  };
  int out = 0;
  if (seg(L.Rc, 2, out)) return out;
  for (int k = 0; k < L.nrows; ++k) {
    if (seg(L.rK[k], 2, out)) return out;
    if (seg(L.rM[k], 1, out)) return out;
  }
  return x;
}

// First entry of share q of group grp = b * H_kv + g.  Per-group ranks
// (flat_shares == 0): rank q of NC, split_begin above.  Stream-K
// (flat_shares == S > #groups Gt): CTA s owns the interval [s*Gt, (s+1)*Gt) of
// the line where group grp is [grp*S, (grp+1)*S), every group's bytes being
// one unit; share q of grp is its intersection with CTA floor(grp*S/Gt) + q,
// so its boundaries are the byte-balanced points (s*Gt - grp*S) / S.
template <bool kFlat = true>
__device__ __forceinline__ int share_begin(const AttendParams& p, const GroupLayout& L, int grp, int q,
                                           int NC) {
  if (!kFlat || p.flat_shares == 0) return split_begin(L, q, NC);
  const int64_t S = p.flat_shares, Gt = static_cast<int64_t>(p.batch) * p.kv_heads;
  const int64_t s_first = grp * S / Gt;
  int64_t num = q == 0 ? 0 : (s_first + q) * Gt - grp * S;
  if (num > S) num = S;
  return split_begin(L, static_cast<int>(num), static_cast<int>(S));
}

// One thread: the tile table of entries [e_b, e_b + E) of the group's list —
// runs of K+V entries (recent / critical) in 16-row tiles, runs of V-only
// (marginal) entries in 32-row tiles (both fill one 8 KB stage, so the tile
// count tracks the bytes); variant f2: marginal runs in 16-row tiles whose K
// half carries the per-head weights.  tt[0] = count, tt[1 + i] = tile i packed
// (first entry - e_b) | count << 16 | vonly << 24 | per-head << 25.
__device__ void build_tile_table(const GroupLayout& L, int e_b, int E, bool group_sel, uint32_t* tt) {
  int nt = 0, x = 0;
  const uint32_t mflag = group_sel ? (1u << 25) : (1u << 24);
  auto run = [&](int len, bool vonly) {
    const int a = max(x, e_b), z = min(x + len, e_b + E);
    const int ts = vonly && !group_sel ? 2 * kTile : kTile;
    for (int y = a; y < z; y += ts)
      tt[1 + nt++] = static_cast<uint32_t>(y - e_b) | (static_cast<uint32_t>(min(ts, z - y)) << 16) |
                     (vonly ? mflag : 0u);
    x += len;
  };
  run(L.Rc, false);
  for (int k = 0; k < L.nrows; ++k) {
    run(L.rK[k], false);
    run(L.rM[k], true);
  }
  tt[0] = static_cast<uint32_t>(nt);
}

// Entry x of a group's virtual list [recent | crit(r_0) | marg(r_0) | crit(r_1) | ...]:
// its position, head mask (bits 0..7 critical, 8..15 marginal), and the
// marginal weight of a per-row selection (0 for recent / critical entries and
// for group selections, whose per-head weights live elsewhere).
struct ListEntry {
  int pos;
  uint32_t mask;
  float w;
};
__device__ __forceinline__ ListEntry list_entry(const AttendParams& p, const GroupLayout& L, int b,
                                                int x, uint32_t allc) {
  if (x < L.Rc) return {L.n - L.Rc + x, allc, 0.f};
  x -= L.Rc;
  int k = 0;
  while (k < L.nrows - 1 && x >= L.rK[k] + L.rM[k]) {
    x -= L.rK[k] + L.rM[k];
    ++k;
  }
  const int64_t rb = static_cast<int64_t>(L.rj[k]) * p.batch + b;
  if (x < L.rK[k]) return {__ldg(p.crit_idx + rb * p.max_crit + x), L.rhm[k], 0.f};
  const int m = x - L.rK[k];
  return {__ldg(p.marg_idx + rb * p.max_marg + m), L.rhm[k] << 8,
          p.group_sel ? 0.f : __ldg(p.marg_w + rb * p.max_marg + m)};
}

// All threads: stage entries [e_b, e_b + E) of the group's virtual list:
// row offset in the layer's pool (elements), head mask, marginal weight.
// Two dependent rounds of loads (list values, page table).
template <int D>
__device__ void stage_entries(const AttendParams& p, const GroupLayout& L, int b, int g, int e_b,
                              int E, uint32_t* soff, uint32_t* smk, float* sw) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int G = p.heads / p.kv_heads;
  const uint32_t allc = (1u << G) - 1u;
  for (int i = tid; i < E; i += nthr) {
    const ListEntry le = list_entry(p, L, b, e_b + i, allc);
    soff[i] = static_cast<uint32_t>(le.pos);
    smk[i] = le.mask;
    sw[i] = le.w;
  }
  __syncthreads();
  if (p.entry_slot) {
    // variant f4: rows live in the group's hot-pool slots
    const int32_t* es = p.entry_slot + ((static_cast<int64_t>(p.layer) * p.batch + b) * p.kv_heads + g) * p.hot_cap;
    for (int i = tid; i < E; i += nthr)
      soff[i] = static_cast<uint32_t>(((static_cast<int64_t>(b) * p.kv_heads + g) * p.hot_cap + __ldg(es + e_b + i)) * D);
    __syncthreads();
    return;
  }
  const int32_t* bt = p.block_table + static_cast<int64_t>(b) * p.max_blocks;
  for (int i = tid; i < E; i += nthr) {
    const int pos = static_cast<int>(soff[i]);
    const int page = __ldg(bt + (pos >> p.ps_shift));
    soff[i] = static_cast<uint32_t>(
        ((static_cast<int64_t>(page) * p.kv_heads + g) * p.page_size + (pos & (p.page_size - 1))) * D);
  }
  __syncthreads();
}

// K3a — gather plan for every layer of the step (one launch after select):
// CTA (g, layer*B + b) stages the first batch of every cluster rank's share
// of the group's list: 2 rounds of loads, 4 entries in flight per thread.
#ifndef SKV_PLAN_THREADS
#define SKV_PLAN_THREADS 128
#endif
constexpr int kPlanThreads = SKV_PLAN_THREADS;
template <int D>
__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const AttendParams p) {
  __shared__ __align__(16) GroupLayout L;
  const int g = blockIdx.x;
  const int layer = blockIdx.y / p.batch, b = blockIdx.y % p.batch;
  const int NC = p.max_chunks;
  const int G = p.heads / p.kv_heads;
  const uint32_t allc = (1u << G) - 1u;
  // the first attend of the step may be scheduled during this grid's tail: it
  // runs without the overlap flag, so it waits for our completion before
  // reading the plan (include/smallkv.h, smallkv_attend `flags`)
  griddep_launch_dependents();
  griddep_wait();
  build_layout(p, layer, b, g, L);
  uint8_t* rec = p.plan + ((static_cast<int64_t>(layer) * p.batch + b) * p.kv_heads + g) *
                              plan_record_bytes(NC);
  // this CTA's ranks [c_lo, c_hi) of the record (blockIdx.z: a group's list
  // split over many ranks — small batches — is staged by several CTAs)
  const int per = (NC + static_cast<int>(gridDim.z) - 1) / static_cast<int>(gridDim.z);
  const int c_lo = static_cast<int>(blockIdx.z) * per, c_hi = min(NC, c_lo + per);
  if (blockIdx.z == 0 && threadIdx.x < sizeof(GroupLayout) / 4)
    reinterpret_cast<int*>(rec)[threadIdx.x] = reinterpret_cast<const int*>(&L)[threadIdx.x];
  // variant f4: a list longer than the hot pool was skipped by tier_update (its
  // entry slots are stale); the header alone tells the attend to write NaN
  if ((p.entry_slot && L.T > p.hot_cap) || c_lo >= c_hi) return;
  const int nr = c_hi - c_lo;
  const int32_t* bt = p.block_table + static_cast<int64_t>(b) * p.max_blocks;
  // flattened over the group's list: entry x belongs to the rank whose
  // byte-balanced share contains it and is staged if it is in that rank's
  // first batch (s_split[k] = start of rank c_lo + k)
  __shared__ int s_split[33];
  if (threadIdx.x <= nr) s_split[threadIdx.x] = share_begin(p, L, b * p.kv_heads + g, c_lo + threadIdx.x, NC);
  __syncthreads();
  // only the staged entries are visited: flattened over the ranks' first
  // batches (s_pre[k] = staged entries of this CTA's ranks before c_lo + k)
  // (thread 32: the tile-table builders below are threads < nr <= 32, and
  // their serial builds overlap the staging loop)
  __shared__ int s_pre[33];
  if (threadIdx.x == 32) {
    int a = 0;
    for (int k = 0; k < nr; ++k) {
      s_pre[k] = a;
      a += min(kBatch, s_split[k + 1] - s_split[k]);
    }
    s_pre[nr] = a;
  }
  __syncthreads();
  if (threadIdx.x < nr) {   // each rank's first-batch tile table
    const int k = threadIdx.x, e0 = s_split[k];
    build_tile_table(L, e0, min(kBatch, s_split[k + 1] - e0), p.group_sel != 0,
                     reinterpret_cast<uint32_t*>(rec + kHdrBytes + (c_lo + k) * kTileTableBytes));
  }
  constexpr int U = 1024 / kPlanThreads;
  const int F = s_pre[nr];
  if (nr == 1 && !p.entry_slot) {
    // one rank (every CTA unless a record's two ranks share it): entries
    // x0 = split + f, one slot array, no rank search per entry
    const int x_base = s_split[0];
    uint32_t* slot = reinterpret_cast<uint32_t*>(rec + plan_slot_offset(NC, c_lo));
    for (int base = threadIdx.x; base < F; base += U * kPlanThreads) {
      int pos[U];
      uint32_t mk[U];
      float wt[U];
      if (L.nrows == 1) {
        // one SLM row (group-coherent maps): list bases hoisted out of the entries
        const int64_t rb0 = static_cast<int64_t>(L.rj[0]) * p.batch + b;
        const int32_t* cb = p.crit_idx + rb0 * p.max_crit;
        const int32_t* mb = p.marg_idx + rb0 * p.max_marg;
        const float* wb = p.marg_w + rb0 * p.max_marg;
        const int Rc = L.Rc, K0 = L.rK[0], n0 = L.n - L.Rc;
        const uint32_t hm = L.rhm[0];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int f = base + u * kPlanThreads;
          const int x = x_base + f;
          pos[u] = 0;
          mk[u] = 0u;
          wt[u] = 0.f;
          if (f < F) {
            if (x < Rc) {
              pos[u] = n0 + x;
              mk[u] = allc;
            } else if (x - Rc < K0) {
              pos[u] = __ldg(cb + (x - Rc));
              mk[u] = hm;
            } else {
              pos[u] = __ldg(mb + (x - Rc - K0));
              mk[u] = hm << 8;
              wt[u] = p.group_sel ? 0.f : __ldg(wb + (x - Rc - K0));
            }
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int f = base + u * kPlanThreads;
          pos[u] = 0;
          mk[u] = 0u;
          wt[u] = 0.f;
          if (f < F) {
            const ListEntry le = list_entry(p, L, b, x_base + f, allc);
            pos[u] = le.pos;
            mk[u] = le.mask;
            wt[u] = le.w;
          }
        }
      }
      int page[U];
#pragma unroll
      for (int u = 0; u < U; ++u) page[u] = base + u * kPlanThreads < F ? __ldg(bt + (pos[u] >> p.ps_shift)) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int f = base + u * kPlanThreads;
        if (f >= F) continue;
        slot[f] = static_cast<uint32_t>(((static_cast<int64_t>(page[u]) * p.kv_heads + g) * p.page_size +
                                         (pos[u] & (p.page_size - 1))) * D);
        slot[kBatch + f] = mk[u];
        reinterpret_cast<float*>(slot)[2 * kBatch + f] = wt[u];
      }
    }
    return;
  }
  for (int base = threadIdx.x; base < F; base += U * kPlanThreads) {
    int pos[U], slot_i[U];
    uint32_t mk[U];
    float wt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int f = base + u * kPlanThreads;
      slot_i[u] = -1;
      pos[u] = 0;
      mk[u] = 0u;
      wt[u] = 0.f;
      if (f >= F) continue;
      int k = 0;
      while (k < nr - 1 && f >= s_pre[k + 1]) ++k;
      const int i = f - s_pre[k];
      const int x0 = s_split[k] + i;
      slot_i[u] = k * kBatch + i;   // (local rank k: rank c_lo + k)
      const ListEntry le = list_entry(p, L, b, x0, allc);
      pos[u] = le.pos;
      mk[u] = le.mask;
      wt[u] = le.w;
    }
    uint32_t ro[U];
    if (p.entry_slot) {
      // variant f4: the entry's hot-pool slot, row ((b*H_kv + g)*cap + slot)
      const int32_t* es = p.entry_slot + ((static_cast<int64_t>(layer) * p.batch + b) * p.kv_heads + g) * p.hot_cap;
#pragma unroll
      for (int u = 0; u < U; ++u)
        ro[u] = slot_i[u] < 0 ? 0u : static_cast<uint32_t>(
            ((static_cast<int64_t>(b) * p.kv_heads + g) * p.hot_cap + __ldg(es + s_split[slot_i[u] / kBatch] + slot_i[u] % kBatch)) * D);
    } else {
      int page[U];
#pragma unroll
      for (int u = 0; u < U; ++u) page[u] = slot_i[u] >= 0 ? __ldg(bt + (pos[u] >> p.ps_shift)) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        ro[u] = static_cast<uint32_t>(((static_cast<int64_t>(page[u]) * p.kv_heads + g) * p.page_size +
                                       (pos[u] & (p.page_size - 1))) * D);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (slot_i[u] < 0) continue;
      const int c = c_lo + slot_i[u] / kBatch, i = slot_i[u] % kBatch;
      uint32_t* slot = reinterpret_cast<uint32_t*>(rec + plan_slot_offset(NC, c));
      slot[i] = ro[u];
      slot[kBatch + i] = mk[u];
      reinterpret_cast<float*>(slot)[2 * kBatch + i] = wt[u];
    }
  }
}

// kAsync: batch x+1 is staged asynchronously during batch x (long lists);
// otherwise CTA-synchronously at the start of batch x (short lists rarely have
// a second batch, and the leaner kernel keeps fewer registers live)
// One share (c of the group's NC record slots) of group (b, g); nmerge = the
// group's shares that the global merge waits for (= NC unless stream-K).
template <int D, bool kAsync, bool kFlat>
__device__ __forceinline__ void attend_share(const AttendParams& p, const int c, const int g, const int b,
                                             const int NC, const int nmerge) {
  constexpr int NSTAGE = stages_for<D>();
  constexpr int ROWB = D * 2;                // bytes per K or V row
  constexpr int KV_BYTES = kTile * ROWB;
  constexpr int SB = stage_bytes<D>();

  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* soff = reinterpret_cast<uint32_t*>(smem);   // row offset in the layer's pool (elements)
  uint32_t* smk = soff + kBatch;
  float* sw = reinterpret_cast<float*>(smk + kBatch);
  uint8_t* stages = reinterpret_cast<uint8_t*>(sw + kBatch);
  // batch buffers: x & 1 selects [row offset | mask | weight] and the tile table
  uint32_t* soff1 = reinterpret_cast<uint32_t*>(stages + static_cast<size_t>(kWarps) * NSTAGE * SB);
  __shared__ __align__(16) GroupLayout L;
  __shared__ __align__(16) uint32_t s_tt[kTileTableBytes / 4];    // [count][tiles], batch buffer 0
  __shared__ __align__(16) uint32_t s_tt1[kTileTableBytes / 4];   // batch buffer 1
  __shared__ __align__(8) uint64_t bar_staged[2];                  // batch buffer b staged
  int32_t* spg = reinterpret_cast<int32_t*>(soff1 + 3 * kBatch);   // [kBatch] pages / slots
  auto BOFF = [&](int x) { return (x & 1) ? soff1 : soff; };
  auto BMK = [&](int x) { return (x & 1) ? soff1 + kBatch : smk; };
  auto BW = [&](int x) { return reinterpret_cast<float*>((x & 1) ? soff1 + 2 * kBatch : smk + kBatch); };
  auto BTT = [&](int x) { return (x & 1) ? s_tt1 : s_tt; };

  // Without the overlap flag nothing is read before the previous kernel on the
  // stream has completed.  With it, the prologue below (plan / selection
  // outputs, page tables, K/V tiles) may run during that kernel's tail.
#ifdef SKV_TRACE
  const int skv_tl = p.layer;   // trace slot (diagnostic builds only)
  long long skv_stage_ns = 0;
#endif
  SKV_T(7);
  if (!p.overlap_prologue) griddep_wait();
  SKV_T(0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = p.heads / p.kv_heads;
  const uint8_t* rec = p.plan ? p.plan + ((static_cast<int64_t>(p.layer) * p.batch + b) *
                                              p.kv_heads + g) * plan_record_bytes(NC)
                              : nullptr;
  uint8_t* wst = stages + warp * NSTAGE * SB;
  const uint16_t* kpool = p.k + p.layer_offset;
  const uint16_t* vpool = p.v + p.layer_offset;
  if (rec) {
    // one round: header + this rank's pre-staged first batch (cp.async, 16 B)
    for (int i = tid; i < static_cast<int>(sizeof(GroupLayout)) / 16; i += kThreads)
      cp_async16(smem_u32(reinterpret_cast<uint8_t*>(&L) + 16 * i), rec + 16 * i, true);
    const uint8_t* tts = rec + kHdrBytes + static_cast<int64_t>(c) * kTileTableBytes;
    for (int i = tid; i < kTileTableBytes / 16; i += kThreads)
      cp_async16(smem_u32(reinterpret_cast<uint8_t*>(s_tt) + 16 * i), tts + 16 * i, true);
    const uint8_t* slot = rec + plan_slot_offset(NC, c);
    for (int i = tid; i < kBatch * 12 / 16; i += kThreads)
      cp_async16(smem_u32(smem + 16 * i), slot + 16 * i, true);
    cp_async_commit();
    // the next layer's record of this (sequence, group, rank) -> L2: the plan of
    // all layers is written once per step, so by a late layer it has been
    // evicted by the K/V stream and its read would otherwise be an HBM miss on
    // that launch's critical path
    if (p.layer + 1 < p.n_layers) {
      const uint8_t* nx = rec + static_cast<int64_t>(p.batch) * p.kv_heads * plan_record_bytes(NC);
      constexpr int kHdrLines = (kHdrBytes + kTileTableBytes) / 128 + 1;
      if (tid < kHdrLines + kBatch * 12 / 128) {
        const uint8_t* a = tid < kHdrLines
                               ? nx + (tid < kHdrBytes / 128 ? 128 * tid
                                                             : kHdrBytes + static_cast<int64_t>(c) * kTileTableBytes +
                                                                   128 * (tid - kHdrBytes / 128))
                               : nx + plan_slot_offset(NC, c) + 128 * (tid - kHdrLines);
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a));
      }
    }
  }
  // Early tiles (issued after the plan copy, waited for separately): the list starts with the recent window [n-R', n), whose rows
  // need only the sequence length, the recent budget and the block table
  // (small, L2-resident) — so a single-CTA group issues its first tiles'
  // K/V copies before (and in parallel with) the plan / list loads.
  int early = 0;
  if (NC == 1 && !p.entry_slot) {
    const int n = p.seq_lens[b];
    const int Rc = min(max(p.n_recent[b], 0), n);
    const int32_t* bt = p.block_table + static_cast<int64_t>(b) * p.max_blocks;
    constexpr int NE = NSTAGE - 1;
    int ne = 0;   // early stages of this warp: tiles warp + i*kWarps of the recent run
#pragma unroll
    for (int i = 0; i < NE; ++i)
      if (kTile * (warp + i * kWarps) < Rc && ne == i) ne = i + 1;
    // every page-table entry first (one round trip), then the copies
    int page[NE][kTile / 4];
#pragma unroll
    for (int i = 0; i < NE; ++i)
#pragma unroll
      for (int grp = 0; grp < kTile / 4; ++grp) {
        const int j = warp + i * kWarps;
        const int eo = grp * 4 + (lane >> 3);
        const int pos = n - Rc + kTile * j + eo;
        page[i][grp] = (i < ne && kTile * j + eo < Rc) ? __ldg(bt + (pos >> p.ps_shift)) : 0;
      }
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      if (i >= ne) break;
      const int j = warp + i * kWarps;
      const int cnt = min(kTile, Rc - kTile * j);
      uint8_t* st = wst + i * SB;
#pragma unroll
      for (int grp = 0; grp < kTile / 4; ++grp) {
        const int eo = grp * 4 + (lane >> 3);
        const bool ev = eo < cnt;
        const int pos = n - Rc + kTile * j + eo;
        const uint32_t ro = ev ? static_cast<uint32_t>(
                                     ((static_cast<int64_t>(page[i][grp]) * p.kv_heads + g) * p.page_size +
                                      (pos & (p.page_size - 1))) * D)
                               : 0u;
#pragma unroll
        for (int hf = 0; hf < D / 64; ++hf) {
          const int ch = hf * 8 + (lane & 7);
          const int sw_ = (ch ^ (eo & 7)) << 4;
          if (ev) cp_async16(smem_u32(st + eo * ROWB + sw_), kpool + ro + ch * 8, true);
          cp_async16(smem_u32(st + KV_BYTES + eo * ROWB + sw_), vpool + ro + ch * 8, ev);
        }
      }
      cp_async_commit();
      ++early;
    }
  }
  if (tid == 0) {
    mbar_init(&bar_staged[0], kThreads);
    mbar_init(&bar_staged[1], kThreads);
    fence_barrier_init();
  }
  if (rec) {
    // wait for the plan group only (the oldest); the early tiles stay in flight
    if (early == 3) cp_async_wait<3>();
    else if (early == 2) cp_async_wait<2>();
    else if (early == 1) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
  } else {
    build_layout(p, p.layer, b, g, L);
  }
  const int T = L.T;
  if (p.entry_slot && T > p.hot_cap) {
    // variant f4 capacity overflow: tier_update skipped this group, so its
    // entry slots are stale; nothing is read and the outputs are NaN
    cp_async_wait<0>();
    griddep_wait();
    griddep_launch_dependents();
    if (c == 0) {
      const int64_t bo = static_cast<int64_t>(b) * p.heads + g * G;
      for (int i = tid; i < G * D; i += kThreads) p.out[bo * D + i] = __int_as_float(0x7fc00000);
    }
    return;
  }
  const int e_lo = share_begin<kFlat>(p, L, b * p.kv_heads + g, c, NC);
  const int e_hi = share_begin<kFlat>(p, L, b * p.kv_heads + g, c + 1, NC);
  (void)T;
  SKV_T(1);

  const int gq = lane >> 2, tq = lane & 3;

  uint32_t qa[D / 16][2];
  bool q_ready = false;
  // q (and, in a real model, everything the previous kernel produces) is read
  // only after the programmatic grid dependency is resolved.
  auto wait_and_load_q = [&]() {
    griddep_wait();
    griddep_launch_dependents();
    const uint16_t* qg = p.q + (static_cast<int64_t>(b) * p.heads + g * G) * D;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int cc = 16 * kk + 2 * tq;
      qa[kk][0] = gq < G ? *reinterpret_cast<const uint32_t*>(qg + gq * D + cc) : 0u;
      qa[kk][1] = gq < G ? *reinterpret_cast<const uint32_t*>(qg + gq * D + cc + 8) : 0u;
    }
    q_ready = true;
  };

  // O^T accumulators (MMA rows = d, columns = heads): lane holds d = 16*mt +
  // gq (+8) for heads 2*tq, 2*tq+1.  oc: softmax part (critical ∪ recent),
  // om: marginal compensation (Eq. 6 second branch).
  constexpr int MT = D / 16;
  float oc[MT][4], om[MT][4];
#pragma unroll
  for (int t = 0; t < MT; ++t) {
    oc[t][0] = oc[t][1] = oc[t][2] = oc[t][3] = 0.f;
    om[t][0] = om[t][1] = om[t][2] = om[t][3] = 0.f;
  }
  // running max (log2 units) and partial sums of this lane's heads 2tq, 2tq+1
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int mi = lane >> 3;
  const int h0 = 2 * tq, h1 = 2 * tq + 1;

  // ---- the share's entries in batches of kBatch, double-buffered: batch x+1
  // is staged (list values, page table -> row offsets, tile table) into the
  // other buffer at the start of batch x, while batch x's first tiles are in
  // flight, and each warp's cp.async ring runs on into batch x+1's first tiles
  // during batch x's last ones (no drain at the batch boundary).
  const int nbatch = e_hi > e_lo ? (e_hi - e_lo + kBatch - 1) / kBatch : 0;
  auto nmy_of = [&](int x) {
    const int nt = static_cast<int>(BTT(x)[0]);
    return nt > warp ? (nt - warp + kWarps - 1) / kWarps : 0;
  };
  // batch 0: pre-staged by the plan kernel (an empty share has an empty tile
  // table there), or staged now
  if (!rec) {
    if (nbatch > 0) {
      stage_entries<D>(p, L, b, g, e_lo, min(kBatch, e_hi - e_lo), soff, smk, sw);
      if (tid == 0) build_tile_table(L, e_lo, min(kBatch, e_hi - e_lo), p.group_sel != 0, s_tt);
    } else if (tid == 0) {
      s_tt[0] = 0u;
    }
    __syncthreads();
  }
  SKV_T(2);

  // Full tiles (all but a run's last) take a lean issue path: per lane the
  // shared-memory offsets (row, swizzled 16-B chunk) and the chunk's byte
  // offset in a row are fixed, so each 16-B copy is one add and one LDGSTS
  // with no zero-fill predicate.
  constexpr int HV = D / 64;   // 128-byte halves of a row
  const uint32_t wst_u32 = smem_u32(wst);
  const int lr = lane >> 3, lc = lane & 7;
  uint32_t ldst[HV][2];   // [half][tile group parity]: row lr of the group, swizzled chunk
  uint32_t lsrc[HV];      // the chunk's byte offset in a row
#pragma unroll
  for (int hf = 0; hf < HV; ++hf) {
    lsrc[hf] = static_cast<uint32_t>((hf * 8 + lc) * 16);
#pragma unroll
    for (int par = 0; par < 2; ++par)
      ldst[hf][par] = static_cast<uint32_t>(lr * ROWB + (((hf * 8 + lc) ^ (par * 4 + lr)) << 4));
  }
  const char* kpool_b = reinterpret_cast<const char*>(kpool);
  const char* vpool_b = reinterpret_cast<const char*>(vpool);
  auto issue = [&](int x, int j, int slot) {
    if (x >= 0) {
      uint8_t* st = wst + (slot % NSTAGE) * SB;
      const uint32_t* xoff = BOFF(x);
      const int e_b = e_lo + x * kBatch;
      const uint32_t td = BTT(x)[1 + warp + j * kWarps];
      const int e0 = static_cast<int>(td & 0xffffu), cnt = static_cast<int>((td >> 16) & 0xffu);
      const uint32_t stb = wst_u32 + static_cast<uint32_t>((slot % NSTAGE) * SB);
      if (!(td >> 24) && cnt == kTile) {
        // full K+V tile: 16 rows, K half then V half
#pragma unroll
        for (int grp = 0; grp < kTile / 4; ++grp) {
          const size_t rb = static_cast<size_t>(xoff[e0 + grp * 4 + lr]) * 2;
#pragma unroll
          for (int hf = 0; hf < HV; ++hf) {
            const uint32_t d = stb + grp * 4 * ROWB + ldst[hf][grp & 1];
            cp_async16_full(d, kpool_b + rb + lsrc[hf]);
            cp_async16_full(d + KV_BYTES, vpool_b + rb + lsrc[hf]);
          }
        }
        cp_async_commit();
        return;
      }
      if ((td >> 24) == 1u && cnt == 2 * kTile) {
        // full V-only tile: 32 V rows fill the stage
#pragma unroll
        for (int grp = 0; grp < 2 * kTile / 4; ++grp) {
          const size_t rb = static_cast<size_t>(xoff[e0 + grp * 4 + lr]) * 2;
#pragma unroll
          for (int hf = 0; hf < HV; ++hf)
            cp_async16_full(stb + grp * 4 * ROWB + ldst[hf][grp & 1], vpool_b + rb + lsrc[hf]);
        }
        cp_async_commit();
        return;
      }
      if (td >> 25) {
        // f2 marginal tile: 16 V rows in the V half, their per-head weights
        // [16][8] fp32 (512 B) at the start of the K half
#pragma unroll
        for (int grp = 0; grp < kTile / 4; ++grp) {
          const int eo = grp * 4 + (lane >> 3);
          const bool ev = eo < cnt;
          const uint32_t ro = ev ? xoff[e0 + eo] : 0u;
#pragma unroll
          for (int hf = 0; hf < D / 64; ++hf) {
            const int ch = hf * 8 + (lane & 7);
            cp_async16(smem_u32(st + KV_BYTES + eo * ROWB + ((ch ^ (eo & 7)) << 4)), vpool + ro + ch * 8, ev);
          }
        }
        const int eo = lane >> 1;
        const int64_t m = static_cast<int64_t>(e_b + e0 + eo) - (L.Rc + L.rK[0]);
        const float* src = p.marg_w + ((static_cast<int64_t>(L.rj[0]) * p.batch + b) * p.max_marg + m) * 8 +
                           (lane & 1) * 4;
        cp_async16(smem_u32(st + lane * 16), eo < cnt ? src : p.marg_w, eo < cnt);
      } else if (td >> 24) {
        // V-only tile: 32 V rows fill the stage
#pragma unroll
        for (int grp = 0; grp < 2 * kTile / 4; ++grp) {
          const int eo = grp * 4 + (lane >> 3);
          const bool ev = eo < cnt;
          const uint32_t ro = ev ? xoff[e0 + eo] : 0u;
#pragma unroll
          for (int hf = 0; hf < D / 64; ++hf) {
            const int ch = hf * 8 + (lane & 7);
            cp_async16(smem_u32(st + eo * ROWB + ((ch ^ (eo & 7)) << 4)), vpool + ro + ch * 8, ev);
          }
        }
      } else {
#pragma unroll
        for (int grp = 0; grp < kTile / 4; ++grp) {
          const int eo = grp * 4 + (lane >> 3);
          const bool ev = eo < cnt;
          const uint32_t ro = ev ? xoff[e0 + eo] : 0u;
#pragma unroll
          for (int hf = 0; hf < D / 64; ++hf) {
            const int ch = hf * 8 + (lane & 7);
            const int sw_ = (ch ^ (eo & 7)) << 4;
            if (ev) cp_async16(smem_u32(st + eo * ROWB + sw_), kpool + ro + ch * 8, true);
            cp_async16(smem_u32(st + KV_BYTES + eo * ROWB + sw_), vpool + ro + ch * 8, ev);
          }
        }
      }
    }
    cp_async_commit();
  };


  int tbase = 0;   // tiles this warp consumed in earlier batches (ring slots)
  {
    const int nmy0 = nbatch > 0 ? nmy_of(0) : 0;
#pragma unroll
    for (int i = 0; i < NSTAGE - 1; ++i)
      if (!(i < early)) issue(i < nmy0 ? 0 : -1, i, i);   // the early tiles are in flight already
  }
  if (!q_ready) wait_and_load_q();
  // ---- asynchronous staging of batch x+1: every thread stages its entries
  // tid + k*kThreads in three steps interleaved with its warp's batch-x tiles —
  // A list values and weights (4-byte cp.async) + masks, B page-table entries
  // (cp.async into spg), C row offsets (+ thread 0: the tile table) and an
  // arrive on the buffer's mbarrier; a warp waits on it only when its ring
  // reaches batch x+1, so no warp stops for the staging round trips.
  const int32_t* es = p.entry_slot
      ? p.entry_slot + ((static_cast<int64_t>(p.layer) * p.batch + b) * p.kv_heads + g) * p.hot_cap
      : nullptr;
  const int64_t grp_row0 = (static_cast<int64_t>(b) * p.kv_heads + g) * p.hot_cap;   // f4
  const int32_t* btg = p.block_table + static_cast<int64_t>(b) * p.max_blocks;
  const bool gs = p.group_sel != 0;
  const uint32_t allc = (1u << G) - 1u;
  int sstep = 3;   // steps of the staged batch this thread has done (3: all)
  auto stage_step = [&](int y) {
    const int eb = e_lo + y * kBatch, E = min(kBatch, e_hi - eb);
    uint32_t* yoff = BOFF(y);
    uint32_t* ymk = BMK(y);
    float* yw = BW(y);
    if (sstep == 0 && L.nrows == 1) {
      // one SLM row (group-coherent maps): its list bases once per batch
      const uint32_t yoff32 = smem_u32(yoff), yw32 = smem_u32(yw), spg32 = smem_u32(spg);
      const int64_t rb0 = static_cast<int64_t>(L.rj[0]) * p.batch + b;
      const int32_t* cb = p.crit_idx + rb0 * p.max_crit;
      const int32_t* mb = p.marg_idx + rb0 * p.max_marg;
      const float* wb = p.marg_w + rb0 * p.max_marg;
      const int K0 = L.rK[0];
      const uint32_t hm = L.rhm[0];
      for (int k = 0; k < kBatch / kThreads; ++k) {
        const int i = tid + k * kThreads;
        if (i >= E) break;
        const int xv = eb + i;
        if (es) cp_async4(spg32 + 4u * i, es + xv);
        if (xv < L.Rc) {
          yoff[i] = static_cast<uint32_t>(L.n - L.Rc + xv);
          ymk[i] = allc;
          yw[i] = 0.f;
          continue;
        }
        const int xr = xv - L.Rc;
        if (xr < K0) {
          cp_async4(yoff32 + 4u * i, cb + xr);
          ymk[i] = hm;
          yw[i] = 0.f;
        } else {
          cp_async4(yoff32 + 4u * i, mb + (xr - K0));
          ymk[i] = hm << 8;
          if (!gs) cp_async4(yw32 + 4u * i, wb + (xr - K0));
          else yw[i] = 0.f;
        }
      }
    } else if (sstep == 0) {
      for (int k = 0; k < kBatch / kThreads; ++k) {
        const int i = tid + k * kThreads;
        if (i >= E) break;
        const int xv = eb + i;
        if (es) cp_async4(smem_u32(spg + i), es + xv);
        if (xv < L.Rc) {
          yoff[i] = static_cast<uint32_t>(L.n - L.Rc + xv);
          ymk[i] = allc;
          yw[i] = 0.f;
          continue;
        }
        int xr = xv - L.Rc, kk = 0;
        while (kk < L.nrows - 1 && xr >= L.rK[kk] + L.rM[kk]) {
          xr -= L.rK[kk] + L.rM[kk];
          ++kk;
        }
        const int64_t rbk = static_cast<int64_t>(L.rj[kk]) * p.batch + b;
        if (xr < L.rK[kk]) {
          cp_async4(smem_u32(yoff + i), p.crit_idx + rbk * p.max_crit + xr);
          ymk[i] = L.rhm[kk];
          yw[i] = 0.f;
        } else {
          const int m = xr - L.rK[kk];
          cp_async4(smem_u32(yoff + i), p.marg_idx + rbk * p.max_marg + m);
          ymk[i] = L.rhm[kk] << 8;
          if (!gs) cp_async4(smem_u32(yw + i), p.marg_w + rbk * p.max_marg + m);
          else yw[i] = 0.f;
        }
      }
    } else if (sstep == 1) {
      const uint32_t spg32 = smem_u32(spg);
      if (!es)
        for (int k = 0; k < kBatch / kThreads; ++k) {
          const int i = tid + k * kThreads;
          if (i >= E) break;
          cp_async4(spg32 + 4u * i, btg + (static_cast<int>(yoff[i]) >> p.ps_shift));
        }
    } else if (sstep == 2) {
      for (int k = 0; k < kBatch / kThreads; ++k) {
        const int i = tid + k * kThreads;
        if (i >= E) break;
        const int pos = static_cast<int>(yoff[i]);
        yoff[i] = es ? static_cast<uint32_t>((grp_row0 + spg[i]) * D)
                     : static_cast<uint32_t>(((static_cast<int64_t>(spg[i]) * p.kv_heads + g) * p.page_size +
                                              (pos & (p.page_size - 1))) * D);
        // the weight arrived by this thread's cp.async, which the wait made
        // visible to this thread only: an ordinary store publishes it with the
        // arrive below (the other warps read it after their wait)
        const float wv = yw[i];
        asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(smem_u32(yw + i)), "f"(wv) : "memory");
      }
      if (tid == 0) build_tile_table(L, eb, E, gs, BTT(y));
      mbar_arrive(&bar_staged[y & 1]);
    }
    ++sstep;
  };
  for (int x = 0; x < nbatch; ++x) {
    const bool more = x + 1 < nbatch;
    sstep = more ? 0 : 3;
    if (more && (!kAsync || p.sync_stage == 1)) {
      // diagnostics: the whole staging of batch x+1 now, CTA-synchronously
#ifdef SKV_TRACE
      const long long t_st = gtimer();
#endif
      const int eb1 = e_lo + (x + 1) * kBatch, E1 = min(kBatch, e_hi - eb1);
      stage_entries<D>(p, L, b, g, eb1, E1, BOFF(x + 1), BMK(x + 1), BW(x + 1));
      if (tid == 0) build_tile_table(L, eb1, E1, gs, BTT(x + 1));
      mbar_arrive(&bar_staged[(x + 1) & 1]);
      sstep = 3;
#ifdef SKV_TRACE
      skv_stage_ns += gtimer() - t_st;
#endif
    }
    const int nmy = nmy_of(x);
    int nmy_next = -1;   // known once batch x+1 is staged
    auto wait_next = [&]() {   // batch x+1's entries and tile table are in place
      if (nmy_next >= 0) return;
      while (sstep < 3) {   // this thread's remaining steps first (drains its copies;
        cp_async_commit();  // wait_group covers committed groups only)
        cp_async_wait<0>();
        stage_step(x + 1);
      }
      mbar_wait(&bar_staged[(x + 1) & 1], static_cast<uint32_t>((x >> 1) & 1));
      nmy_next = nmy_of(x + 1);
    };
    const uint32_t* cmk = BMK(x);
    const float* cw = BW(x);
    if (kAsync && more && p.sync_stage == 2) {
      // diagnostics: this thread's three steps now (full waits), barrier hand-off kept
      while (sstep < 3) {
        cp_async_commit();
        cp_async_wait<0>();
        stage_step(x + 1);
      }
    }
    for (int i = 0; i < nmy; ++i) {
      if (kAsync && more && i == 0 && sstep == 0) stage_step(x + 1);   // A: joins this iteration's commit group
      // ring slot of the tile NSTAGE-1 ahead: this batch's, else the next batch's
      const int ti = i + NSTAGE - 1;
      if (ti < nmy) {
        issue(x, ti, tbase + ti);
      } else if (more) {
        wait_next();
        issue(ti - nmy < nmy_next ? x + 1 : -1, ti - nmy, tbase + ti);
      } else {
        issue(-1, 0, tbase + ti);
      }
      if (kAsync && more && sstep < 3 && (i == 1 || i == 3)) {
        // B at iteration 1, C at 3: the previous step's group (one iteration
        // older than the ring needs) is waited for here
        cp_async_wait<NSTAGE - 2>();
        stage_step(x + 1);
      }
      cp_async_wait<NSTAGE - 1>();
      __syncwarp();
      if (i == 0) { SKV_T(3); }
      const uint8_t* st = wst + ((tbase + i) % NSTAGE) * SB;
      const uint8_t* kb = st;
      const uint8_t* vb = st + KV_BYTES;
      // (shared-window addresses for ldmatrix: one conversion per tile)
      const uint32_t kb32 = wst_u32 + static_cast<uint32_t>(((tbase + i) % NSTAGE) * SB);
      const uint32_t vb32 = kb32 + KV_BYTES;
      const uint32_t td = BTT(x)[1 + warp + i * kWarps];
      const int e0 = static_cast<int>(td & 0xffffu), cnt = static_cast<int>((td >> 16) & 0xffu);
      if (td >> 25) {
        // ---- f2 marginal tile, 16 rows: O_m^T += V^T · A'^T with per-head
        // weights a'_{f(h)} staged in the K half ([16][8], head slot gq)
        const float* wst8 = reinterpret_cast<const float*>(st);
        float wm[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int tok = (u >> 1) * 8 + 2 * tq + (u & 1);
          wm[u] = tok < cnt ? wst8[tok * 8 + gq] : 0.f;
        }
        uint32_t bh0_, bl0_, bh1_, bl1_;
        split_bf16x2(wm[0], wm[1], bh0_, bl0_);
        split_bf16x2(wm[2], wm[3], bh1_, bl1_);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int r = ((mi >> 1) << 3) + (lane & 7);
          const int ch = 2 * mt + (mi & 1);
          uint32_t a0, a1, a2, a3;
          ldsm_x4_t(vb32 + r * ROWB + ((ch ^ (r & 7)) << 4), a0, a1, a2, a3);
          mma_bf16(om[mt], a0, a1, a2, a3, bh0_, bh1_);
          mma_bf16(om[mt], a0, a1, a2, a3, bl0_, bl1_);
        }
        __syncwarp();
        continue;
      }
      if (td >> 24) {
        // ---- V-only tile (marginal entries), 32 rows: O_m^T += V^T · a'^T.
        // B operand: a' of head gq at tokens 2tq, 2tq+1 (+8), hi + lo bf16.
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float wm[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int tok = half * 16 + (u >> 1) * 8 + 2 * tq + (u & 1);
            const uint32_t mk = tok < cnt ? cmk[e0 + tok] : 0u;
            wm[u] = ((mk >> (8 + gq)) & 1u) ? cw[e0 + tok] : 0.f;
          }
          uint32_t bh0_, bl0_, bh1_, bl1_;
          split_bf16x2(wm[0], wm[1], bh0_, bl0_);
          split_bf16x2(wm[2], wm[3], bh1_, bl1_);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int r = half * 16 + ((mi >> 1) << 3) + (lane & 7);
            const int ch = 2 * mt + (mi & 1);
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(smem_u32(st + r * ROWB + ((ch ^ (r & 7)) << 4)), a0, a1, a2, a3);
            mma_bf16(om[mt], a0, a1, a2, a3, bh0_, bh1_);
            mma_bf16(om[mt], a0, a1, a2, a3, bl0_, bl1_);
          }
        }
        __syncwarp();
        continue;
      }
      // S^T = K · Q^T : rows = 16 tokens, columns = 8 heads (one n8 tile);
      // lane holds tokens gq, gq+8 x heads 2tq, 2tq+1.  Four accumulation chains.
      float sc[4][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f},
                        {0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int r = ((mi & 1) << 3) + (lane & 7);
        const int ch = 2 * kk + (mi >> 1);
        uint32_t a0, a1, a2, a3;
        ldsm_x4(kb32 + r * ROWB + ((ch ^ (r & 7)) << 4), a0, a1, a2, a3);
        mma_bf16(sc[kk & 3], a0, a1, a2, a3, qa[kk][0], qa[kk][1]);
      }
      float s4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) s4[u] = (sc[0][u] + sc[1][u]) + (sc[2][u] + sc[3][u]);
      const uint32_t mkA = gq < cnt ? cmk[e0 + gq] : 0u;
      const uint32_t mkB = gq + 8 < cnt ? cmk[e0 + gq + 8] : 0u;
      const float sv0 = ((mkA >> h0) & 1u) ? s4[0] * p.scale_log2 : -INFINITY;   // tok gq,   head h0
      const float sv1 = ((mkA >> h1) & 1u) ? s4[1] * p.scale_log2 : -INFINITY;   // tok gq,   head h1
      const float sv2 = ((mkB >> h0) & 1u) ? s4[2] * p.scale_log2 : -INFINITY;   // tok gq+8, head h0
      const float sv3 = ((mkB >> h1) & 1u) ? s4[3] * p.scale_log2 : -INFINITY;   // tok gq+8, head h1
      float x0 = fmaxf(sv0, sv2), x1 = fmaxf(sv1, sv3);
      // lazy online softmax: the base of a head is raised (with the O rescale)
      // only when a score exceeds it by more than kRescaleSlack; one vote in
      // the common case, the cross-lane max only when some lane needs it
      if (__any_sync(0xffffffffu, x0 > m0 + kRescaleSlack || x1 > m1 + kRescaleSlack)) {
#pragma unroll
        for (int sh = 4; sh < 32; sh <<= 1) {
          x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, sh));
          x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, sh));
        }
        if (x0 > m0 + kRescaleSlack) {
          const float al = exp2f(m0 - x0);   // 0 when m0 = -inf
          l0 *= al;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            oc[mt][0] *= al;
            oc[mt][2] *= al;
          }
          m0 = x0;
        }
        if (x1 > m1 + kRescaleSlack) {
          const float al = exp2f(m1 - x1);
          l1 *= al;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            oc[mt][1] *= al;
            oc[mt][3] *= al;
          }
          m1 = x1;
        }
      }
      const float mu0 = m0 == -INFINITY ? 0.f : m0, mu1 = m1 == -INFINITY ? 0.f : m1;
      const float p0 = exp2f(sv0 - mu0), p1 = exp2f(sv1 - mu1);
      const float p2 = exp2f(sv2 - mu0), p3 = exp2f(sv3 - mu1);
      l0 += p0 + p2;
      l1 += p1 + p3;
      // P^T fragments (tokens x heads, hi + lo) -> B operand (tokens 2tq.., head gq)
      uint32_t h01, l01, h23, l23;
      split_bf16x2(p0, p1, h01, l01);
      split_bf16x2(p2, p3, h23, l23);
      const uint32_t bh0_ = movmatrix_t(h01), bh1_ = movmatrix_t(h23);
      const uint32_t bl0_ = movmatrix_t(l01), bl1_ = movmatrix_t(l23);
      // O_c^T += V^T · P^T
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int r = ((mi >> 1) << 3) + (lane & 7);
        const int ch = 2 * mt + (mi & 1);
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vb32 + r * ROWB + ((ch ^ (r & 7)) << 4), a0, a1, a2, a3);
        mma_bf16(oc[mt], a0, a1, a2, a3, bh0_, bh1_);
        mma_bf16(oc[mt], a0, a1, a2, a3, bl0_, bl1_);
      }
      __syncwarp();
    }
    if (more) wait_next();   // (a warp with few tiles in batch x)
    tbase += nmy;
    __syncthreads();   // batch x's buffer is free for batch x+2
  }
  cp_async_wait<0>();
  __syncthreads();   // the stages are free for the merge
  if (!q_ready) wait_and_load_q();   // empty share: still order the output writes
#pragma unroll
  for (int sh = 4; sh < 32; sh <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, sh);
    l1 += __shfl_xor_sync(0xffffffffu, l1, sh);
  }
  SKV_T(4);
#ifdef SKV_TRACE
  {
    int smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    SKV_TS(10, e_hi - e_lo);
    SKV_TS(11, smid);
    SKV_TS(12, skv_stage_ns);
    SKV_TS(13, nbatch);
  }
#endif

  // ---- merge warps (fixed order)
  float* wm_s = reinterpret_cast<float*>(stages);              // [kWarps][8]
  float* wl_s = wm_s + kWarps * 8;                              // [kWarps][8]
  float* wo_s = wl_s + kWarps * 8;                              // [kWarps][16][D + 4]: O_c rows h, O_m rows 8+h
  constexpr int RSW = D + 4;   // padded row stride of the per-warp partials (banks)
  if (gq == 0) {
    wm_s[warp * 8 + h0] = m0;
    wm_s[warp * 8 + h1] = m1;
    wl_s[warp * 8 + h0] = l0;
    wl_s[warp * 8 + h1] = l1;
  }
  if (NC == 1) {
    // One CTA per group: every warp folds its softmax normalisation into its
    // own partial first — c_w = O_c,w · 2^(m_w - M) / L + O_m,w with the
    // group-wide M and L from the (m, l) of all warps — so only [8][D] floats
    // per warp go through shared memory and the final merge is a plain sum.
    __syncthreads();
    SKV_T(8);
    // (h0, h1 = h0 + 1) are adjacent: one 8-byte load per warp for each of m, l
    float2 wm[kWarps], wl[kWarps];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      wm[w] = *reinterpret_cast<const float2*>(wm_s + w * 8 + h0);
      wl[w] = *reinterpret_cast<const float2*>(wl_s + w * 8 + h0);
    }
    float M0 = -INFINITY, M1 = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      M0 = fmaxf(M0, wm[w].x);
      M1 = fmaxf(M1, wm[w].y);
    }
    const float M0u = M0 == -INFINITY ? 0.f : M0, M1u = M1 == -INFINITY ? 0.f : M1;
    float L0 = 0.f, L1 = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      L0 += wl[w].x * exp2f(wm[w].x - M0u);
      L1 += wl[w].y * exp2f(wm[w].y - M1u);
    }
    const float f0 = L0 > 0.f ? exp2f(m0 - M0u) / L0 : 0.f;
    const float f1 = L1 > 0.f ? exp2f(m1 - M1u) / L1 : 0.f;
    // rows padded to D + 4 floats: the 4 head rows a warp's lanes write (tq)
    // fall in different banks
    constexpr int RS = D + 4;
    float* myc = wo_s + warp * 8 * RS;                          // [kWarps][8][D + 4]
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int d0 = 16 * mt + gq;
      myc[h0 * RS + d0] = oc[mt][0] * f0 + om[mt][0];
      myc[h1 * RS + d0] = oc[mt][1] * f1 + om[mt][1];
      myc[h0 * RS + d0 + 8] = oc[mt][2] * f0 + om[mt][2];
      myc[h1 * RS + d0 + 8] = oc[mt][3] * f1 + om[mt][3];
    }
    __syncthreads();
    const int64_t bo = static_cast<int64_t>(b) * p.heads + g * G;
    for (int it = tid; it < G * (D / 4); it += kThreads) {
      const int h = it / (D / 4), c4 = (it % (D / 4)) * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const float4 a = *reinterpret_cast<const float4*>(wo_s + (w * 8 + h) * RS + c4);
        acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
      }
      *reinterpret_cast<float4*>(p.out + (bo + h) * D + c4) = acc;
    }
    SKV_T(5);
    return;
  }
  {
    float* myo = wo_s + warp * 16 * RSW;                       // rows padded (bank-conflict free)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int d0 = 16 * mt + gq;
      myo[h0 * RSW + d0] = oc[mt][0];
      myo[h1 * RSW + d0] = oc[mt][1];
      myo[h0 * RSW + d0 + 8] = oc[mt][2];
      myo[h1 * RSW + d0 + 8] = oc[mt][3];
      myo[(8 + h0) * RSW + d0] = om[mt][0];
      myo[(8 + h1) * RSW + d0] = om[mt][1];
      myo[(8 + h0) * RSW + d0 + 8] = om[mt][2];
      myo[(8 + h1) * RSW + d0 + 8] = om[mt][3];
    }
  }
  __syncthreads();
  const int64_t bh0 = static_cast<int64_t>(b) * p.heads + g * G;
  // this CTA's merged state: [M 8][L 8][O_c 8 x D][O_m 8 x D] (read by rank 0 over DSMEM)
  float* cst = reinterpret_cast<float*>(stages + (kWarps * 16 * RSW + 2 * kWarps * 8) * 4);
  for (int it = tid; it < G * (D / 4); it += kThreads) {
    const int h = it / (D / 4), c4 = (it % (D / 4)) * 4;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, wm_s[w * 8 + h]);
    const float Mu = M == -INFINITY ? 0.f : M;
    float L = 0.f;
    float4 oc = make_float4(0.f, 0.f, 0.f, 0.f), om = oc;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float f = exp2f(wm_s[w * 8 + h] - Mu);
      L += wl_s[w * 8 + h] * f;
      const float4 a = *reinterpret_cast<const float4*>(wo_s + (w * 16 + h) * RSW + c4);
      const float4 m = *reinterpret_cast<const float4*>(wo_s + (w * 16 + h + 8) * RSW + c4);
      oc.x += a.x * f; oc.y += a.y * f; oc.z += a.z * f; oc.w += a.w * f;
      om.x += m.x; om.y += m.y; om.z += m.z; om.w += m.w;
    }
    if (NC == 1) {
      const float li = L > 0.f ? 1.f / L : 0.f;
      *reinterpret_cast<float4*>(p.out + (bh0 + h) * D + c4) =
          make_float4(oc.x * li + om.x, oc.y * li + om.y, oc.z * li + om.z, oc.w * li + om.w);
    } else {
      if (c4 == 0) {
        cst[h] = M;
        cst[8 + h] = L;
      }
      *reinterpret_cast<float4*>(cst + 16 + h * D + c4) = oc;
      *reinterpret_cast<float4*>(cst + 16 + 8 * D + h * D + c4) = om;
    }
  }
  SKV_T(5);
  if (NC == 1) return;

  if (p.global_merge) {
    // ---- K4 without a cluster: every rank stores its state, the last rank of
    // the group to arrive merges all of them in rank order (deterministic)
    __syncthreads();   // the state was written by all threads
    const int64_t grp = static_cast<int64_t>(b) * p.kv_heads + g;
    float* part = p.partials + (grp * NC + c) * kAttendPartFloats;
    constexpr int kPart4 = (16 + 16 * D) / 4;
    for (int i = tid; i < kPart4; i += kThreads)
      reinterpret_cast<float4*>(part)[i] = reinterpret_cast<const float4*>(cst)[i];
    __threadfence();
    __syncthreads();
    __shared__ int s_last;
    if (tid == 0) s_last = atomicAdd(p.tickets + grp, 1) == nmerge - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* gp = p.partials + grp * NC * kAttendPartFloats;
    // every rank's (m, l) at once, then per head the rank weights 2^(m_q - M)
    // and L in rank order; the O rows with 8 ranks' loads in flight per thread
    __shared__ float s_m[32][8], s_l[32][8], s_L[8];
    if (tid < nmerge * 8) {
      const int q = tid >> 3, h = tid & 7;
      s_m[q][h] = __ldcg(gp + q * kAttendPartFloats + h);
      s_l[q][h] = __ldcg(gp + q * kAttendPartFloats + 8 + h);
    }
    __syncthreads();
    if (tid < G) {
      float M = -INFINITY;
      for (int q = 0; q < nmerge; ++q) M = fmaxf(M, s_m[q][tid]);
      const float Mu = M == -INFINITY ? 0.f : M;
      float L = 0.f;
      for (int q = 0; q < nmerge; ++q) {
        const float f = exp2f(s_m[q][tid] - Mu);
        L += s_l[q][tid] * f;
        s_m[q][tid] = f;   // (now the rank's weight)
      }
      s_L[tid] = L;
    }
    __syncthreads();
    for (int it = tid; it < G * (D / 4); it += kThreads) {
      const int h = it / (D / 4), c4 = (it % (D / 4)) * 4;
      float4 oc = make_float4(0.f, 0.f, 0.f, 0.f), om = oc;
#pragma unroll 8
      for (int q = 0; q < nmerge; ++q) {
        const float* pq = gp + q * kAttendPartFloats;
        const float f = s_m[q][h];
        const float4 a = __ldcg(reinterpret_cast<const float4*>(pq + 16 + h * D + c4));
        const float4 m = __ldcg(reinterpret_cast<const float4*>(pq + 16 + 8 * D + h * D + c4));
        oc.x += a.x * f; oc.y += a.y * f; oc.z += a.z * f; oc.w += a.w * f;
        om.x += m.x; om.y += m.y; om.z += m.z; om.w += m.w;
      }
      const float L = s_L[h];
      const float li = L > 0.f ? 1.f / L : 0.f;
      *reinterpret_cast<float4*>(p.out + (bh0 + h) * D + c4) =
          make_float4(oc.x * li + om.x, oc.y * li + om.y, oc.z * li + om.z, oc.w * li + om.w);
    }
    if (tid == 0) p.tickets[grp] = 0;   // ready for the next launch
    return;
  }

  // ---- fused K4: the group's CTAs form one thread-block cluster; the ranks
  // merge every rank's state in rank order through distributed shared memory.
  cluster_sync();
  {
    // every rank merges its share of the (head, 4-column) items in rank order
    const uint32_t base = smem_u32(cst);
    for (int it = c * kThreads + tid; it < G * (D / 4); it += NC * kThreads) {
      const int h = it / (D / 4), c4 = (it % (D / 4)) * 4;
      float M = -INFINITY;
      for (int q = 0; q < NC; ++q) M = fmaxf(M, ld_dsmem_f32(base + h * 4, q));
      const float Mu = M == -INFINITY ? 0.f : M;
      float L = 0.f;
      float4 oc = make_float4(0.f, 0.f, 0.f, 0.f), om = oc;
      for (int q = 0; q < NC; ++q) {
        const float f = exp2f(ld_dsmem_f32(base + h * 4, q) - Mu);
        L += ld_dsmem_f32(base + (8 + h) * 4, q) * f;
        const float4 a = ld_dsmem_f32x4(base + (16 + h * D + c4) * 4, q);
        const float4 m = ld_dsmem_f32x4(base + (16 + 8 * D + h * D + c4) * 4, q);
        oc.x += a.x * f; oc.y += a.y * f; oc.z += a.z * f; oc.w += a.w * f;
        om.x += m.x; om.y += m.y; om.z += m.z; om.w += m.w;
      }
      const float li = L > 0.f ? 1.f / L : 0.f;
      *reinterpret_cast<float4*>(p.out + (bh0 + h) * D + c4) =
          make_float4(oc.x * li + om.x, oc.y * li + om.y, oc.z * li + om.z, oc.w * li + om.w);
    }
  }
  cluster_sync();   // keep every rank's shared memory alive until all reads are done
  SKV_T(6);
}

template <int D, bool kAsync, bool kFlat>
__global__ void __launch_bounds__(kThreads, 8 / kWarps) attend_kernel(const AttendParams p) {
  if constexpr (!kFlat) {
    attend_share<D, kAsync, false>(p, blockIdx.x, blockIdx.y, blockIdx.z, p.max_chunks, p.max_chunks);
    return;
  }
  // per-group ranks: grid (NC, H_kv, B), one share each.  Stream-K: grid (S),
  // CTA s runs the shares of the (at most two when S > #groups) groups its
  // interval meets, in group order (share_begin).
  const int64_t S = p.flat_shares, Gt = static_cast<int64_t>(p.batch) * p.kv_heads;
  const int s = blockIdx.x;
  const int grp_lo = S ? static_cast<int>(s * Gt / S) : 0;
  const int grp_hi = S ? static_cast<int>(((s + 1) * Gt - 1) / S) : 0;
  for (int grp = grp_lo; grp <= grp_hi; ++grp) {
    int c = blockIdx.x, g = blockIdx.y, b = blockIdx.z, nmerge = p.max_chunks;
    if (S) {
      const int64_t s_first = grp * S / Gt, s_last = ((grp + 1) * S + Gt - 1) / Gt - 1;
      c = static_cast<int>(s - s_first);
      nmerge = static_cast<int>(s_last - s_first + 1);
      g = grp % p.kv_heads;
      b = grp / p.kv_heads;
    }
    if (grp > grp_lo) {   // the previous share's copies, barriers and shared memory are done
      cp_async_wait<0>();
      __syncthreads();
    }
    attend_share<D, kAsync, kFlat>(p, c, g, b, p.max_chunks, nmerge);
  }
}

// ---------------------------------------------------------------------------
// Variant f4: host-tiered KV.  The full paged pool lives in
// host memory; each (layer, sequence, kv-group) keeps the rows its current
// list needs in an HBM hot pool of `cap` slots.  Per step and layer, one CTA
// per group: (1) decode the list's positions (the attend kernel's own layout)
// and mark them, with "needs K" for critical / recent entries; (2) free the
// slots of positions no longer needed; (3) give every newly needed position a
// free slot; (4) fetch from host memory (zero-copy over the host link) only
// what is missing — V for every new position, K only where a critical /
// recent entry needs it; (5) write each entry's slot for the attend kernel.
// Rows resident at the previous step are not moved (migrate the
// change, in parallel with the forward).
constexpr int kTierThreads = 256;
template <int D>
__global__ void __launch_bounds__(kTierThreads) tier_update_kernel(const TierParams t) {
  const AttendParams& p = t.a;
  __shared__ __align__(16) GroupLayout L;
  __shared__ int s_nfree, s_nmiss;
  // per-position bitmaps (3 x ceil(max_seq_len / 32) words: 48 KB at 128K tokens)
  extern __shared__ uint32_t bitmaps[];
  const int nw = (t.max_seq_len + 31) / 32;
  uint32_t* need_v = bitmaps;
  uint32_t* need_k = bitmaps + nw;
  uint32_t* claimed = bitmaps + 2 * nw;
  const int g = blockIdx.x, b = blockIdx.y, layer = t.layer_begin + blockIdx.z, tid = threadIdx.x;
  build_layout(p, layer, b, g, L);
  const int n = L.n, T = L.T;
  const int64_t grp = (static_cast<int64_t>(layer) * p.batch + b) * p.kv_heads + g;
  if (T > t.cap) {   // the list does not fit the group's slots: reported, nothing changed
    if (tid == 0) {
      atomicAdd(t.counters + 1, 1ull);
      t.njob[grp] = 0;
    }
    return;
  }
  // per-entry scratch in global memory (L2): [cap] entry positions | [cap]
  // free slots | [cap] missing positions
  int* s_pos = t.scratch + grp * 3 * t.cap;
  int* s_free = s_pos + t.cap;
  int* s_miss = s_pos + 2 * t.cap;
  int32_t* sop = t.slot_of_pos + grp * t.max_seq_len;
  int32_t* pos_of = t.pos_of_slot + grp * t.cap;
  uint8_t* flags = t.slot_flags + grp * t.cap;
  int32_t* es = t.entry_slot + grp * t.cap;
  for (int i = tid; i < (n + 31) / 32; i += kTierThreads) need_v[i] = need_k[i] = claimed[i] = 0u;
  if (tid == 0) s_nfree = s_nmiss = 0;
  __syncthreads();
  // (1) the list's positions (decoded once) and their needs: K+V for recent /
  // critical entries, V for marginal ones.  s_pos keeps (position | K needed
  // << 31) of the last refresh: an identical list leaves nothing to do (the
  // steady state), which one comparison per entry detects.
  int changed = T != t.prev_T[grp];
  for (int x = tid; x < T; x += kTierThreads) {
    const ListEntry le = list_entry(p, L, b, x, 0xffu);
    const int pos = le.pos;
    const bool k = (le.mask & 0xffu) != 0u;   // critical / recent: K needed
    const int code = pos | (k ? static_cast<int>(0x80000000u) : 0);
    changed |= s_pos[x] != code;
    s_pos[x] = code;
    atomicOr(&need_v[pos >> 5], 1u << (pos & 31));
    if (k) atomicOr(&need_k[pos >> 5], 1u << (pos & 31));
  }
  if (!__syncthreads_or(changed)) {
    if (tid == 0) t.njob[grp] = 0;
    return;
  }
  // (2) free the slots of positions no longer needed; collect free slots
  for (int sl = tid; sl < t.cap; sl += kTierThreads) {
    int pos = pos_of[sl];
    if (pos >= 0 && !((need_v[pos >> 5] >> (pos & 31)) & 1u)) {
      pos_of[sl] = -1;
      flags[sl] = 0;
      sop[pos] = -1;
      pos = -1;
    }
    if (pos < 0) s_free[atomicAdd(&s_nfree, 1)] = sl;
  }
  __syncthreads();
  // (3) newly needed positions (each once), then their slots
  for (int x = tid; x < T; x += kTierThreads) {
    const int pos = s_pos[x] & 0x7fffffff;
    if (sop[pos] < 0 && !((atomicOr(&claimed[pos >> 5], 1u << (pos & 31)) >> (pos & 31)) & 1u))
      s_miss[atomicAdd(&s_nmiss, 1)] = pos;
  }
  __syncthreads();
  const int nmiss = s_nmiss, nfree = s_nfree;
  if (tid == 0) {
    if (nmiss > nfree) atomicAdd(t.counters + 1, 1ull);
    t.prev_T[grp] = nmiss > nfree ? -1 : T;   // (an overflow: refresh in full next time)
  }
  for (int i = tid; i < min(nmiss, nfree); i += kTierThreads) {
    const int pos = s_miss[i], sl = s_free[i];
    pos_of[sl] = pos;
    flags[sl] = 0;
    sop[pos] = sl;
  }
  __syncthreads();
  // (4) entries' slots, residency flags, and one fetch job per position that
  // misses V (new) or K (needed by a critical / recent entry); each position is
  // handled by its first entry (claimed bits are reused)
  for (int i = tid; i < (n + 31) / 32; i += kTierThreads) claimed[i] = 0u;
  if (tid == 0) s_nmiss = 0;
  __syncthreads();
  int* s_job = s_free;   // slot | getv << 30 | getk << 31
  int* s_jpos = s_miss;  // its position
  for (int x = tid; x < T; x += kTierThreads) {
    const int pos = s_pos[x] & 0x7fffffff;
    const int sl = sop[pos];
    es[x] = sl < 0 ? 0 : sl;
    if (sl < 0) continue;
    if ((atomicOr(&claimed[pos >> 5], 1u << (pos & 31)) >> (pos & 31)) & 1u) continue;
    const uint8_t f = flags[sl];
    const bool nk = (need_k[pos >> 5] >> (pos & 31)) & 1u;
    const bool getv = !(f & 1u), getk = nk && !(f & 2u);
    flags[sl] = static_cast<uint8_t>(f | 1u | (nk ? 2u : 0u));
    if (!getv && !getk) continue;
    const int j = atomicAdd(&s_nmiss, 1);
    s_job[j] = sl | (getv ? (1 << 30) : 0) | (getk ? (1u << 31) : 0);
    s_jpos[j] = pos;
  }
  __syncthreads();
  // (5) the copies: the next launch (tier_copy_kernel), whose threads keep
  // more host loads in flight than this kernel's register budget allows
  if (tid == 0) t.njob[grp] = s_nmiss;
}

// The host-link copies of tier_update's fetch jobs: 16-byte chunks,
// consecutive threads on consecutive chunks of a row (V then K: 2 x D*2
// contiguous bytes per job), kTierU chunk loads in flight per thread before
// their stores (zero-copy loads of pinned host memory over the link).
template <int D>
__global__ void __launch_bounds__(kTierThreads) tier_copy_kernel(const TierParams t) {
  const AttendParams& p = t.a;
  const int g = blockIdx.x, b = blockIdx.y, layer = t.layer_begin + blockIdx.z, tid = threadIdx.x;
  const int64_t grp = (static_cast<int64_t>(layer) * p.batch + b) * p.kv_heads + g;
  const int njob = t.njob[grp];
  if (njob == 0) return;
  const int* s_job = t.scratch + grp * 3 * t.cap + t.cap;        // slot | getv << 30 | getk << 31
  const int* s_jpos = t.scratch + grp * 3 * t.cap + 2 * t.cap;   // its position
  // host layer slot: layer mod the host pool's layers (a caller may rotate a subset)
  const int64_t hl = layer % t.host_layers;
  const uint16_t* host_k = t.host_k + hl * t.host_layer_stride;
  const uint16_t* host_v = t.host_v + hl * t.host_layer_stride;
  const int64_t hot0 = (static_cast<int64_t>(layer) * p.batch + b) * p.kv_heads + g;
  uint16_t* hot_k = t.hot_k + hot0 * t.cap * D;
  uint16_t* hot_v = t.hot_v + hot0 * t.cap * D;
  const int32_t* bt = p.block_table + static_cast<int64_t>(b) * p.max_blocks;
  constexpr int CH = D / 8;
#ifndef SKV_TIER_U
#define SKV_TIER_U 16
#endif
  constexpr int kTierU = SKV_TIER_U;
  unsigned long long rows = 0;
  for (int it0 = tid; it0 < njob * 2 * CH; it0 += kTierU * kTierThreads) {
    uint4 v[kTierU];
    uint4* dst[kTierU];
#pragma unroll
    for (int u = 0; u < kTierU; ++u) {
      const int it = it0 + u * kTierThreads;
      dst[u] = nullptr;
      if (it >= njob * 2 * CH) continue;
      const int j = it / (2 * CH), which = (it / CH) & 1, c = it % CH;   // which: 0 V, 1 K
      const uint32_t job = static_cast<uint32_t>(s_job[j]);
      if (!((job >> (30 + which)) & 1u)) continue;
      const int pos = s_jpos[j], sl = static_cast<int>(job & 0x3fffffffu);
      const int64_t src = ((static_cast<int64_t>(__ldg(bt + (pos >> p.ps_shift))) * p.kv_heads + g) *
                               p.page_size + (pos & (p.page_size - 1))) * D;
      v[u] = reinterpret_cast<const uint4*>((which ? host_k : host_v) + src)[c];
      dst[u] = reinterpret_cast<uint4*>((which ? hot_k : hot_v) + static_cast<int64_t>(sl) * D) + c;
      if (c == 0) ++rows;
    }
#pragma unroll
    for (int u = 0; u < kTierU; ++u)
      if (dst[u]) *dst[u] = v[u];
  }
  if (rows) atomicAdd(t.counters, rows);
}

}  // namespace

#ifdef SKV_TRACE
extern "C" int skv_debug_set_trace(long long* buf) {
  return cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 1;
}
#endif

// Largest cluster the GPU co-schedules `want` of at once (one attend CTA per SM),
// from the occupancy calculator; clusters above 8 CTAs are non-portable.
static int32_t clusters_fit(int nc) {
  static int cache[17] = {0};
  if (cache[nc]) return cache[nc] > 0 ? cache[nc] : 0;
  auto kern = attend_kernel<128, true, false>;
  const size_t sm = smem_bytes<128>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  if (nc > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nc, 1, 1);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = nc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = nc <= 8 ? 148 / nc : 0;
  }
  cache[nc] = n > 0 ? n : -1;
  return n;
}

// CTAs per (sequence, kv-group) = cluster size: the largest NC <= 16 with
// NC * groups <= #SMs whose clusters the GPU co-schedules in a single wave
// (one 8-warp CTA per SM), so a layer fills the GPU without a second wave.
// (Config 2: 128 groups -> 1; config 4 at one GPU: 64 groups -> 2; at one
// sequence per GPU: 8 groups -> up to 16.)
static int32_t num_sms() {
  static const int32_t sms = [] {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;   // B200
    }
    return n;
  }();
  return sms;
}

// CTAs per (sequence, kv-group): NC = #SMs / #groups (capped at 32), so a
// layer fills the GPU in one wave of one 8-warp CTA per SM.  When the GPU
// co-schedules a cluster of NC CTAs for every group at once (occupancy
// calculator; non-portable above 8), the ranks merge in distributed shared
// memory; otherwise the CTAs are launched without a cluster and merge through
// a global workspace (attend_split_in_cluster false).
// (Config 2: 128 groups -> 1; config 4 at one GPU: 64 groups -> 2, cluster;
// at one sequence per GPU: 8 groups -> 18, global merge.)
// Stream-K: when the groups do not divide the SMs, #SMs CTAs take equal byte
// shares of all groups laid end to end, so no SM idles (config 4: 64 groups
// leave 20 of 148 SMs without a stream of their own; with more groups than
// SMs, the last wave's tail).  At most 32 shares per group.  On by default for long lists
// (max_seq_len >= 65536) over >= 32 groups, where it measured faster (config 4
// +2.1%, its B = 4 rank +3.6%); short lists lose the cross-layer overlap and
// pay a second prologue (config 2: -32%).  SMALLKV_ATTEND_FLAT=0 / 1 forces it.
int32_t attend_flat_shares(int32_t batch, int32_t kv_heads, int32_t max_seq_len) {
  static const int32_t mode = [] {
    const char* e = getenv("SMALLKV_ATTEND_FLAT");   // tuning knob: 0 / 1
    return e ? atoi(e) : -1;
  }();
  if (mode == 0) return 0;
  const int64_t groups = static_cast<int64_t>(batch) * kv_heads, S = num_sms();
  if (groups <= 0 || S % groups == 0) return 0;
  // more groups than SMs (config 5: 512 groups = 3.46 waves): forced only
  if (groups >= S && (mode != 1 || groups % S == 0)) return 0;
  if ((S + groups - 1) / groups + 1 > 32) return 0;
  if (mode < 0 && (max_seq_len < 65536 || groups < 32)) return 0;
  return static_cast<int32_t>(S);
}

int32_t attend_ctas_per_group(int32_t batch, int32_t kv_heads, int32_t max_seq_len) {
  if (const int32_t S = attend_flat_shares(batch, kv_heads, max_seq_len)) {
    const int32_t groups = batch * kv_heads;
    return (S + groups - 1) / groups + 1;   // record slots: shares per group at most
  }
  static const int32_t forced = [] {
    const char* e = getenv("SMALLKV_ATTEND_CTAS");   // tuning knob
    return e ? atoi(e) : 0;
  }();
  if (forced > 0) return forced > 32 ? 32 : forced;
  const int64_t groups = static_cast<int64_t>(batch) * kv_heads;
  const int64_t nc = groups > 0 ? num_sms() / groups : 1;
  return nc < 1 ? 1 : (nc > 32 ? 32 : static_cast<int32_t>(nc));
}

bool attend_split_in_cluster(int32_t batch, int32_t kv_heads, int32_t max_seq_len) {
  static const int32_t force_global = [] {
    const char* e = getenv("SMALLKV_ATTEND_GLOBAL_MERGE");   // tuning knob
    return e ? atoi(e) : 0;
  }();
  if (attend_flat_shares(batch, kv_heads, max_seq_len)) return false;
  const int32_t nc = attend_ctas_per_group(batch, kv_heads, max_seq_len);
  if (nc <= 1) return true;
  if (force_global || nc > 16) return false;
  const int64_t groups = static_cast<int64_t>(batch) * kv_heads;
  return static_cast<int64_t>(clusters_fit(nc)) >= groups;
}

template <int D, bool kAsync, bool kFlat>
static cudaError_t launch_dk(const AttendParams& p, cudaStream_t s) {
  const size_t sm = smem_bytes<D>();
  cudaError_t e = cudaFuncSetAttribute(attend_kernel<D, kAsync, kFlat>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm));
  if (e != cudaSuccess) return e;
  if (p.flat_shares && !p.global_merge) return cudaErrorInvalidValue;
  if (p.max_chunks > 8 && !p.global_merge) {
    e = cudaFuncSetAttribute(attend_kernel<D, kAsync, kFlat>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  e = cudaFuncSetAttribute(attend_kernel<D, kAsync, kFlat>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = p.flat_shares ? dim3(p.flat_shares) : dim3(p.max_chunks, p.kv_heads, p.batch);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = p.max_chunks;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.global_merge ? 1 : 2;   // the global merge needs no cluster
  return cudaLaunchKernelEx(&cfg, attend_kernel<D, kAsync, kFlat>, p);
}

template <int D, bool kAsync>
static cudaError_t launch_d(const AttendParams& p, cudaStream_t s) {
  return p.flat_shares ? launch_dk<D, kAsync, true>(p, s) : launch_dk<D, kAsync, false>(p, s);
}

int64_t plan_bytes(int32_t n_layers, int32_t batch, int32_t kv_heads, int32_t max_seq_len) {
  return static_cast<int64_t>(n_layers) * batch * kv_heads *
         plan_record_bytes(attend_ctas_per_group(batch, kv_heads, max_seq_len));
}

cudaError_t launch_plan(const AttendParams& p, int32_t n_layers, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  // a record split over many ranks (small batches) is staged by one CTA per
  // rank; one CTA per record otherwise
  cfg.gridDim = dim3(p.kv_heads, n_layers * p.batch, p.max_chunks > 2 ? p.max_chunks : 1);
  cfg.blockDim = dim3(kPlanThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = p.head_dim == 64 ? cudaLaunchKernelEx(&cfg, plan_kernel<64>, p)
                                   : cudaLaunchKernelEx(&cfg, plan_kernel<128>, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_tier_update(const TierParams& t, cudaStream_t s) {
  const size_t sm = static_cast<size_t>((t.max_seq_len + 31) / 32) * 3 * sizeof(uint32_t);
  dim3 grid(t.a.kv_heads, t.a.batch, t.layer_count);
  auto k = t.a.head_dim == 64 ? tier_update_kernel<64> : tier_update_kernel<128>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k<<<grid, kTierThreads, sm, s>>>(t);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  auto kc = t.a.head_dim == 64 ? tier_copy_kernel<64> : tier_copy_kernel<128>;
  kc<<<grid, kTierThreads, 0, s>>>(t);
  return cudaGetLastError();
}

cudaError_t launch_attend(const AttendParams& p, cudaStream_t s) {
  static const int forced = [] {
    const char* e = getenv("SMALLKV_ATTEND_ASYNC");   // tuning knob: 0 / 1
    return e ? atoi(e) : -1;
  }();
  const bool async = forced >= 0 ? forced != 0 : p.row_stride > kAsyncStageMinLen;
  cudaError_t e = p.head_dim == 64 ? (async ? launch_d<64, true>(p, s) : launch_d<64, false>(p, s))
                                   : (async ? launch_d<128, true>(p, s) : launch_d<128, false>(p, s));
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace skv
