// slm_score.cu — K1: the SLM's decode attention logits over its FULL cache.
//
// Alg. 1 l.7 "Forward process of M_s(x+t) to update A'_j", scored over
// the never-compressed SLM cache C^s_all.  For SLM layer j_l, kv-head
// g', sequence b this kernel streams K'[0, n) once and produces, for every
// q-head h of the group that the head map references (rows of image(f)),
//   s'_v = q'_h · K'[v] / sqrt(d_s)          (fp32 accumulate)
// The softmax statistics (m', lse') and the split are computed by K2 from these
// rows (select.cu).
//
// B200 design: one CTA = (token chunk, kv-head, layer*B+b); a producer warp
// streams 64-token K' tiles with 2-D TMA (cp.async.bulk.tensor, 128-byte
// swizzle) page by page through an mbarrier ring; 4 consumer warps each take 16
// tokens of a tile and contract them with the whole GQA query group on the
// tensor cores (mma.sync m16n8k16: heads = M (padded to 16), tokens = N,
// head_dim = K).  The path is HBM-bound (≈G_s flop/B); the tensor cores only
// keep the ALU off the critical path.
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace skv {

namespace {
constexpr int kTile = 64;       // tokens per pipeline stage
constexpr int kConsumers = 4;   // compute warps (16 tokens each)
constexpr int kThreads = (kConsumers + 1) * 32;

// 4 x 8 KB stages (d = 64): measured best of 2..8 — smaller CTAs, more of them per SM
template <int D>
constexpr int stages_for() { return 4; }

template <int D>
constexpr int smem_bytes() {
  return stages_for<D>() * kTile * D * 2 + 2 * stages_for<D>() * 8 + 1024;
}

template <int D>
__global__ void __launch_bounds__(kThreads)
slm_score_kernel(const __grid_constant__ CUtensorMap map, const SlmScoreParams p) {
  constexpr int NSTAGE = stages_for<D>();
  constexpr int HALVES = D / 64;                 // 128-byte column halves of a row
  constexpr int STAGE_BYTES = kTile * D * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
  uint64_t* empty = full + NSTAGE;

  const int kvh = blockIdx.y;
  const int layer = p.layer_begin + static_cast<int>(blockIdx.z) / p.batch;
  const int b = blockIdx.z % p.batch;
  // the select kernel of the previous layer chunk may run alongside (PDL)
  griddep_launch_dependents();
  // launched with programmatic dependent launch behind row_flags: the CTAs
  // become resident while it runs; nothing global is read before it completes
  griddep_wait();
  const int G = p.heads / p.kv_heads;
  const int n = p.seq_lens[b];
  const int t_begin = blockIdx.x * p.chunk_tokens;
  if (t_begin >= n) return;
  const int t_end = min(n, t_begin + p.chunk_tokens);
  const int ntiles = (t_end - t_begin + kTile - 1) / kTile;
  const int head0 = layer * p.heads + kvh * G;   // flat SLM head of the group's first q-head
  uint32_t need = 0;
  for (int h = 0; h < G; ++h) need |= (p.row_needed[head0 + h] ? 1u : 0u) << h;
  if (need == 0) return;                         // no LLM head maps into this group

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumers) {
    // ---------------- TMA producer: the warp stages the chunk's page-table
    // entries (one round), then one elected lane streams the tiles
    __shared__ int sbt[1024];
    const int first_blk = t_begin / p.page_size;
    const int nblk = (t_end - 1) / p.page_size - first_blk + 1;   // <= 1024 (chunk <= 1024 tokens)
    const int32_t* btb = p.block_table + static_cast<int64_t>(b) * p.max_blocks + first_blk;
    for (int i = lane; i < nblk; i += 32) sbt[i] = btb[i];
    __syncwarp();
    if (lane == 0) {
      prefetch_tmap(&map);
      const int boxes_per_tile = kTile / p.box_rows;
      for (int it = 0; it < ntiles; ++it) {
        const int s = it % NSTAGE;
        if (it >= NSTAGE) mbar_wait(&empty[s], ((it / NSTAGE) & 1) ^ 1);
        const int t0 = t_begin + it * kTile;
        int nbox = 0;
        for (int bx = 0; bx < boxes_per_tile; ++bx) nbox += (t0 + bx * p.box_rows < n) ? 1 : 0;
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nbox * HALVES * p.box_rows * 128));
        for (int bx = 0; bx < nbox; ++bx) {
          const int t = t0 + bx * p.box_rows;
          const int page = sbt[t / p.page_size - first_blk];
          const int64_t row64 =
              ((static_cast<int64_t>(layer) * p.num_pages + page) * p.kv_heads + kvh) * p.page_size +
              t % p.page_size;
          const int row = static_cast<int>(row64);
#pragma unroll
          for (int hf = 0; hf < HALVES; ++hf)
            tma_load_2d(smem_u32(smem + s * STAGE_BYTES + hf * kTile * 128 + bx * p.box_rows * 128),
                        &map, &full[s], hf * 64, row);
        }
      }
    }
    return;
  }

  // ---------------- consumers: S[16 heads x 16 tokens] per warp per tile
  const int gq = lane >> 2, tq = lane & 3;
  const uint16_t* qg = p.q + ((static_cast<int64_t>(layer) * p.batch + b) * p.heads + kvh * G) * D;
  uint32_t qa[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const int c = 16 * kk + 2 * tq;
    qa[kk][0] = gq < G ? *reinterpret_cast<const uint32_t*>(qg + gq * D + c) : 0u;
    qa[kk][1] = gq + 8 < G ? *reinterpret_cast<const uint32_t*>(qg + (gq + 8) * D + c) : 0u;
    qa[kk][2] = gq < G ? *reinterpret_cast<const uint32_t*>(qg + gq * D + c + 8) : 0u;
    qa[kk][3] = gq + 8 < G ? *reinterpret_cast<const uint32_t*>(qg + (gq + 8) * D + c + 8) : 0u;
  }
  const bool w_lo = gq < G && ((need >> gq) & 1u);
  const bool w_hi = gq + 8 < G && ((need >> (gq + 8)) & 1u);
  float* row_lo = w_lo ? p.logits + (static_cast<int64_t>(head0 + gq) * p.batch + b) * p.row_stride : nullptr;
  float* row_hi = w_hi ? p.logits + (static_cast<int64_t>(head0 + gq + 8) * p.batch + b) * p.row_stride : nullptr;
  const uint32_t swz = p.swz;
  const int mi = lane >> 3;
  const int r_ld = warp * 16 + ((mi >> 1) << 3) + (lane & 7);   // token row this lane addresses
  // per-row statistics of this chunk for K2 (rows gq and gq+8 of this lane):
  // (max, Σexp rel. max) over [0, n) and (min, max) over the ranked [0, N)
  const int N = n - min(max(p.n_recent[b], 0), n);
  float st_m[2] = {-FLT_MAX, -FLT_MAX}, st_s[2] = {0.f, 0.f};
  float st_lo[2] = {FLT_MAX, FLT_MAX}, st_hi[2] = {-FLT_MAX, -FLT_MAX};

  for (int it = 0; it < ntiles; ++it) {
    const int s = it % NSTAGE;
    mbar_wait(&full[s], (it / NSTAGE) & 1);
    const uint8_t* st = smem + s * STAGE_BYTES;
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int c = 2 * kk + (mi & 1);           // 16-byte chunk over the row
      const int hf = c >> 3, cc = c & 7;
      const uint32_t addr =
          smem_u32(st + hf * kTile * 128 + r_ld * 128 + ((cc ^ (r_ld & swz)) << 4));
      uint32_t b0, b1, b2, b3;
      ldsm_x4(addr, b0, b1, b2, b3);
      mma_bf16(acc[0], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
      mma_bf16(acc[1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    const int tw = t_begin + it * kTile + warp * 16;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float* row = hr == 0 ? row_lo : row_hi;
      if (!row) continue;   // padding head or a row no LLM head uses
      float v[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int pos = tw + (u >> 1) * 8 + 2 * tq + (u & 1);
        v[u] = acc[u >> 1][2 * hr + (u & 1)] * p.scale;
        ok[u] = pos < t_end;
        if (ok[u] && pos < N) {
          st_lo[hr] = fminf(st_lo[hr], v[u]);
          st_hi[hr] = fmaxf(st_hi[hr], v[u]);
        }
      }
      float tm = -FLT_MAX;
#pragma unroll
      for (int u = 0; u < 4; ++u) tm = ok[u] ? fmaxf(tm, v[u]) : tm;
      const float nm = fmaxf(st_m[hr], tm);
      float acc_s = st_s[hr] * __expf(st_m[hr] - nm);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc_s += ok[u] ? __expf(v[u] - nm) : 0.f;
      st_m[hr] = nm;
      st_s[hr] = acc_s;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (ok[u]) row[tw + (u >> 1) * 8 + 2 * tq + (u & 1)] = v[u];
    }
  }

  // ---- chunk statistics: lanes of a row (tq = 0..3), then the 4 warps (fixed order)
  __shared__ float4 sst[kConsumers][16];
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, st_m[hr], o);
      const float s2 = __shfl_xor_sync(0xffffffffu, st_s[hr], o);
      const float nm = fmaxf(st_m[hr], m2);
      st_s[hr] = st_s[hr] * __expf(st_m[hr] - nm) + s2 * __expf(m2 - nm);
      st_m[hr] = nm;
      st_lo[hr] = fminf(st_lo[hr], __shfl_xor_sync(0xffffffffu, st_lo[hr], o));
      st_hi[hr] = fmaxf(st_hi[hr], __shfl_xor_sync(0xffffffffu, st_hi[hr], o));
    }
    if (tq == 0) sst[warp][gq + 8 * hr] = make_float4(st_m[hr], st_s[hr], st_lo[hr], st_hi[hr]);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");   // consumers only
  if (warp == 0 && lane < 16 && lane < G && ((need >> lane) & 1u)) {
    float4 a = sst[0][lane];
#pragma unroll
    for (int w = 1; w < kConsumers; ++w) {
      const float4 c = sst[w][lane];
      const float nm = fmaxf(a.x, c.x);
      a.y = a.y * __expf(a.x - nm) + c.y * __expf(c.x - nm);
      a.x = nm;
      a.z = fminf(a.z, c.z);
      a.w = fmaxf(a.w, c.w);
    }
    p.stats[(static_cast<int64_t>(head0 + lane) * p.batch + b) * p.n_chunks + blockIdx.x] = a;
  }
}

// One CTA: flags of the head map's image and its compact, ascending list.
__global__ void row_flags_kernel(const int32_t* __restrict__ head_map, int32_t n_llm,
                                 int32_t n_slm, int32_t heads_per_layer,
                                 uint8_t* __restrict__ needed, int32_t* __restrict__ rows,
                                 int32_t* __restrict__ n_rows, int32_t* __restrict__ layer_off,
                                 int32_t* __restrict__ todo_count) {
  extern __shared__ uint8_t flags[];
  griddep_launch_dependents();   // K1 may be scheduled now; it waits for our completion
  if (threadIdx.x == 0) {
    todo_count[0] = 0;   // to-do list of the split (count, consumer ticket)
    todo_count[1] = 0;
  }
  for (int i = threadIdx.x; i < n_slm; i += blockDim.x) flags[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n_llm; i += blockDim.x) {
    const int j = head_map[i];
    if (j >= 0 && j < n_slm) flags[j] = 1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_slm; i += blockDim.x) needed[i] = flags[i];
  // one warp: the compact ascending list, and layer_off[l] = number of image
  // rows with flat head < l * heads_per_layer taken from the same running count
  if (threadIdx.x < 32) {
    const int n_layers = n_slm / heads_per_layer;
    int base = 0;
    for (int i0 = 0; i0 < n_slm; i0 += 32) {
      const int i = i0 + threadIdx.x;
      const bool f = i < n_slm && flags[i];
      const uint32_t bal = __ballot_sync(0xffffffffu, f);
      const uint32_t below = __popc(bal & lanemask_lt());
      if (f) rows[base + below] = i;
      // lane k: the layer boundary l * heads_per_layer that falls on position i
      if (i % heads_per_layer == 0 && i / heads_per_layer <= n_layers) layer_off[i / heads_per_layer] = base + below;
      base += __popc(bal);
    }
    if (threadIdx.x == 0) {
      *n_rows = base;
      layer_off[n_layers] = base;
    }
  }
}
}  // namespace

cudaError_t launch_row_flags(const int32_t* head_map, int32_t n_llm_heads, int32_t n_slm_heads,
                             int32_t heads_per_layer, uint8_t* row_needed, int32_t* rows,
                             int32_t* n_rows, int32_t* layer_off, int32_t* todo_count,
                             cudaStream_t s) {
  row_flags_kernel<<<1, 1024, n_slm_heads, s>>>(head_map, n_llm_heads, n_slm_heads,
                                               heads_per_layer, row_needed, rows, n_rows,
                                               layer_off, todo_count);
  return cudaGetLastError();
}

cudaError_t launch_slm_score(const SlmScoreParams& p, const CUtensorMap& map, int max_seq_len,
                             cudaStream_t s) {
  dim3 grid((max_seq_len + p.chunk_tokens - 1) / p.chunk_tokens, p.kv_heads,
            (p.layer_end - p.layer_begin) * p.batch);
  // programmatic dependent launch: the grid is scheduled during the previous
  // kernel's tail (row_flags) and waits for its completion in griddep_wait()
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (p.head_dim == 64) {
    constexpr int sm = smem_bytes<64>();
    cudaFuncSetAttribute(slm_score_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cfg.dynamicSmemBytes = sm;
    e = cudaLaunchKernelEx(&cfg, slm_score_kernel<64>, map, p);
  } else {
    constexpr int sm = smem_bytes<128>();
    cudaFuncSetAttribute(slm_score_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cfg.dynamicSmemBytes = sm;
    e = cudaLaunchKernelEx(&cfg, slm_score_kernel<128>, map, p);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace skv
