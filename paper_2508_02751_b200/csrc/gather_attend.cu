// gather_attend.cu — K3 (+ fused K4): SmallKV's compensated decode attention.
//
// Alg. 1 l.11-14, App. D SmallKV_attention_forward:
//   O_c = softmax over the critical ∪ recent tokens (R2: FlashAttention over
//         the selected K/V),
//   O_m = Σ_{k ∈ marginal} A'_{f(i)}[k] · V[k]   (Eq. 6 second branch),
//   O   = O_c + O_m                                (no renormalisation, R3).
//
// B200 design.  One CTA = (position chunk, LLM kv-group g, sequence b).  Every
// q-head h of the group may map to a different SLM row (D6), so the CTA first
// builds, in shared memory, a per-position 16-bit mask over its chunk (bits
// 0..7: h is critical/recent, bits 8..15: h is marginal) from the ascending
// lists of the DISTINCT rows its heads use (warp 32-ary searches bound the
// chunk's slice of each list), then compacts the positions with a non-zero
// mask.  Each K/V row is thus read from HBM once per group, however many
// heads select it; marginal-only rows read V only (their K is never touched,
// R11).  Each warp then streams its own 16-row tiles with cp.async (16-byte
// LDGSTS through the page table, XOR-swizzled rows, zero-filled tails) into a
// private multi-stage ring and runs, on the tensor cores (mma.sync m16n8k16):
//   S[16 x 16] = Q_group[16 x d] · K_tile^T        (heads = M, tokens = N)
//   O[16 x d] += A[16 x 16] · V_tile               (A rows 0..7: online-softmax
//                                                    weights p of head h;
//                                                    rows 8..15: marginal
//                                                    weights a' of head h)
// so the marginal compensation shares the PV contraction with the critical
// part (register-resident A, FA2-style), with A split into bf16 hi + lo parts
// (two MMAs) to keep ~2^-17 relative precision on the weights.  Warps merge in
// shared memory in a fixed order; chunks merge through a deterministic
// last-CTA log-sum-exp combine (K4 fused), so the result is bit-reproducible.
#include <float.h>
#include <limits.h>

#include "common.cuh"
#include "kernels.h"

namespace skv {

namespace {
constexpr int kTile = 16;      // rows (tokens) per warp tile
constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxChunk = 2048;   // positions are packed in 16 bits of the list

template <int D>
constexpr int stages_for() { return 3; }

template <int D>
constexpr int stage_bytes() {
  return 2 * kTile * D * 2 + kTile * 8 * 4 + kTile * 4;
}

// [list: chunk x u32][stages: kWarps x NSTAGE x stage]; the position mask of
// the prologue aliases the stage ring (dead until the tiles start).
template <int D>
constexpr size_t smem_bytes(int chunk) {
  return static_cast<size_t>(chunk) * 4 +
         static_cast<size_t>(kWarps) * stages_for<D>() * stage_bytes<D>();
}

// first index i in [0, len) with L[i] >= x (len if none); L ascending; whole warp.
__device__ __forceinline__ int warp_lower_bound(const int32_t* __restrict__ L, int len, int x) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = len;
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int idx = lo + lane * step;
    const int v = idx < hi ? __ldg(L + idx) : INT_MAX;
    const int c = __popc(__ballot_sync(0xffffffffu, v < x));
    if (c == 0) {
      hi = lo;
    } else {
      const int nlo = lo + (c - 1) * step + 1;
      hi = min(hi, lo + c * step);
      lo = nlo;
    }
  }
  const int idx = lo + lane;
  const int v = idx < hi ? __ldg(L + idx) : INT_MAX;
  return lo + __popc(__ballot_sync(0xffffffffu, v < x));
}

template <int D>
__global__ void __launch_bounds__(kThreads, 2) attend_kernel(const AttendParams p) {
  constexpr int NSTAGE = stages_for<D>();
  constexpr int ROWB = D * 2;                // bytes per K or V row
  constexpr int CH = D / 8;                  // 16-byte chunks per row
  constexpr int KV_BYTES = kTile * ROWB;
  constexpr int SB = stage_bytes<D>();
  constexpr int EPI = 32 / (2 * CH);         // entries loaded per warp iteration
  constexpr int NT = D / 8;                  // n8 tiles of the output

  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* list = reinterpret_cast<uint32_t*>(smem);
  uint8_t* stages = reinterpret_cast<uint8_t*>(list + p.chunk);
  uint32_t* mask = reinterpret_cast<uint32_t*>(stages);
  __shared__ int s_j[8], s_K[8], s_M[8];
  __shared__ float s_lse[8];
  __shared__ int s_wcnt[kWarps];
  __shared__ int s_last;

  const int c = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
  const int n = p.seq_lens[b];
  const int nch = (n + p.chunk - 1) / p.chunk;
  if (c >= nch) return;
  const int c0 = c * p.chunk, c1 = min(n, c0 + p.chunk), S = c1 - c0;
  const int G = p.heads / p.kv_heads;
  const int Rc = min(max(p.n_recent[b], 0), n);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t allc = (1u << G) - 1u;

  if (tid < G) {
    const int j = p.head_map[p.layer * p.heads + g * G + tid];
    const int64_t rb = static_cast<int64_t>(j) * p.batch + b;
    s_j[tid] = j;
    s_K[tid] = p.counts[rb * 2];
    s_M[tid] = p.counts[rb * 2 + 1];
    s_lse[tid] = p.lse[rb * 2 + 1];
  }
  for (int i = tid; i < S; i += kThreads) mask[i] = (c0 + i >= n - Rc) ? allc : 0u;
  __syncthreads();

  // ---- per-position head masks from the distinct rows' lists
  for (int li = warp; li < 2 * G; li += kWarps) {
    const int h = li % G;
    const bool isM = li >= G;
    const int j = s_j[h];
    bool dup = false;
    uint32_t bits = 0;
    for (int h2 = 0; h2 < G; ++h2) {
      if (s_j[h2] == j) {
        bits |= 1u << h2;
        if (h2 < h) dup = true;
      }
    }
    if (dup) continue;
    if (isM) bits <<= 8;
    const int64_t rb = static_cast<int64_t>(j) * p.batch + b;
    const int32_t* L = isM ? p.marg_idx + rb * p.max_marg : p.crit_idx + rb * p.max_crit;
    const int len = isM ? s_M[h] : s_K[h];
    const int lo = warp_lower_bound(L, len, c0);
    const int hi = warp_lower_bound(L, len, c1);
    for (int i = lo + lane; i < hi; i += 32) atomicOr(&mask[__ldg(L + i) - c0], bits);
  }
  __syncthreads();

  // ---- compact positions with a non-empty mask (ascending)
  const uint32_t ltm = lanemask_lt();
  {
    const int seg = ((S + kThreads - 1) / kThreads) * 32;
    const int s0 = warp * seg, s1 = min(S, s0 + seg);
    int cnt = 0;
    for (int base = s0; base < s1; base += 32) {
      const int i = base + lane;
      cnt += __popc(__ballot_sync(0xffffffffu, i < s1 && mask[i] != 0u));
    }
    if (lane == 0) s_wcnt[warp] = cnt;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += s_wcnt[w];
    for (int base = s0; base < s1; base += 32) {
      const int i = base + lane;
      const uint32_t mk = i < s1 ? mask[i] : 0u;
      const uint32_t bal = __ballot_sync(0xffffffffu, mk != 0u);
      if (mk) list[off + __popc(bal & ltm)] = (static_cast<uint32_t>(i) << 16) | (mk & 0xffffu);
      off += __popc(bal);
    }
  }
  __syncthreads();
  int E = 0;
  for (int w = 0; w < kWarps; ++w) E += s_wcnt[w];

  // ---- per-warp streaming over its tiles
  const int gq = lane >> 2, tq = lane & 3;
  const int ntile = (E + kTile - 1) / kTile;
  const int nmy = ntile > warp ? (ntile - warp + kWarps - 1) / kWarps : 0;
  uint8_t* wst = stages + warp * NSTAGE * SB;
  const uint16_t* kpool = p.k + p.layer_offset;
  const uint16_t* vpool = p.v + p.layer_offset;
  const int32_t* bt = p.block_table + static_cast<int64_t>(b) * p.max_blocks;

  uint32_t qa[D / 16][2];
  {
    const uint16_t* qg = p.q + (static_cast<int64_t>(b) * p.heads + g * G) * D;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int cc = 16 * kk + 2 * tq;
      qa[kk][0] = gq < G ? *reinterpret_cast<const uint32_t*>(qg + gq * D + cc) : 0u;
      qa[kk][1] = gq < G ? *reinterpret_cast<const uint32_t*>(qg + gq * D + cc + 8) : 0u;
    }
  }
  const float lse_h = gq < G ? s_lse[gq] : 0.f;

  auto issue = [&](int i) {
    if (i < nmy) {
      const int tile = warp + i * kWarps;
      uint8_t* st = wst + (i % NSTAGE) * SB;
      uint32_t* smask = reinterpret_cast<uint32_t*>(st + 2 * KV_BYTES + kTile * 8 * 4);
      float* sml = reinterpret_cast<float*>(st + 2 * KV_BYTES);
      const int e = tile * kTile + (lane & 15);
      const bool ev = e < E;
      const uint32_t pk = ev ? list[e] : 0u;
      const int pos = c0 + static_cast<int>(pk >> 16);
      const uint32_t mk = pk & 0xffffu;
      int64_t roff = 0;
      if (ev) {
        const int page = bt[pos / p.page_size];
        roff = ((static_cast<int64_t>(page) * p.kv_heads + g) * p.page_size + pos % p.page_size) * D;
      }
      if (lane < kTile) smask[lane] = mk;
#pragma unroll
      for (int e0 = 0; e0 < kTile; e0 += EPI) {
        const int eo = e0 + lane / (2 * CH);       // entry this lane copies
        const int ch = lane % (2 * CH);            // chunk 0..2CH-1 (K then V)
        const int64_t ro = __shfl_sync(0xffffffffu, roff, eo);
        const uint32_t me = __shfl_sync(0xffffffffu, mk, eo);
        const bool ve = __shfl_sync(0xffffffffu, ev, eo);
        if (ch < CH) {
          if (me & 0xffu) {
            const uint32_t dst = smem_u32(st + eo * ROWB + ((ch ^ (eo & 7)) << 4));
            cp_async16(dst, kpool + ro + ch * 8, true);
          }
        } else {
          const int cv = ch - CH;
          const uint32_t dst = smem_u32(st + KV_BYTES + eo * ROWB + ((cv ^ (eo & 7)) << 4));
          cp_async16(dst, vpool + (ve ? ro + cv * 8 : 0), ve);
        }
      }
      // marginal logits a'-numerators: 16 entries x 8 heads
#pragma unroll
      for (int q4 = 0; q4 < (kTile * 8) / 32; ++q4) {
        const int idx = q4 * 32 + lane;
        const int eo = idx >> 3, h = idx & 7;
        const uint32_t me = __shfl_sync(0xffffffffu, mk, eo);
        const int po = __shfl_sync(0xffffffffu, pos, eo);
        if (h < G && ((me >> (8 + h)) & 1u))
          cp_async4(smem_u32(sml + idx),
                    p.logits + (static_cast<int64_t>(s_j[h]) * p.batch + b) * p.row_stride + po);
      }
    }
    cp_async_commit();
  };

  float o[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  const int mi = lane >> 3;

#pragma unroll
  for (int i = 0; i < NSTAGE - 1; ++i) issue(i);
  for (int i = 0; i < nmy; ++i) {
    issue(i + NSTAGE - 1);
    cp_async_wait<NSTAGE - 1>();
    __syncwarp();
    const uint8_t* st = wst + (i % NSTAGE) * SB;
    const uint8_t* kb = st;
    const uint8_t* vb = st + KV_BYTES;
    const float* sml = reinterpret_cast<const float*>(st + 2 * KV_BYTES);
    const uint32_t* smask = reinterpret_cast<const uint32_t*>(st + 2 * KV_BYTES + kTile * 8 * 4);

    // S = Q K^T : rows = heads, cols = 16 tokens (two n8 tiles)
    float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int r = ((mi >> 1) << 3) + (lane & 7);
      const int ch = 2 * kk + (mi & 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(smem_u32(kb + r * ROWB + ((ch ^ (r & 7)) << 4)), b0, b1, b2, b3);
      mma_bf16(sacc[0], qa[kk][0], 0u, qa[kk][1], 0u, b0, b1);
      mma_bf16(sacc[1], qa[kk][0], 0u, qa[kk][1], 0u, b2, b3);
    }
    // masks / weights for this lane's head gq and tokens {2tq, 2tq+1, 8+2tq, 9+2tq}
    float sv[4], wm[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int tok = (u >> 1) * 8 + 2 * tq + (u & 1);
      const uint32_t mk = smask[tok];
      const bool crit = gq < G && ((mk >> gq) & 1u);
      const bool marg = gq < G && ((mk >> (8 + gq)) & 1u);
      sv[u] = crit ? sacc[u >> 1][u & 1] * p.scale_log2 : -INFINITY;
      wm[u] = marg ? expf(sml[tok * 8 + gq] - lse_h) : 0.f;
    }
    float tmax = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float m_new = fmaxf(m_run, tmax);
    const float m_use = m_new == -INFINITY ? 0.f : m_new;
    const float alpha = exp2f(m_run - m_use);
    float pw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) pw[u] = exp2f(sv[u] - m_use);
    l_run = l_run * alpha + (pw[0] + pw[1] + pw[2] + pw[3]);
    m_run = m_new;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      o[t][0] *= alpha;
      o[t][1] *= alpha;
    }
    // A fragments (rows gq: p; rows gq+8: a'), hi + lo
    uint32_t ah[4], al[4];
    split_bf16x2(pw[0], pw[1], ah[0], al[0]);
    split_bf16x2(wm[0], wm[1], ah[1], al[1]);
    split_bf16x2(pw[2], pw[3], ah[2], al[2]);
    split_bf16x2(wm[2], wm[3], ah[3], al[3]);
    // O += A · V
#pragma unroll
    for (int t = 0; t < NT; t += 2) {
      const int r = ((mi & 1) << 3) + (lane & 7);
      const int ch = t + (mi >> 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(smem_u32(vb + r * ROWB + ((ch ^ (r & 7)) << 4)), b0, b1, b2, b3);
      mma_bf16(o[t], ah[0], ah[1], ah[2], ah[3], b0, b1);
      mma_bf16(o[t], al[0], al[1], al[2], al[3], b0, b1);
      mma_bf16(o[t + 1], ah[0], ah[1], ah[2], ah[3], b2, b3);
      mma_bf16(o[t + 1], al[0], al[1], al[2], al[3], b2, b3);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  __syncthreads();   // every warp is done with its stages: reuse them for the merge

  // ---- merge warps (fixed order)
  float* wm_s = reinterpret_cast<float*>(stages);              // [kWarps][8]
  float* wl_s = wm_s + kWarps * 8;                              // [kWarps][8]
  float* wo_s = wl_s + kWarps * 8;                              // [kWarps][16][D]
  {
    float* myo = wo_s + warp * 16 * D;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int col = t * 8 + 2 * tq;
      myo[gq * D + col] = o[t][0];
      myo[gq * D + col + 1] = o[t][1];
      myo[(gq + 8) * D + col] = o[t][2];
      myo[(gq + 8) * D + col + 1] = o[t][3];
    }
    if (tq == 0) {
      wm_s[warp * 8 + gq] = m_run;
      wl_s[warp * 8 + gq] = l_run;
    }
  }
  __syncthreads();
  const int H = p.heads;
  const int64_t bh0 = static_cast<int64_t>(b) * H + g * G;
  for (int idx = tid; idx < G * D; idx += kThreads) {
    const int h = idx / D, col = idx % D;
    float M = -INFINITY;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, wm_s[w * 8 + h]);
    const float Mu = M == -INFINITY ? 0.f : M;
    float L = 0.f, oc = 0.f, om = 0.f;
    for (int w = 0; w < kWarps; ++w) {
      const float sc = exp2f(wm_s[w * 8 + h] - Mu);
      L += wl_s[w * 8 + h] * sc;
      oc += wo_s[(w * 16 + h) * D + col] * sc;
      om += wo_s[(w * 16 + h + 8) * D + col];
    }
    if (nch == 1) {
      p.out[(bh0 + h) * D + col] = (L > 0.f ? oc / L : 0.f) + om;
    } else {
      float* part = p.partials + ((bh0 + h) * p.max_chunks + c) * (2 + 2 * D);
      if (col == 0) {
        part[0] = M;
        part[1] = L;
      }
      part[2 + col] = oc;
      part[2 + D + col] = om;
    }
  }
  if (nch == 1) return;

  // ---- fused K4: the last chunk CTA of (b, g) combines all chunks in order
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int prev = atomicAdd(&p.counters[b * p.kv_heads + g], 1);
    s_last = prev == nch - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int idx = tid; idx < G * D; idx += kThreads) {
    const int h = idx / D, col = idx % D;
    const float* part0 = p.partials + (bh0 + h) * p.max_chunks * (2 + 2 * D);
    float M = -INFINITY;
    for (int q = 0; q < nch; ++q) M = fmaxf(M, __ldcg(part0 + q * (2 + 2 * D)));
    const float Mu = M == -INFINITY ? 0.f : M;
    float L = 0.f, oc = 0.f, om = 0.f;
    for (int q = 0; q < nch; ++q) {
      const float* pq = part0 + q * (2 + 2 * D);
      const float sc = exp2f(__ldcg(pq) - Mu);
      L += __ldcg(pq + 1) * sc;
      oc += __ldcg(pq + 2 + col) * sc;
      om += __ldcg(pq + 2 + D + col);
    }
    p.out[(bh0 + h) * D + col] = (L > 0.f ? oc / L : 0.f) + om;
  }
  if (tid == 0) p.counters[b * p.kv_heads + g] = 0;
}
}  // namespace

int32_t attend_chunk_size(int32_t max_seq_len) {
  (void)max_seq_len;
  static_assert(1024 <= kMaxChunk, "chunk too large for the packed list");
  return 1024;
}

size_t attend_partials_floats(int32_t batch, int32_t heads, int32_t head_dim, int32_t max_chunks) {
  return static_cast<size_t>(batch) * heads * max_chunks * (2 + 2 * head_dim);
}

cudaError_t launch_attend(const AttendParams& p, cudaStream_t s) {
  dim3 grid(p.max_chunks, p.kv_heads, p.batch);
  if (p.head_dim == 64) {
    const size_t sm = smem_bytes<64>(p.chunk);
    cudaFuncSetAttribute(attend_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm));
    attend_kernel<64><<<grid, kThreads, sm, s>>>(p);
  } else {
    const size_t sm = smem_bytes<128>(p.chunk);
    cudaFuncSetAttribute(attend_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm));
    attend_kernel<128><<<grid, kThreads, sm, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace skv
