// smallkv_api.cu — the C ABI of libsmallkv.so (include/smallkv.h): argument
// validation, workspace layout, TMA descriptor encoding and kernel launches.
// No device memory is allocated and no stream is synchronised here.
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"
#include "smallkv.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SMALLKV_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }
bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }
size_t round256(size_t x) { return (x + 255) & ~size_t(255); }

int check_device() {
  static std::atomic<int> state[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(SMALLKV_ERR_DEVICE, "device index %d out of range", dev);
  int st = state[dev].load(std::memory_order_relaxed);
  if (st == 0) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    st = (major == 10 && minor == 0) ? 1 : 2;
    state[dev].store(st, std::memory_order_relaxed);
  }
  if (st != 1) return fail(SMALLKV_ERR_DEVICE, "device %d is not sm_100 (B200)", dev);
  return SMALLKV_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int check_cache(const smallkv_cache* c, bool need_v, const char* name) {
  if (!c) return fail(SMALLKV_ERR_NULL, "%s cache is NULL", name);
  if (!c->k || !c->block_table || (need_v && !c->v))
    return fail(SMALLKV_ERR_NULL, "%s cache: k/v/block_table NULL", name);
  if (c->head_dim != 64 && c->head_dim != 128)
    return fail(SMALLKV_ERR_SHAPE, "%s head_dim %d not in {64,128}", name, c->head_dim);
  if (!pow2(c->page_size) || c->page_size > 256)
    return fail(SMALLKV_ERR_SHAPE, "%s page_size %d not a power of two in [1,256]", name,
                c->page_size);
  if (c->num_layers < 1 || c->num_q_heads < 1 || c->num_kv_heads < 1 || c->num_pages < 1 ||
      c->max_blocks < 1)
    return fail(SMALLKV_ERR_SHAPE, "%s cache: non-positive dimension", name);
  if (c->num_q_heads % c->num_kv_heads != 0)
    return fail(SMALLKV_ERR_SHAPE, "%s: %d q heads not a multiple of %d kv heads", name,
                c->num_q_heads, c->num_kv_heads);
  if (!aligned(c->k, 16) || (c->v && !aligned(c->v, 16)) || !aligned(c->block_table, 4))
    return fail(SMALLKV_ERR_ALIGN, "%s cache pools must be 16-byte aligned", name);
  return SMALLKV_OK;
}

int check_batch(const smallkv_batch* b, const smallkv_cache* c) {
  if (!b || !b->seq_lens) return fail(SMALLKV_ERR_NULL, "batch or seq_lens NULL");
  if (b->batch < 1 || b->batch > 65535 || b->max_seq_len < 1)
    return fail(SMALLKV_ERR_SHAPE, "batch %d / max_seq_len %d out of range", b->batch,
                b->max_seq_len);
  if (static_cast<int64_t>(c->max_blocks) * c->page_size < b->max_seq_len)
    return fail(SMALLKV_ERR_SHAPE, "block table covers %lld tokens < max_seq_len %d",
                static_cast<long long>(c->max_blocks) * c->page_size, b->max_seq_len);
  return SMALLKV_OK;
}

int check_budgets(const smallkv_budgets* bu) {
  if (!bu || !bu->k_crit || !bu->n_recent || !bu->k_marg)
    return fail(SMALLKV_ERR_NULL, "budgets NULL");
  if (bu->max_crit < 1 || bu->max_marg < 1)
    return fail(SMALLKV_ERR_SHAPE, "max_crit/max_marg must be >= 1");
  return SMALLKV_OK;
}

constexpr int kScoreChunk = 1024;   // tokens per K1 CTA = per row-statistics chunk (512/2048 measured no better)

struct SelectWs {
  size_t flags, rows, nrows, layer_off, todo_count, todo, stats, total;
};
SelectWs select_ws_layout(int32_t n_slm, int32_t n_layers, int32_t batch, int32_t max_seq_len) {
  SelectWs w;
  w.flags = 0;
  w.rows = round256(static_cast<size_t>(n_slm));
  w.nrows = w.rows + round256(static_cast<size_t>(n_slm) * 4);
  w.layer_off = w.nrows + 256;
  w.todo_count = w.layer_off + round256(static_cast<size_t>(n_layers + 1) * 4);
  w.todo = w.todo_count + 256;
  w.stats = w.todo + round256(static_cast<size_t>(n_slm) * batch * 4);
  const size_t nch = (static_cast<size_t>(max_seq_len) + kScoreChunk - 1) / kScoreChunk;
  w.total = w.stats + round256(static_cast<size_t>(n_slm) * batch * nch * 16);
  return w;
}

// smallkv_select_group: the SelectWs block, then the group rows' split inputs
// (identity row list, layer offsets, one statistics chunk per row) and scratch
// for the split's single-weight outputs (replaced by the per-head weights).
struct GroupWs {
  size_t rows, layer_off, gstats, lse, mw, todo, total;
};
GroupWs group_ws_layout(const smallkv_cache* slm, const smallkv_batch* b, int32_t max_marg,
                        int32_t n_llm_layers, int32_t llm_kv_heads) {
  GroupWs w;
  const size_t base =
      select_ws_layout(slm->num_layers * slm->num_q_heads, slm->num_layers, b->batch, b->max_seq_len).total;
  const size_t ng = static_cast<size_t>(n_llm_layers) * llm_kv_heads;
  w.rows = base;
  w.layer_off = w.rows + round256(ng * 4);
  w.gstats = w.layer_off + 256;
  w.lse = w.gstats + round256(ng * b->batch * 16);
  w.mw = w.lse + round256(ng * b->batch * 8);
  w.todo = w.mw + round256(ng * b->batch * static_cast<size_t>(max_marg) * 4);
  w.total = w.todo + round256(ng * b->batch * 4);
  return w;
}

struct AttendWs {
  size_t partials, tickets, total;
  int32_t ctas;
  bool cluster;
};
// The attend kernel merges a group's split work inside a thread-block cluster
// (distributed shared memory) when the GPU co-schedules it; otherwise through
// per-CTA partial states in the workspace and a per-group ticket (zeroed once
// by the caller, left zeroed by every launch).
AttendWs attend_ws_layout(const smallkv_cache* llm, const smallkv_batch* b) {
  AttendWs w;
  w.ctas = skv::attend_ctas_per_group(b->batch, llm->num_kv_heads, b->max_seq_len);
  w.cluster = skv::attend_split_in_cluster(b->batch, llm->num_kv_heads, b->max_seq_len);
  const size_t groups = static_cast<size_t>(b->batch) * llm->num_kv_heads;
  w.tickets = 0;
  w.partials = round256(groups * 4);
  w.total = w.cluster ? 256
                      : w.partials + round256(groups * w.ctas * skv::kAttendPartFloats * sizeof(float));
  return w;
}

}  // namespace

extern "C" {

const char* smallkv_last_error(void) { return g_err.c_str(); }
const char* smallkv_version(void) { return "smallkv-b200 0.1 (sm_100a)"; }

int smallkv_budget_from_tau(double tau, int32_t n, int32_t* k_crit, int32_t* n_recent,
                            int32_t* k_marg) {
  if (!k_crit || !n_recent || !k_marg) return fail(SMALLKV_ERR_NULL, "NULL output");
  if (!(tau > 0.0 && tau <= 1.0) || n < 0)
    return fail(SMALLKV_ERR_SHAPE, "tau %g must be in (0,1], n %d >= 0", tau, n);
  // 2:1:2 critical:recent:marginal; marginal costs half (V only), so the
  // token fractions are tau/2, tau/4, tau/2.  The epsilon absorbs binary
  // rounding of tau*n (e.g. 0.35*200 = 69.999..).
  const double x = tau * static_cast<double>(n);
  *k_crit = static_cast<int32_t>(std::floor(x / 2.0 + 1e-9));
  *n_recent = static_cast<int32_t>(std::floor(x / 4.0 + 1e-9));
  *k_marg = static_cast<int32_t>(std::floor(x / 2.0 + 1e-9));
  return SMALLKV_OK;
}

size_t smallkv_select_workspace_size(const smallkv_cache* slm, const smallkv_batch* batch,
                                     int32_t n_llm_heads) {
  if (!slm || !batch || n_llm_heads < 1) return 0;
  return select_ws_layout(slm->num_layers * slm->num_q_heads, slm->num_layers, batch->batch,
                          batch->max_seq_len).total;
}

}  // extern "C"

namespace {
// Shared front half of smallkv_select / smallkv_select_group: argument checks,
// the SLM K' tensor map, the image-of-f flags (row_flags launch on `s`) and the
// K1 / K2 parameter blocks.  ws holds the SelectWs layout at offset 0.
struct ScoringSetup {
  CUtensorMap map;
  skv::SlmScoreParams sp;
  skv::SelectParams se;
};
int setup_scoring(const uint16_t* slm_q, const smallkv_cache* slm, const smallkv_batch* batch,
                  const int32_t* head_map, int32_t n_llm_heads, const smallkv_budgets* budgets,
                  float* slm_logits, float* slm_lse, void* ws, size_t ws_bytes, size_t ws_need,
                  cudaStream_t s, ScoringSetup& S) {
  int rc;
  if ((rc = check_cache(slm, false, "slm")) != SMALLKV_OK) return rc;
  if ((rc = check_batch(batch, slm)) != SMALLKV_OK) return rc;
  if ((rc = check_budgets(budgets)) != SMALLKV_OK) return rc;
  if (!slm_q || !head_map || !slm_logits || !slm_lse)
    return fail(SMALLKV_ERR_NULL, "smallkv_select: NULL input/output pointer");
  if (n_llm_heads < 1) return fail(SMALLKV_ERR_SHAPE, "n_llm_heads must be >= 1");
  const int G_s = slm->num_q_heads / slm->num_kv_heads;
  if (G_s > 16) return fail(SMALLKV_ERR_SHAPE, "SLM GQA group %d > 16", G_s);
  const int n_slm = slm->num_layers * slm->num_q_heads;
  if (n_slm > 32768) return fail(SMALLKV_ERR_SHAPE, "l*H_s = %d > 32768", n_slm);
  if (static_cast<int64_t>(slm->num_layers) * batch->batch > 65535)
    return fail(SMALLKV_ERR_SHAPE, "l*B = %lld > 65535",
                static_cast<long long>(slm->num_layers) * batch->batch);
  const int64_t rows_total =
      static_cast<int64_t>(slm->num_layers) * slm->num_pages * slm->num_kv_heads * slm->page_size;
  if (rows_total >= (int64_t(1) << 31))
    return fail(SMALLKV_ERR_SHAPE, "SLM pool has %lld rows (>= 2^31)",
                static_cast<long long>(rows_total));
  if (!aligned(slm_q, 4)) return fail(SMALLKV_ERR_ALIGN, "slm_q must be 4-byte aligned");
  const SelectWs L = select_ws_layout(n_slm, slm->num_layers, batch->batch, batch->max_seq_len);
  if (!ws || ws_bytes < ws_need)
    return fail(SMALLKV_ERR_WORKSPACE, "select workspace %zu < %zu bytes", ws_bytes, ws_need);
  if ((rc = check_device()) != SMALLKV_OK) return rc;

  auto fn = encode_fn();
  if (!fn) return fail(SMALLKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int d = slm->head_dim;
  const int box_rows = slm->page_size < 64 ? slm->page_size : 64;
  const bool swz = slm->page_size >= 8;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows_total)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(d) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = fn(&S.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(slm->k), gdim,
                   gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(SMALLKV_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", cr);

  uint8_t* wsb = static_cast<uint8_t*>(ws);
  uint8_t* flags = wsb + L.flags;
  int32_t* rows = reinterpret_cast<int32_t*>(wsb + L.rows);
  int32_t* nrows = reinterpret_cast<int32_t*>(wsb + L.nrows);
  int32_t* layer_off = reinterpret_cast<int32_t*>(wsb + L.layer_off);
  int32_t* todo_count = reinterpret_cast<int32_t*>(wsb + L.todo_count);
  cudaError_t e = skv::launch_row_flags(head_map, n_llm_heads, n_slm, slm->num_q_heads, flags,
                                        rows, nrows, layer_off, todo_count, s);
  if (e != cudaSuccess) return cuda_fail(e, "row_flags launch");

  skv::SlmScoreParams& sp = S.sp;
  sp = skv::SlmScoreParams{};
  sp.q = slm_q;
  sp.block_table = slm->block_table;
  sp.seq_lens = batch->seq_lens;
  sp.row_needed = flags;
  sp.logits = slm_logits;
  sp.num_pages = slm->num_pages;
  sp.max_blocks = slm->max_blocks;
  sp.page_size = slm->page_size;
  sp.layers = slm->num_layers;
  sp.heads = slm->num_q_heads;
  sp.kv_heads = slm->num_kv_heads;
  sp.head_dim = d;
  sp.batch = batch->batch;
  sp.row_stride = batch->max_seq_len;
  sp.chunk_tokens = kScoreChunk;
  sp.n_recent = budgets->n_recent;
  sp.stats = reinterpret_cast<float4*>(wsb + L.stats);
  sp.n_chunks = (batch->max_seq_len + kScoreChunk - 1) / kScoreChunk;
  sp.box_rows = box_rows;
  sp.swz = swz ? 7u : 0u;
  sp.scale = 1.0f / std::sqrt(static_cast<float>(d));
  skv::SelectParams& se = S.se;
  se = skv::SelectParams{};
  se.logits = slm_logits;
  se.seq_lens = batch->seq_lens;
  se.rows = rows;
  se.layer_off = layer_off;
  se.k_crit = budgets->k_crit;
  se.n_recent = budgets->n_recent;
  se.k_marg = budgets->k_marg;
  se.lse = slm_lse;
  se.batch = batch->batch;
  se.row_stride = batch->max_seq_len;
  se.max_crit = budgets->max_crit;
  se.max_marg = budgets->max_marg;
  se.stats = sp.stats;
  se.n_chunks = sp.n_chunks;
  se.chunk_tokens = kScoreChunk;
  se.todo_count = todo_count;
  se.todo = reinterpret_cast<int32_t*>(wsb + L.todo);
  return SMALLKV_OK;
}

// K2 over SLM layers [se.layer_begin, se.layer_end): long rows by thread-block
// clusters (select_cluster.cu; f1's in-place running sums stay on the
// single-CTA split), others by one CTA per row
cudaError_t launch_split(const skv::SelectParams& se, int32_t max_rows, int32_t max_seq_len,
                         bool overlap_previous, cudaStream_t s) {
  // measured on B200 (config 4, 131072 tokens): with >= 1024 (row, sequence)
  // pairs one CTA per pair fills the GPU (B = 8: 3.13 ms vs 3.29 with clusters
  // of 4); with fewer, clusters of 2 halve the split (B = 1: 0.58 vs 1.05 ms)
  static const bool forced = getenv("SMALLKV_SPLIT_CLUSTER") != nullptr;   // tuning knob (select_cluster.cu)
  const int64_t pairs = static_cast<int64_t>(max_rows) * se.batch;
  if (!se.acc && max_seq_len > skv::kClusterSplitMinLen && (pairs < 1024 || forced))
    return skv::launch_select_cluster(se, max_rows, pairs < 256 ? 4 : 2, s);
  return skv::launch_select(se, max_rows, max_seq_len, overlap_previous, s);
}
}  // namespace

extern "C" {

int smallkv_select(const uint16_t* slm_q, const smallkv_cache* slm, const smallkv_batch* batch,
                   const int32_t* head_map, int32_t n_llm_heads, const smallkv_budgets* budgets,
                   float* slm_logits, float* slm_lse, int32_t* crit_idx, int32_t* marg_idx,
                   float* marg_w, int32_t* counts, float* acc, void* ws, size_t ws_bytes,
                   void* stream, void* aux_stream) {
  int rc0;
  if ((rc0 = check_cache(slm, false, "slm")) != SMALLKV_OK) return rc0;
  if ((rc0 = check_batch(batch, slm)) != SMALLKV_OK) return rc0;
  if ((rc0 = check_budgets(budgets)) != SMALLKV_OK) return rc0;
  if (!crit_idx || !marg_idx || !marg_w || !counts)
    return fail(SMALLKV_ERR_NULL, "smallkv_select: NULL input/output pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ScoringSetup S;
  const size_t need = smallkv_select_workspace_size(slm, batch, n_llm_heads > 0 ? n_llm_heads : 1);
  int rc = setup_scoring(slm_q, slm, batch, head_map, n_llm_heads, budgets, slm_logits, slm_lse,
                         ws, ws_bytes, need, s, S);
  if (rc != SMALLKV_OK) return rc;
  cudaError_t e;
  skv::SlmScoreParams& sp = S.sp;
  skv::SelectParams& se = S.se;
  const CUtensorMap& map = S.map;
  se.crit_idx = crit_idx;
  se.marg_idx = marg_idx;
  se.marg_w = marg_w;
  se.counts = counts;
  se.acc = acc;
  // Score the SLM layers in chunks.  With an auxiliary stream the split of
  // chunk i (ALU-bound K2) runs on it concurrently with the scoring of chunk
  // i+1 (HBM-bound K1) on the main stream — the paper's "update KV cache in
  // parallel" (Alg. 1 l.8-9) applied inside the selection; the main
  // stream then waits for the last split.  Without one, the chunks run in order.
  const int nl = slm->num_layers;
  static const int chunks_env = [] {
    const char* e = getenv("SMALLKV_SELECT_CHUNKS");   // tuning knob
    return e ? atoi(e) : 0;
  }();
  // With an auxiliary stream the chunks are sized so that a chunk's score rows
  // stay L2-resident until its split reads them (kChunkRowBytes of rows per
  // chunk, at least one SLM layer): K2 then re-reads them from L2 while K1
  // streams the next chunk's K' from HBM.
  constexpr size_t kChunkRowBytes = size_t(48) << 20;
  const size_t layer_rows = static_cast<size_t>(slm->num_q_heads) * batch->batch * batch->max_seq_len * 4;
  int per_chunk = static_cast<int>(kChunkRowBytes / (layer_rows > 0 ? layer_rows : 1));
  if (per_chunk < 1) per_chunk = 1;
  int want = chunks_env > 0 ? chunks_env : (aux_stream ? (nl + per_chunk - 1) / per_chunk : 1);
  if (want < 1) want = 1;
  const int nchunk = nl < want ? nl : want;
  cudaStream_t aux = static_cast<cudaStream_t>(aux_stream);
  auto chunk_lo = [&](int i) { return (nl * i) / nchunk; };
  auto launch_k2 = [&](int i, cudaStream_t st) {
    se.layer_begin = chunk_lo(i);
    se.layer_end = chunk_lo(i + 1);
    const int rows_max = (se.layer_end - se.layer_begin) * slm->num_q_heads;
    return launch_split(se, rows_max < n_llm_heads ? rows_max : n_llm_heads, batch->max_seq_len,
                        true, st);
  };
  const int nev = aux && nchunk > 1 ? nchunk + 1 : 0;
  std::vector<cudaEvent_t> evs(static_cast<size_t>(nev), nullptr);
  for (int i = 0; i < nev; ++i) {
    e = cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      for (int k = 0; k < i; ++k) cudaEventDestroy(evs[k]);
      return cuda_fail(e, "cudaEventCreate");
    }
  }
  int rc2 = SMALLKV_OK;
  for (int i = 0; i < nchunk && rc2 == SMALLKV_OK; ++i) {
    sp.layer_begin = chunk_lo(i);
    sp.layer_end = chunk_lo(i + 1);
    e = skv::launch_slm_score(sp, map, batch->max_seq_len, s);
    if (e != cudaSuccess) { rc2 = cuda_fail(e, "slm_score launch"); break; }
    if (nev) {
      if ((e = cudaEventRecord(evs[i], s)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(aux, evs[i], 0)) != cudaSuccess) {
        rc2 = cuda_fail(e, "fork to aux stream");
        break;
      }
      e = launch_k2(i, aux);
    } else {
      e = launch_k2(i, s);
    }
    if (e != cudaSuccess) rc2 = cuda_fail(e, "select launch");
  }
  if (nev && rc2 == SMALLKV_OK) {
    if ((e = cudaEventRecord(evs[nchunk], aux)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s, evs[nchunk], 0)) != cudaSuccess)
      rc2 = cuda_fail(e, "join from aux stream");
  }
  for (int i = 0; i < nev; ++i) cudaEventDestroy(evs[i]);
  return rc2;
}

size_t smallkv_select_group_workspace_size(const smallkv_cache* slm, const smallkv_batch* batch,
                                           const smallkv_budgets* budgets, int32_t n_llm_layers,
                                           int32_t llm_kv_heads) {
  if (!slm || !batch || !budgets || n_llm_layers < 1 || llm_kv_heads < 1 || batch->batch < 1 ||
      batch->max_seq_len < 1 || budgets->max_marg < 1)
    return 0;
  return group_ws_layout(slm, batch, budgets->max_marg, n_llm_layers, llm_kv_heads).total;
}

int smallkv_select_group(const uint16_t* slm_q, const smallkv_cache* slm, const smallkv_batch* batch,
                         const int32_t* head_map, int32_t n_llm_layers, int32_t llm_q_heads,
                         int32_t llm_kv_heads, const smallkv_budgets* budgets, float* slm_logits,
                         float* slm_lse, float* group_score, int32_t* crit_idx, int32_t* marg_idx,
                         float* marg_w, int32_t* counts, void* ws, size_t ws_bytes, void* stream) {
  int rc0;
  if ((rc0 = check_cache(slm, false, "slm")) != SMALLKV_OK) return rc0;
  if ((rc0 = check_batch(batch, slm)) != SMALLKV_OK) return rc0;
  if ((rc0 = check_budgets(budgets)) != SMALLKV_OK) return rc0;
  if (!group_score || !crit_idx || !marg_idx || !marg_w || !counts)
    return fail(SMALLKV_ERR_NULL, "smallkv_select_group: NULL output pointer");
  if (n_llm_layers < 1 || llm_q_heads < 1 || llm_kv_heads < 1 || llm_q_heads % llm_kv_heads != 0)
    return fail(SMALLKV_ERR_SHAPE, "LLM layers/heads (%d, %d, %d) invalid", n_llm_layers, llm_q_heads,
                llm_kv_heads);
  if (llm_q_heads / llm_kv_heads > 8)
    return fail(SMALLKV_ERR_SHAPE, "LLM GQA group %d > 8 not supported", llm_q_heads / llm_kv_heads);
  if (static_cast<int64_t>(n_llm_layers) * llm_kv_heads > 65535)
    return fail(SMALLKV_ERR_SHAPE, "L*H_kv > 65535");
  if (!aligned(marg_w, 16)) return fail(SMALLKV_ERR_ALIGN, "marg_w must be 16-byte aligned");
  const size_t need =
      smallkv_select_group_workspace_size(slm, batch, budgets, n_llm_layers, llm_kv_heads);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ScoringSetup S;
  const int32_t n_llm_heads = n_llm_layers * llm_q_heads;
  int rc = setup_scoring(slm_q, slm, batch, head_map, n_llm_heads, budgets, slm_logits, slm_lse, ws,
                         ws_bytes, need, s, S);
  if (rc != SMALLKV_OK) return rc;
  // K1 over all SLM layers
  S.sp.layer_begin = 0;
  S.sp.layer_end = slm->num_layers;
  cudaError_t e = skv::launch_slm_score(S.sp, S.map, batch->max_seq_len, s);
  if (e != cudaSuccess) return cuda_fail(e, "slm_score launch");
  // group score rows
  const GroupWs W = group_ws_layout(slm, batch, budgets->max_marg, n_llm_layers, llm_kv_heads);
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  skv::GroupParams gp{};
  gp.logits = slm_logits;
  gp.stats = S.sp.stats;
  gp.n_chunks = S.sp.n_chunks;
  gp.chunk_tokens = S.sp.chunk_tokens;
  gp.head_map = head_map;
  gp.seq_lens = batch->seq_lens;
  gp.n_recent = budgets->n_recent;
  gp.slm_lse = slm_lse;
  gp.score = group_score;
  gp.gstats = reinterpret_cast<float4*>(wsb + W.gstats);
  gp.rows = reinterpret_cast<int32_t*>(wsb + W.rows);
  gp.layer_off = reinterpret_cast<int32_t*>(wsb + W.layer_off);
  gp.counts = counts;
  gp.marg_idx = marg_idx;
  gp.marg_w8 = marg_w;
  gp.L = n_llm_layers;
  gp.H = llm_q_heads;
  gp.H_kv = llm_kv_heads;
  gp.batch = batch->batch;
  gp.row_stride = batch->max_seq_len;
  gp.max_marg = budgets->max_marg;
  if ((e = skv::launch_group_score(gp, s)) != cudaSuccess) return cuda_fail(e, "group_score launch");
  // the split (K2) on the group rows: ranked by F_g; its single-weight outputs
  // go to scratch and are replaced by the per-head weights below
  skv::SelectParams se = S.se;
  se.logits = group_score;
  se.rows = gp.rows;
  se.layer_off = gp.layer_off;
  se.layer_begin = 0;
  se.layer_end = 1;
  se.lse = reinterpret_cast<float*>(wsb + W.lse);
  se.crit_idx = crit_idx;
  se.marg_idx = marg_idx;
  se.marg_w = reinterpret_cast<float*>(wsb + W.mw);
  se.counts = counts;
  se.stats = gp.gstats;
  se.acc = nullptr;
  se.n_chunks = 1;
  se.chunk_tokens = batch->max_seq_len;
  se.log_bins = 1;
  se.todo = reinterpret_cast<int32_t*>(wsb + W.todo);
  if ((e = launch_split(se, n_llm_layers * llm_kv_heads, batch->max_seq_len, false, s)) != cudaSuccess)
    return cuda_fail(e, "select launch");
  if ((e = skv::launch_group_weights(gp, s)) != cudaSuccess) return cuda_fail(e, "group_weights launch");
  return SMALLKV_OK;
}

size_t smallkv_attend_workspace_size(const smallkv_cache* llm, const smallkv_batch* batch) {
  if (!llm || !batch || batch->batch < 1 || batch->max_seq_len < 1) return 0;
  return attend_ws_layout(llm, batch).total;
}

size_t smallkv_plan_size(const smallkv_cache* llm, const smallkv_batch* batch,
                         int32_t n_llm_layers) {
  if (!llm || !batch || batch->batch < 1 || batch->max_seq_len < 1 || n_llm_layers < 1) return 0;
  return static_cast<size_t>(skv::plan_bytes(n_llm_layers, batch->batch, llm->num_kv_heads,
                                             batch->max_seq_len));
}

namespace {
// shared argument checks + parameter block of smallkv_plan / smallkv_attend
int fill_attend_params(skv::AttendParams& ap, const smallkv_cache* llm, const smallkv_batch* batch,
                       const int32_t* head_map, int32_t n_llm_layers, int32_t slm_heads_total,
                       const smallkv_budgets* budgets, const int32_t* crit_idx,
                       const int32_t* marg_idx, const float* marg_w, const int32_t* counts) {
  int rc;
  if ((rc = check_cache(llm, true, "llm")) != SMALLKV_OK) return rc;
  if ((rc = check_batch(batch, llm)) != SMALLKV_OK) return rc;
  if ((rc = check_budgets(budgets)) != SMALLKV_OK) return rc;
  if (!head_map || !crit_idx || !marg_idx || !marg_w || !counts)
    return fail(SMALLKV_ERR_NULL, "NULL selection / head-map pointer");
  if (n_llm_layers < 1) return fail(SMALLKV_ERR_SHAPE, "n_llm_layers must be >= 1");
  if (slm_heads_total < 1) return fail(SMALLKV_ERR_SHAPE, "slm_heads_total must be >= 1");
  const int G = llm->num_q_heads / llm->num_kv_heads;
  if (G > 8) return fail(SMALLKV_ERR_SHAPE, "LLM GQA group %d > 8 not supported", G);
  if (static_cast<int64_t>(llm->num_pages) * llm->num_kv_heads * llm->page_size * llm->head_dim >=
      (int64_t(1) << 32))
    return fail(SMALLKV_ERR_SHAPE, "one layer of the LLM pool must have < 2^32 elements");
  ap = skv::AttendParams{};
  ap.k = llm->k;
  ap.v = llm->v;
  ap.block_table = llm->block_table;
  ap.seq_lens = batch->seq_lens;
  ap.head_map = head_map;
  ap.n_recent = budgets->n_recent;
  ap.k_crit = budgets->k_crit;
  ap.k_marg = budgets->k_marg;
  ap.crit_idx = crit_idx;
  ap.marg_idx = marg_idx;
  ap.marg_w = marg_w;
  ap.counts = counts;
  ap.num_pages = llm->num_pages;
  ap.max_blocks = llm->max_blocks;
  ap.page_size = llm->page_size;
  ap.ps_shift = 0;
  while ((1 << ap.ps_shift) < llm->page_size) ++ap.ps_shift;
  ap.heads = llm->num_q_heads;
  ap.kv_heads = llm->num_kv_heads;
  ap.head_dim = llm->head_dim;
  ap.batch = batch->batch;
  ap.n_layers = n_llm_layers;
  ap.row_stride = batch->max_seq_len;
  ap.max_crit = budgets->max_crit;
  ap.max_marg = budgets->max_marg;
  static const int sync_stage_env = [] {
    const char* e = getenv("SMALLKV_ATTEND_SYNC_STAGE");   // diagnostics
    return e ? atoi(e) : 0;
  }();
  ap.sync_stage = sync_stage_env;
  ap.max_chunks = skv::attend_ctas_per_group(batch->batch, llm->num_kv_heads, batch->max_seq_len);
  ap.global_merge = skv::attend_split_in_cluster(batch->batch, llm->num_kv_heads, batch->max_seq_len) ? 0 : 1;
  ap.flat_shares = skv::attend_flat_shares(batch->batch, llm->num_kv_heads, batch->max_seq_len);
  ap.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(llm->head_dim));
  return SMALLKV_OK;
}
}  // namespace

int smallkv_plan(const smallkv_cache* llm, const smallkv_batch* batch, const int32_t* head_map,
                 int32_t n_llm_layers, int32_t slm_heads_total, const smallkv_budgets* budgets,
                 const int32_t* crit_idx, const int32_t* marg_idx, const float* marg_w,
                 const int32_t* counts, void* plan, size_t plan_bytes, void* stream) {
  skv::AttendParams ap;
  int rc = fill_attend_params(ap, llm, batch, head_map, n_llm_layers, slm_heads_total, budgets,
                              crit_idx, marg_idx, marg_w, counts);
  if (rc != SMALLKV_OK) return rc;
  const size_t need = smallkv_plan_size(llm, batch, n_llm_layers);
  if (!plan || plan_bytes < need)
    return fail(SMALLKV_ERR_WORKSPACE, "plan buffer %zu < %zu bytes", plan_bytes, need);
  if (!aligned(plan, 16)) return fail(SMALLKV_ERR_ALIGN, "plan must be 16-byte aligned");
  if (static_cast<int64_t>(n_llm_layers) * batch->batch > 65535)
    return fail(SMALLKV_ERR_SHAPE, "L*B > 65535");   // plan grid.y
  if ((rc = check_device()) != SMALLKV_OK) return rc;
  ap.plan = static_cast<uint8_t*>(plan);
  cudaError_t e = skv::launch_plan(ap, n_llm_layers, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "plan launch");
  return SMALLKV_OK;
}

int smallkv_plan_group(const smallkv_cache* llm, const smallkv_batch* batch, const int32_t* head_map,
                       int32_t n_llm_layers, const smallkv_budgets* budgets, const int32_t* crit_idx,
                       const int32_t* marg_idx, const float* marg_w, const int32_t* counts, void* plan,
                       size_t plan_bytes, void* stream) {
  skv::AttendParams ap;
  int rc = fill_attend_params(ap, llm, batch, head_map, n_llm_layers, 1, budgets, crit_idx, marg_idx,
                              marg_w, counts);
  if (rc != SMALLKV_OK) return rc;
  const size_t need = smallkv_plan_size(llm, batch, n_llm_layers);
  if (!plan || plan_bytes < need)
    return fail(SMALLKV_ERR_WORKSPACE, "plan buffer %zu < %zu bytes", plan_bytes, need);
  if (!aligned(plan, 16)) return fail(SMALLKV_ERR_ALIGN, "plan must be 16-byte aligned");
  if (static_cast<int64_t>(n_llm_layers) * batch->batch > 65535)
    return fail(SMALLKV_ERR_SHAPE, "L*B > 65535");   // plan grid.y
  if ((rc = check_device()) != SMALLKV_OK) return rc;
  ap.plan = static_cast<uint8_t*>(plan);
  ap.group_sel = 1;
  cudaError_t e = skv::launch_plan(ap, n_llm_layers, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "plan launch");
  return SMALLKV_OK;
}

int smallkv_attend(int32_t llm_layer, int32_t cache_layer, const uint16_t* q,
                   const smallkv_cache* llm, const smallkv_batch* batch, const int32_t* head_map,
                   int32_t n_llm_layers, int32_t slm_heads_total, const smallkv_budgets* budgets,
                   const int32_t* crit_idx, const int32_t* marg_idx, const float* marg_w,
                   const int32_t* counts, const void* plan, float* out, int32_t flags, void* ws,
                   size_t ws_bytes, void* stream) {
  skv::AttendParams ap;
  int rc = fill_attend_params(ap, llm, batch, head_map, n_llm_layers, slm_heads_total, budgets,
                              crit_idx, marg_idx, marg_w, counts);
  if (rc != SMALLKV_OK) return rc;
  if (!q || !out) return fail(SMALLKV_ERR_NULL, "smallkv_attend: NULL q/out");
  if (llm_layer < 0 || llm_layer >= n_llm_layers)
    return fail(SMALLKV_ERR_SHAPE, "llm_layer %d outside [0,%d)", llm_layer, n_llm_layers);
  if (cache_layer < 0 || cache_layer >= llm->num_layers)
    return fail(SMALLKV_ERR_SHAPE, "cache_layer %d outside [0,%d)", cache_layer,
                llm->num_layers);
  if (flags & ~(SMALLKV_ATTEND_OVERLAP_PROLOGUE | SMALLKV_ATTEND_GROUP_SELECTION))
    return fail(SMALLKV_ERR_SHAPE, "unknown smallkv_attend flags 0x%x", flags);
  if ((flags & SMALLKV_ATTEND_GROUP_SELECTION) && !aligned(marg_w, 16))
    return fail(SMALLKV_ERR_ALIGN, "group selection: marg_w must be 16-byte aligned");
  if (!aligned(q, 4) || !aligned(out, 16) || (plan && !aligned(plan, 16)))
    return fail(SMALLKV_ERR_ALIGN, "q must be 4-byte, out and plan 16-byte aligned");
  const AttendWs L = attend_ws_layout(llm, batch);
  if (!ws || ws_bytes < L.total)
    return fail(SMALLKV_ERR_WORKSPACE, "attend workspace %zu < %zu bytes", ws_bytes, L.total);
  if ((rc = check_device()) != SMALLKV_OK) return rc;
  ap.q = q;
  ap.out = out;
  ap.layer = llm_layer;
  ap.layer_offset = static_cast<int64_t>(cache_layer) * llm->num_pages * llm->num_kv_heads *
                    llm->page_size * llm->head_dim;
  ap.overlap_prologue = (flags & SMALLKV_ATTEND_OVERLAP_PROLOGUE) ? 1 : 0;
  ap.group_sel = (flags & SMALLKV_ATTEND_GROUP_SELECTION) ? 1 : 0;
  ap.plan = const_cast<uint8_t*>(static_cast<const uint8_t*>(plan));
  ap.tickets = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + L.tickets);
  ap.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + L.partials);
  cudaError_t e = skv::launch_attend(ap, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "attend launch");
  return SMALLKV_OK;
}

namespace {
struct TierState {
  size_t sop, pos_of, entry, prev_t, flags, njob, counters, scratch, total;
};
TierState tier_layout(const smallkv_cache* llm, const smallkv_batch* b, int32_t L, int32_t cap) {
  TierState t;
  const size_t groups = static_cast<size_t>(L) * b->batch * llm->num_kv_heads;
  t.sop = 0;
  t.pos_of = round256(groups * b->max_seq_len * 4);
  t.entry = t.pos_of + round256(groups * cap * 4);
  t.prev_t = t.entry + round256(groups * cap * 4);
  t.flags = t.prev_t + round256(groups * 4);
  t.njob = t.flags + round256(groups * cap);
  t.scratch = t.njob + round256(groups * 4);
  t.counters = t.scratch + round256(groups * cap * 3 * 4);   // last 256 bytes (TieredKV.counters)
  t.total = t.counters + 256;
  return t;
}
// the update's position bitmaps (3 bits per position) live in shared memory
constexpr int32_t kTierMaxSeq = 524288;
constexpr int32_t kTierMaxCap = 1 << 24;
int check_tier(const smallkv_cache* llm, const smallkv_batch* batch, int32_t L, int32_t cap) {
  if (!llm || !batch) return fail(SMALLKV_ERR_NULL, "tier: NULL cache/batch");
  if (L < 1 || cap < 4 || cap % 4 != 0 || cap > kTierMaxCap)
    return fail(SMALLKV_ERR_SHAPE, "tier: layers %d / capacity %d (multiple of 4 in [4,%d])", L, cap,
                kTierMaxCap);
  if (batch->max_seq_len > kTierMaxSeq)
    return fail(SMALLKV_ERR_SHAPE, "tier: max_seq_len %d > %d", batch->max_seq_len, kTierMaxSeq);
  return SMALLKV_OK;
}
}  // namespace

size_t smallkv_tier_state_size(const smallkv_cache* llm, const smallkv_batch* batch,
                               int32_t n_llm_layers, int32_t capacity) {
  if (check_tier(llm, batch, n_llm_layers, capacity) != SMALLKV_OK) return 0;
  return tier_layout(llm, batch, n_llm_layers, capacity).total;
}

int smallkv_tier_init(void* state, size_t state_bytes, const smallkv_cache* llm,
                      const smallkv_batch* batch, int32_t n_llm_layers, int32_t capacity,
                      void* stream) {
  int rc;
  if ((rc = check_tier(llm, batch, n_llm_layers, capacity)) != SMALLKV_OK) return rc;
  const TierState T = tier_layout(llm, batch, n_llm_layers, capacity);
  if (!state || state_bytes < T.total)
    return fail(SMALLKV_ERR_WORKSPACE, "tier state %zu < %zu bytes", state_bytes, T.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* st = static_cast<uint8_t*>(state);
  cudaError_t e = cudaMemsetAsync(st, 0xff, T.flags, s);            // maps = -1
  if (e == cudaSuccess) e = cudaMemsetAsync(st + T.flags, 0, T.total - T.flags, s);
  if (e != cudaSuccess) return cuda_fail(e, "tier init");
  return SMALLKV_OK;
}

int smallkv_tier_update(int32_t layer_begin, int32_t layer_count, const smallkv_cache* host_llm,
                        uint16_t* hot_k, uint16_t* hot_v, int32_t capacity,
                        const smallkv_batch* batch, const int32_t* head_map, int32_t n_llm_layers,
                        int32_t slm_heads_total, const smallkv_budgets* budgets,
                        const int32_t* crit_idx, const int32_t* marg_idx, const float* marg_w,
                        const int32_t* counts, int32_t flags, void* state, size_t state_bytes,
                        void* stream) {
  skv::TierParams tp{};
  int rc = fill_attend_params(tp.a, host_llm, batch, head_map, n_llm_layers, slm_heads_total,
                              budgets, crit_idx, marg_idx, marg_w, counts);
  if (rc != SMALLKV_OK) return rc;
  if ((rc = check_tier(host_llm, batch, n_llm_layers, capacity)) != SMALLKV_OK) return rc;
  if (!hot_k || !hot_v) return fail(SMALLKV_ERR_NULL, "tier: NULL hot pool");
  if (flags & ~SMALLKV_ATTEND_GROUP_SELECTION) return fail(SMALLKV_ERR_SHAPE, "tier: unknown flags");
  if (layer_begin < 0 || layer_count < 1 || layer_begin + layer_count > n_llm_layers ||
      host_llm->num_layers < 1 || layer_count > 65535)
    return fail(SMALLKV_ERR_SHAPE, "tier: layers [%d,%d) vs %d LLM / %d pool layers", layer_begin,
                layer_begin + layer_count, n_llm_layers, host_llm->num_layers);
  const TierState T = tier_layout(host_llm, batch, n_llm_layers, capacity);
  if (!state || state_bytes < T.total)
    return fail(SMALLKV_ERR_WORKSPACE, "tier state %zu < %zu bytes", state_bytes, T.total);
  if (!aligned(hot_k, 16) || !aligned(hot_v, 16)) return fail(SMALLKV_ERR_ALIGN, "hot pools 16-byte aligned");
  if ((rc = check_device()) != SMALLKV_OK) return rc;
  uint8_t* st = static_cast<uint8_t*>(state);
  tp.a.group_sel = (flags & SMALLKV_ATTEND_GROUP_SELECTION) ? 1 : 0;
  tp.host_k = host_llm->k;
  tp.host_v = host_llm->v;
  tp.host_layer_stride = static_cast<int64_t>(host_llm->num_pages) * host_llm->num_kv_heads *
                         host_llm->page_size * host_llm->head_dim;
  tp.host_layers = host_llm->num_layers;
  tp.scratch = reinterpret_cast<int32_t*>(st + T.scratch);
  tp.prev_T = reinterpret_cast<int32_t*>(st + T.prev_t);
  tp.njob = reinterpret_cast<int32_t*>(st + T.njob);
  tp.hot_k = hot_k;
  tp.hot_v = hot_v;
  tp.slot_of_pos = reinterpret_cast<int32_t*>(st + T.sop);
  tp.pos_of_slot = reinterpret_cast<int32_t*>(st + T.pos_of);
  tp.entry_slot = reinterpret_cast<int32_t*>(st + T.entry);
  tp.slot_flags = st + T.flags;
  tp.counters = reinterpret_cast<unsigned long long*>(st + T.counters);
  tp.cap = capacity;
  tp.max_seq_len = batch->max_seq_len;
  tp.layer_begin = layer_begin;
  tp.layer_count = layer_count;
  cudaError_t e = skv::launch_tier_update(tp, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tier_update launch");
  return SMALLKV_OK;
}

int smallkv_plan_tiered(const smallkv_cache* host_llm, int32_t capacity, const void* state,
                        const smallkv_batch* batch, const int32_t* head_map, int32_t n_llm_layers,
                        int32_t slm_heads_total, const smallkv_budgets* budgets,
                        const int32_t* crit_idx, const int32_t* marg_idx, const float* marg_w,
                        const int32_t* counts, int32_t flags, void* plan, size_t plan_bytes,
                        void* stream) {
  skv::AttendParams ap;
  int rc = fill_attend_params(ap, host_llm, batch, head_map, n_llm_layers, slm_heads_total, budgets,
                              crit_idx, marg_idx, marg_w, counts);
  if (rc != SMALLKV_OK) return rc;
  if ((rc = check_tier(host_llm, batch, n_llm_layers, capacity)) != SMALLKV_OK) return rc;
  if (!state) return fail(SMALLKV_ERR_NULL, "smallkv_plan_tiered: NULL state");
  if (flags & ~SMALLKV_ATTEND_GROUP_SELECTION) return fail(SMALLKV_ERR_SHAPE, "unknown flags 0x%x", flags);
  const size_t need = smallkv_plan_size(host_llm, batch, n_llm_layers);
  if (!plan || plan_bytes < need)
    return fail(SMALLKV_ERR_WORKSPACE, "plan buffer %zu < %zu bytes", plan_bytes, need);
  if (!aligned(plan, 16)) return fail(SMALLKV_ERR_ALIGN, "plan must be 16-byte aligned");
  if (static_cast<int64_t>(n_llm_layers) * batch->batch > 65535)
    return fail(SMALLKV_ERR_SHAPE, "L*B > 65535");
  if ((rc = check_device()) != SMALLKV_OK) return rc;
  const TierState T = tier_layout(host_llm, batch, n_llm_layers, capacity);
  ap.plan = static_cast<uint8_t*>(plan);
  ap.group_sel = (flags & SMALLKV_ATTEND_GROUP_SELECTION) ? 1 : 0;
  ap.entry_slot = reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(state) + T.entry);
  ap.hot_cap = capacity;
  cudaError_t e = skv::launch_plan(ap, n_llm_layers, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "plan launch");
  return SMALLKV_OK;
}

int smallkv_attend_tiered(int32_t llm_layer, const uint16_t* q, const smallkv_cache* host_llm,
                          const uint16_t* hot_k, const uint16_t* hot_v, int32_t capacity,
                          const void* state, const smallkv_batch* batch, const int32_t* head_map,
                          int32_t n_llm_layers, int32_t slm_heads_total,
                          const smallkv_budgets* budgets, const int32_t* crit_idx,
                          const int32_t* marg_idx, const float* marg_w, const int32_t* counts,
                          const void* plan, float* out, int32_t flags, void* ws, size_t ws_bytes,
                          void* stream) {
  skv::AttendParams ap;
  int rc = fill_attend_params(ap, host_llm, batch, head_map, n_llm_layers, slm_heads_total, budgets,
                              crit_idx, marg_idx, marg_w, counts);
  if (rc != SMALLKV_OK) return rc;
  if ((rc = check_tier(host_llm, batch, n_llm_layers, capacity)) != SMALLKV_OK) return rc;
  if (!q || !out || !hot_k || !hot_v || !state)
    return fail(SMALLKV_ERR_NULL, "smallkv_attend_tiered: NULL pointer");
  if (llm_layer < 0 || llm_layer >= n_llm_layers)
    return fail(SMALLKV_ERR_SHAPE, "tiered attend: layer %d outside [0,%d)", llm_layer, n_llm_layers);
  if (flags & ~(SMALLKV_ATTEND_OVERLAP_PROLOGUE | SMALLKV_ATTEND_GROUP_SELECTION))
    return fail(SMALLKV_ERR_SHAPE, "unknown smallkv_attend flags 0x%x", flags);
  if (!aligned(q, 4) || !aligned(out, 16) || !aligned(hot_k, 16) || !aligned(hot_v, 16))
    return fail(SMALLKV_ERR_ALIGN, "q 4-byte, out / hot pools 16-byte aligned");
  if (static_cast<int64_t>(batch->batch) * host_llm->num_kv_heads * capacity * host_llm->head_dim >=
      (int64_t(1) << 32))
    return fail(SMALLKV_ERR_SHAPE, "one layer of the hot pool must have < 2^32 elements");
  const AttendWs W = attend_ws_layout(host_llm, batch);
  if (!ws || ws_bytes < W.total)
    return fail(SMALLKV_ERR_WORKSPACE, "attend workspace %zu < %zu bytes", ws_bytes, W.total);
  if ((rc = check_device()) != SMALLKV_OK) return rc;
  const TierState T = tier_layout(host_llm, batch, n_llm_layers, capacity);
  ap.tickets = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + W.tickets);
  ap.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + W.partials);
  ap.q = q;
  ap.out = out;
  ap.layer = llm_layer;
  ap.k = hot_k;
  ap.v = hot_v;
  ap.layer_offset = static_cast<int64_t>(llm_layer) * batch->batch * host_llm->num_kv_heads * capacity *
                    host_llm->head_dim;
  ap.overlap_prologue = (flags & SMALLKV_ATTEND_OVERLAP_PROLOGUE) ? 1 : 0;
  ap.group_sel = (flags & SMALLKV_ATTEND_GROUP_SELECTION) ? 1 : 0;
  if (plan && !aligned(plan, 16)) return fail(SMALLKV_ERR_ALIGN, "plan must be 16-byte aligned");
  ap.plan = const_cast<uint8_t*>(static_cast<const uint8_t*>(plan));
  ap.entry_slot = reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(state) + T.entry);
  ap.hot_cap = capacity;
  cudaError_t e = skv::launch_attend(ap, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "attend launch");
  return SMALLKV_OK;
}

int smallkv_match_window(int32_t n, int32_t w_min, int32_t w_max, int32_t keep_last,
                         int32_t* start, int32_t* len) {
  if (!start || !len) return fail(SMALLKV_ERR_NULL, "smallkv_match_window: NULL output");
  if (w_min < 1 || w_max < w_min || n < 0)
    return fail(SMALLKV_ERR_SHAPE, "window bounds [%d, %d] / n %d invalid", w_min, w_max, n);
  if (n < w_min) {   // P:174 "delays the timing of similarity matching"
    *start = 0;
    *len = 0;
    return SMALLKV_OK;
  }
  *len = n < w_max ? n : w_max;
  *start = keep_last ? n - *len : 0;
  return SMALLKV_OK;
}

int smallkv_prefill_scores(const uint16_t* q, const smallkv_cache* cache, int32_t seq,
                           int32_t start, int32_t len, float* F, void* stream) {
  int rc;
  if ((rc = check_cache(cache, false, "prefill cache")) != SMALLKV_OK) return rc;
  if (!q || !F) return fail(SMALLKV_ERR_NULL, "smallkv_prefill_scores: NULL q/F");
  if (len < 1 || len > 1024) return fail(SMALLKV_ERR_SHAPE, "window length %d not in [1,1024]", len);
  if (start < 0 || seq < 0 ||
      static_cast<int64_t>(start) + len > static_cast<int64_t>(cache->max_blocks) * cache->page_size)
    return fail(SMALLKV_ERR_SHAPE, "window [%d,%d) / seq %d outside the block table", start,
                start + len, seq);
  if (!aligned(q, 4) || !aligned(F, 4)) return fail(SMALLKV_ERR_ALIGN, "q / F must be 4-byte aligned");
  if ((rc = check_device()) != SMALLKV_OK) return rc;
  skv::PrefillParams pp{};
  pp.q = q;
  pp.k = cache->k;
  pp.block_table = cache->block_table;
  pp.F = F;
  pp.layer_stride = static_cast<int64_t>(cache->num_pages) * cache->num_kv_heads * cache->page_size *
                    cache->head_dim;
  pp.seq = seq;
  pp.start = start;
  pp.len = len;
  pp.layers = cache->num_layers;
  pp.heads = cache->num_q_heads;
  pp.kv_heads = cache->num_kv_heads;
  pp.head_dim = cache->head_dim;
  pp.page_size = cache->page_size;
  pp.ps_shift = 0;
  while ((1 << pp.ps_shift) < cache->page_size) ++pp.ps_shift;
  pp.max_blocks = cache->max_blocks;
  pp.scale = 1.0f / std::sqrt(static_cast<float>(cache->head_dim));
  cudaError_t e = skv::launch_prefill_scores(pp, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "prefill_scores launch");
  return SMALLKV_OK;
}

size_t smallkv_match_heads_workspace_size(int32_t n_llm, int32_t n_slm) {
  if (n_llm < 1 || n_slm < 1) return 0;
  return static_cast<size_t>(n_llm + n_slm) * 16 * 4;
}

int smallkv_match_heads(const float* llm_F, int32_t n_llm, const float* slm_F, int32_t n_slm,
                        int32_t w, int32_t k_match, int32_t* head_map, float* jaccard, void* ws,
                        size_t ws_bytes, void* stream) {
  if (!llm_F || !slm_F || !head_map || !jaccard)
    return fail(SMALLKV_ERR_NULL, "smallkv_match_heads: NULL pointer");
  if (n_llm < 1 || n_slm < 1) return fail(SMALLKV_ERR_SHAPE, "n_llm/n_slm must be >= 1");
  if (w < 1 || w > 512) return fail(SMALLKV_ERR_SHAPE, "window %d outside [1,512]", w);
  if (k_match < 1 || k_match > w) return fail(SMALLKV_ERR_SHAPE, "k_match %d outside [1,%d]", k_match, w);
  const size_t need = smallkv_match_heads_workspace_size(n_llm, n_slm);
  if (!ws || ws_bytes < need)
    return fail(SMALLKV_ERR_WORKSPACE, "match workspace %zu < %zu bytes", ws_bytes, need);
  int rc;
  if ((rc = check_device()) != SMALLKV_OK) return rc;
  cudaError_t e = skv::launch_match_heads(llm_F, n_llm, slm_F, n_slm, w, k_match,
                                          static_cast<uint32_t*>(ws), head_map, jaccard,
                                          static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "match_heads launch");
  return SMALLKV_OK;
}

int smallkv_workspace_init(void* ws, size_t bytes, void* stream) {
  if (!ws) return fail(SMALLKV_ERR_NULL, "workspace NULL");
  cudaError_t e = cudaMemsetAsync(ws, 0, bytes, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  return SMALLKV_OK;
}

}  // extern "C"
