// kernels.h — internal launch interfaces of libsmallkv (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace skv {

// ---------------------------------------------------------------- K1 slm_score
struct SlmScoreParams {
  const uint16_t* q;          // [l][B][H_s][d]
  const int32_t* block_table; // [B][max_blocks]
  const int32_t* seq_lens;    // [B]
  const uint8_t* row_needed;  // [l*H_s]
  float* logits;              // [l*H_s][B][row_stride]
  int64_t num_pages;
  int32_t max_blocks, page_size, layers, heads, kv_heads, head_dim, batch;
  int32_t row_stride;         // max_seq_len
  int32_t chunk_tokens;       // tokens per CTA (multiple of 64)
  int32_t box_rows;           // TMA box rows = min(page_size, 64)
  uint32_t swz;               // 7 = 128B swizzle, 0 = none
  float scale;                // 1/sqrt(d)
  int32_t layer_begin, layer_end;   // SLM layers scored by this launch
  const int32_t* n_recent;    // [B] (ranked range for the chunk statistics)
  float4* stats;              // [l*H_s][B][n_chunks] (max, Σexp, min, max) per row chunk
  int32_t n_chunks;           // chunks of chunk_tokens per row
};
cudaError_t launch_slm_score(const SlmScoreParams& p, const CUtensorMap& map, int max_seq_len,
                             cudaStream_t s);

// row flags + compact list of the head map's image (+ zeroes the long split's to-do count)
cudaError_t launch_row_flags(const int32_t* head_map, int32_t n_llm_heads, int32_t n_slm_heads,
                             int32_t heads_per_layer, uint8_t* row_needed, int32_t* rows,
                             int32_t* n_rows, int32_t* layer_off, int32_t* todo_count,
                             cudaStream_t s);

// ---------------------------------------------------------------- K2 select
struct SelectParams {
  const float* logits;        // [l*H_s][B][row_stride]
  const int32_t* seq_lens;
  const int32_t* rows;        // compact image(f), ascending
  const int32_t* layer_off;   // [l+1] rows of SLM layers < l start at layer_off[l]
  int32_t layer_begin, layer_end;   // SLM layers whose rows this launch selects
  const int32_t *k_crit, *n_recent, *k_marg;
  float* lse;                 // [l*H_s][B][2]
  int32_t* crit_idx;          // [l*H_s][B][max_crit]
  int32_t* marg_idx;          // [l*H_s][B][max_marg]
  float* marg_w;
  int32_t* counts;            // [l*H_s][B][2]
  const float4* stats;        // K1's per-chunk row statistics
  float* acc;                 // f1 running column sums [l*H_s][B][row_stride] or nullptr
  int32_t n_chunks, chunk_tokens;
  int32_t batch, row_stride, max_crit, max_marg;
  int32_t log_bins;           // histogram on log(score) (variant f2's group scores)
  int32_t* todo;              // rows (row * B + b) the cluster / register splits hand to the long split
  int32_t* todo_count;        // [count, consumer ticket]: zeroed by row_flags, emptied by each to-do launch
};
cudaError_t launch_select(const SelectParams& p, int32_t max_rows, int32_t max_seq_len,
                          bool overlap_previous, cudaStream_t s);
// long rows with few (row, sequence) pairs: one thread-block cluster of
// `cluster` CTAs (2, 4, 8 or 16) per pair (select_cluster.cu), then the rows it
// handed over (usually none)
constexpr int32_t kClusterSplitMinLen = 16384;
// the long split over the to-do list the cluster / register splits filled (a
// fixed small grid; returns at once when the list is empty), then empties it
cudaError_t launch_select_todo(const SelectParams& p, cudaStream_t s);
cudaError_t launch_select_cluster(const SelectParams& p, int32_t max_rows, int32_t cluster,
                                  cudaStream_t s);

// ---------------------------------------------------------------- variant f2 (R16)
// Group score rows F_g = Σ_{h in group} a'_{f(l,h)} (+ their ranked-range
// statistics in K1's float4 format, one chunk per row) and, after the split,
// the per-head marginal weights of the shared marginal set.
struct GroupParams {
  const float* logits;        // SLM logits [l*H_s][B][row_stride] (K1)
  const float4* stats;        // K1's per-chunk row statistics
  int32_t n_chunks, chunk_tokens;
  const int32_t* head_map;    // [L*H]
  const int32_t* seq_lens;
  const int32_t* n_recent;
  float* slm_lse;             // [l*H_s][B][2] (m', lse') of the group's rows
  float* score;               // [L*H_kv][B][row_stride]
  float4* gstats;             // [L*H_kv][B] (max, 1, min_ranked, max_ranked)
  int32_t* rows;              // identity list [L*H_kv] for the split
  int32_t* layer_off;         // {0, L*H_kv}
  const int32_t* counts;      // split outputs (group rows)
  const int32_t* marg_idx;
  float* marg_w8;             // [L*H_kv][B][max_marg][8]
  int32_t L, H, H_kv, batch, row_stride, max_marg;
};
cudaError_t launch_group_score(const GroupParams& p, cudaStream_t s);
cudaError_t launch_group_weights(const GroupParams& p, cudaStream_t s);

// ---------------------------------------------------------------- K3 gather_attend (+K4)
struct AttendParams {
  const uint16_t* q;          // [B][H][d]
  const uint16_t* k;          // pool base
  const uint16_t* v;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const int32_t* head_map;    // [L*H]
  const int32_t* n_recent;
  const int32_t* k_crit;
  const int32_t* k_marg;
  const int32_t* crit_idx;
  const int32_t* marg_idx;
  const float* marg_w;        // a' at marg_idx
  const int32_t* counts;
  float* out;                 // [B][H][d]
  int64_t num_pages;
  int64_t layer_offset;       // cache_layer * num_pages * H_kv * page_size * d (elements)
  int32_t max_blocks, page_size, heads, kv_heads, head_dim, batch, layer;
  int32_t ps_shift;           // log2(page_size)
  int32_t row_stride, max_crit, max_marg;
  int32_t max_chunks;         // CTAs (= cluster size) per (sequence, kv-group)
  float scale_log2;           // log2(e)/sqrt(d)
  int32_t overlap_prologue;   // SMALLKV_ATTEND_OVERLAP_PROLOGUE
  int32_t group_sel;          // variant f2: selection rows are (layer, kv-group); marg_w is
                              // [L*H_kv][B][max_marg][8] per-head weights
  uint8_t* plan;              // gather plan (smallkv_plan) or nullptr
  int32_t n_layers;           // LLM layers the plan holds (next-layer L2 prefetch)
  // variant f4 (host-tiered pool): rows come from a per-(layer, b, kv-group) hot pool
  // [B][H_kv][hot_cap][d] per layer slot; entry e of the group's list lives in slot
  // entry_slot[((layer*B + b)*H_kv + g)*hot_cap + e]
  const int32_t* entry_slot;  // nullptr: the paged pool
  int32_t hot_cap;
  int32_t sync_stage;         // diagnostics: stage batch x+1 synchronously at the start of batch x
  // split without a cluster (max_chunks > the clusters the GPU co-schedules):
  // every CTA writes its partial state, the last one of the group merges
  int32_t global_merge;
  // stream-K split (> 0): S CTAs in a 1-D grid over all groups' bytes, CTA s
  // owning [s*Gt, (s+1)*Gt) of the groups laid end to end at S units each;
  // max_chunks is then the record slots per group and the merge is global
  int32_t flat_shares;
  float* partials;            // [B][H_kv][max_chunks][kAttendPartFloats]
  int32_t* tickets;           // [B][H_kv], zero between launches
};
// floats of one CTA's partial state: (m, l) of 8 heads, O_c and O_m of 8 heads x 128
constexpr int kAttendPartFloats = 16 + 16 * 128;

// variant f4: keep each group's needed rows in an HBM hot pool, fetching only
// rows that were not resident at the previous step from the host-resident pool.
struct TierParams {
  AttendParams a;             // layout of the group lists (selection, budgets, head map)
  const uint16_t* host_k;     // paged pool in host memory (UVA pointers), layer l = LLM layer l
  const uint16_t* host_v;
  uint16_t* hot_k;            // [L][B][H_kv][cap][d]
  uint16_t* hot_v;
  int64_t host_layer_stride;  // elements
  int32_t host_layers;        // host pool layer slots: LLM layer l reads slot l mod host_layers
  int32_t* slot_of_pos;       // [L][B][H_kv][max_seq_len]  (-1: not resident)
  int32_t* pos_of_slot;       // [L][B][H_kv][cap]          (-1: free)
  uint8_t* slot_flags;        // [L][B][H_kv][cap]          bit0 V resident, bit1 K resident
  int32_t* entry_slot;        // [L][B][H_kv][cap]
  int32_t* prev_T;            // [L][B][H_kv] list length of the last refresh (-1: none)
  int32_t* njob;              // [L][B][H_kv] fetch jobs the update left for the copy launch
  unsigned long long* counters;   // [0] rows fetched (K or V), [1] capacity overflows
  int32_t* scratch;           // [L][B][H_kv][3][cap] per-entry work lists
  int32_t cap, max_seq_len, layer_begin, layer_count;
};
cudaError_t launch_tier_update(const TierParams& p, cudaStream_t s);
cudaError_t launch_attend(const AttendParams& p, cudaStream_t s);
cudaError_t launch_plan(const AttendParams& p, int32_t n_layers, cudaStream_t s);
int64_t plan_bytes(int32_t n_layers, int32_t batch, int32_t kv_heads, int32_t max_seq_len);
int32_t attend_ctas_per_group(int32_t batch, int32_t kv_heads, int32_t max_seq_len);
bool attend_split_in_cluster(int32_t batch, int32_t kv_heads, int32_t max_seq_len);   // else the global merge
int32_t attend_flat_shares(int32_t batch, int32_t kv_heads, int32_t max_seq_len);      // stream-K CTAs, 0: off

// ---------------------------------------------------------------- variant f3 prefill scores (R17)
struct PrefillParams {
  const uint16_t* q;          // [L][len][H][d] bf16 (the window's queries)
  const uint16_t* k;          // paged pool [layer][page][H_kv][page_size][d]
  const int32_t* block_table; // [B][max_blocks]
  float* F;                   // [L*H][len]
  int64_t layer_stride;       // elements between layers of the pool
  int32_t seq, start, len, layers, heads, kv_heads, head_dim, page_size, ps_shift, max_blocks;
  float scale;                // 1/sqrt(d)
};
cudaError_t launch_prefill_scores(const PrefillParams& p, cudaStream_t s);

// ---------------------------------------------------------------- K0 match_heads
cudaError_t launch_match_heads(const float* llm_F, int32_t n_llm, const float* slm_F,
                               int32_t n_slm, int32_t w, int32_t k, uint32_t* bits_ws,
                               int32_t* head_map, float* jaccard, cudaStream_t s);

}  // namespace skv
