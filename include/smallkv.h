/*
 * smallkv.h — C ABI of libsmallkv.so, the sm_100a (B200) decode hot path of
 * SmallKV (arXiv 2508.02751, "small model assisted compensation of KV cache
 * compression").
 *
 * Citations: "P:n" = PAPER.md line n (section / equation named beside it),
 * "S:n" = SPEC.md line n.  The readings of ambiguous passages are listed in
 * DESIGN.md §3 ("readings") and referred to here as R1..R15.
 *
 * The three hot-path calls follow the decode branch of Algorithm 1
 * (P:196-209):
 *   smallkv_select  — Alg. 1 l.7 + l.9: score the SLM's current query row over
 *                     its full, never-compressed cache C^s_all and split
 *                     every row f(i) the head map references into critical /
 *                     marginal / evicted sets (Eq. 4, Eq. 6).
 *   smallkv_attend  — Alg. 1 l.12-14: per LLM layer, O = O_c + O_m with O_c the
 *                     exact softmax over the critical ∪ recent K/V (P:203,
 *                     App. D) and O_m = Σ_{k∈marginal} A'_{f(i)}[k]·V[k]
 *                     (Eq. 6 second branch P:147, App. D).
 *   smallkv_match_heads — prefill-time Eq. 2 (TopK Jaccard) and
 *                     Eq. 3 (f(i) = argmax_j S).
 *
 * Conventions (all calls):
 *  - Every pointer marked "device" is caller-owned device memory (e.g. torch
 *    tensors); the library never allocates, never synchronises the device and
 *    keeps no state between calls.  All device work is enqueued on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream), so the
 *    calls are CUDA-graph capturable.
 *  - bf16 arrays are passed as `const uint16_t*` (raw bfloat16 bits).
 *  - Return value: SMALLKV_OK (0) or an error code; on error nothing has been
 *    enqueued (host-side validation happens before any launch) except for
 *    SMALLKV_ERR_CUDA, which reports a launch failure.  smallkv_last_error()
 *    returns a thread-local message describing the last non-OK return.
 *  - Data-dependent conditions are NOT errors: budgets larger than a sequence
 *    are clamped on the device (R5: R' = min(R,n), K' = min(K,n-R'),
 *    M' = min(M,n-R'-K')); NaN/Inf inputs give unspecified results.
 *  - Results are deterministic: bit-identical across runs, page-table
 *    permutations and batch partitions.
 *  - Only sm_100 devices are accepted (SMALLKV_ERR_DEVICE otherwise).
 */
#ifndef SMALLKV_H_
#define SMALLKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum smallkv_status {
  SMALLKV_OK = 0,
  SMALLKV_ERR_NULL = 1,        /* a required pointer is NULL                    */
  SMALLKV_ERR_SHAPE = 2,       /* unsupported or inconsistent dimensions        */
  SMALLKV_ERR_ALIGN = 3,       /* a device pointer is not 16-byte aligned       */
  SMALLKV_ERR_WORKSPACE = 4,   /* workspace NULL or smaller than *_workspace_size */
  SMALLKV_ERR_DEVICE = 5,      /* current device is not sm_100                  */
  SMALLKV_ERR_CUDA = 6,        /* a CUDA API call or kernel launch failed       */
  SMALLKV_ERR_UNSUPPORTED = 7  /* valid request for a variant not built yet     */
};

/* Thread-local, NUL-terminated description of the last non-OK return. */
const char* smallkv_last_error(void);
/* Library version string, e.g. "smallkv-b200 0.1". */
const char* smallkv_version(void);

/*
 * One model's paged KV cache, all layers ("V_i ∈ R^{n×d}").
 * Layout of k and v (bf16, head-major within a page, "HND"):
 *     [num_layers][num_pages][num_kv_heads][page_size][head_dim]
 * so the page_size rows of one kv-head inside one page are contiguous.
 * Token `pos` of sequence b lives in physical page block_table[b*max_blocks +
 * pos/page_size] at row pos%page_size.  Physical pages are shared by all
 * layers (one block table per model).
 *   k, v        device; v may be NULL for the SLM (its V is never read, R11).
 *   block_table device int32 [B][max_blocks].
 *   num_pages   physical pages per layer (for index validation / TMA maps).
 *   page_size   power of two, 1..256.
 *   head_dim    64 or 128.  num_q_heads % num_kv_heads == 0.
 */
typedef struct smallkv_cache {
  const uint16_t* k;
  const uint16_t* v;
  const int32_t* block_table;
  int64_t num_pages;
  int32_t max_blocks;
  int32_t page_size;
  int32_t num_layers;
  int32_t num_q_heads;
  int32_t num_kv_heads;
  int32_t head_dim;
} smallkv_cache;

/*
 * The decode batch.  seq_lens[b] = n_b counts cached tokens INCLUDING the
 * current one, whose K/V the caller has already appended to both caches (R12).
 *   seq_lens    device int32 [B], 1 <= n_b <= max_seq_len.
 *   max_seq_len host; row stride of slm_logits and a sizing bound.
 */
typedef struct smallkv_batch {
  const int32_t* seq_lens;
  int32_t batch;
  int32_t max_seq_len;
} smallkv_batch;

/*
 * Per-sequence token budgets (critical : recent : marginal = 2:1:2;
 * Eq. 6's K and P-K).  Device int32 [B] each; clamped on the device
 * (R5).  max_crit / max_marg (host) are the row strides of the selection
 * lists and must bound every k_crit[b] / k_marg[b].
 */
typedef struct smallkv_budgets {
  const int32_t* k_crit;
  const int32_t* n_recent;
  const int32_t* k_marg;
  int32_t max_crit;
  int32_t max_marg;
} smallkv_budgets;

/*
 * Host helper: token counts from a KV budget fraction tau (R6):
 *   K = floor(tau*n/2), R = floor(tau*n/4), M = floor(tau*n/2)
 * i.e. 2:1:2 with marginal tokens at half cost (V only), so that
 * K + R + M/2 <= tau*n.  tau in (0,1]; n >= 0.  Returns SMALLKV_ERR_SHAPE for
 * tau outside (0,1] or n < 0, SMALLKV_ERR_NULL for NULL outputs.
 */
int smallkv_budget_from_tau(double tau, int32_t n, int32_t* k_crit,
                            int32_t* n_recent, int32_t* k_marg);

/*
 * Head map convention (Eq. 3; R9): head_map is device int32
 * [L * H], entry (layer*H + h) = flat SLM head j = slm_layer*H_s + slm_head,
 * 0 <= j < l*H_s.  Maps may cross layers (R9).
 */

/* Bytes of workspace smallkv_select needs (0 on invalid arguments). */
size_t smallkv_select_workspace_size(const smallkv_cache* slm,
                                     const smallkv_batch* batch,
                                     int32_t n_llm_heads);

/*
 * smallkv_select — SLM score rows + three-way split (Alg. 1 l.7, l.9).
 *
 * For every flat SLM head j in image(head_map) and every sequence b
 * ("performs eviction for the i cache of LLM based on the f(i)-th (full)
 * cache of SLM"; Eq. 6; R1 current-row score, R4 marginal band,
 * R3 tie-break):
 *   s'_v  = q'_j · K'_{kv(j)}[v] / sqrt(d_s),   v in [0, n)         (fp32)
 *   m'    = max_v s'_v,  lse' = m' + ln Σ_v exp(s'_v - m')
 *   a'_v  = exp(s'_v - lse')        (the SLM attention row A'_{f(i)})
 *   recent R' = [n-R', n); positions [0, n-R') ranked by (s' desc, v asc):
 *   critical = first K', marginal = next M', evicted = the rest.
 * Inputs:
 *   slm_q       device bf16 [l][B][H_s][d_s] (post-RoPE current-token queries).
 *   slm         SLM cache (v unused).
 *   head_map    device int32 [n_llm_heads] (see above).
 * Outputs (indexed by flat SLM head j; rows not in image(f) untouched):
 *   slm_logits  device fp32 [l*H_s][B][max_seq_len]   s'_v for v < n.
 *   slm_lse     device fp32 [l*H_s][B][2]            (m', lse').
 *   crit_idx    device int32 [l*H_s][B][max_crit]    ascending positions.
 *   marg_idx    device int32 [l*H_s][B][max_marg]    ascending positions.
 *   marg_w      device fp32 [l*H_s][B][max_marg]     a'_v at marg_idx.
 *   counts      device int32 [l*H_s][B][2]           (K', M') after clamping.
 *   acc         NULL: rank by the current row (R1).  Otherwise variant f1
 *               (Eq. 1 running column sums): device fp32
 *               [l*H_s][B][max_seq_len], read and updated in place for the rows
 *               in image(f): acc[v] += a'_v (v < n), and positions are ranked by
 *               the updated acc (desc, index asc).  The caller zero-fills it once
 *               per sequence; marg_w stays the current a' (Eq. 6).
 *   ws          device workspace, >= smallkv_select_workspace_size bytes.
 *   aux_stream  NULL, or a second stream: the SLM layers are then scored in
 *               chunks on `stream` while the split of each finished chunk runs
 *               on aux_stream (Alg. 1 l.8-9 "in parallel"); `stream`
 *               waits for the last split before returning work to the caller.
 *               A chunk holds as many SLM layers as keep its score rows
 *               (H_s * B * max_seq_len * 4 bytes per layer) within 48 MB, at
 *               least one, so the split re-reads them from L2 (long contexts).
 *               Both streams must be on the current device; capturable.
 * Launches (all on `stream` / aux_stream, nothing host-synchronous): the
 * image flags, then per SLM-layer chunk the scoring (K1) and the split (K2).
 * Rows of up to 12288 tokens (without `acc`) take the register split, long
 * rows at small batch the cluster split; both hand the rare rows they do not
 * finish (all scores equal, a boundary bin too full for their pair lists) to a
 * to-do list in `ws` that a small second launch completes right after, with
 * the exact radix-select fallback.  The result does not depend on which split
 * ran.
 * Errors: NULL pointers, H_s % H_kv_s != 0, head_dim not in {64,128},
 * page_size not a power of two in [1,256], misaligned pointers, small ws,
 * non-sm_100 device.
 */
int smallkv_select(const uint16_t* slm_q, const smallkv_cache* slm,
                   const smallkv_batch* batch, const int32_t* head_map,
                   int32_t n_llm_heads, const smallkv_budgets* budgets,
                   float* slm_logits, float* slm_lse, int32_t* crit_idx,
                   int32_t* marg_idx, float* marg_w, int32_t* counts,
                   float* acc, void* ws, size_t ws_bytes, void* stream,
                   void* aux_stream);

/*
 * Variant f2 (R16): per-LLM-KV-head shared selection.
 * For LLM layer l, kv group g (q heads g*G .. g*G+G-1, G = H/H_kv) and
 * sequence b, the group score sums the SLM proxy rows of the group's heads
 * (App. A counts budgets per KV head):
 *   F_g[v] = Σ_{h in group g} a'_{f(l,h)}[v],   a' as in smallkv_select
 * and ONE three-way split of F_g (same clamps, recent window and
 * lower-index tie-break as smallkv_select) is shared by all heads of the
 * group.  The marginal weight of head h at a shared marginal position k stays
 * its own row a'_{f(l,h)}[k] (Eq. 6 second branch).
 * Inputs: as smallkv_select; n_llm_layers = L, llm_q_heads = H,
 *   llm_kv_heads = H_kv (head_map has L*H entries; H % H_kv == 0, G <= 8).
 * Outputs, indexed by group row r = l*H_kv + g:
 *   slm_logits, slm_lse  as smallkv_select (rows in image(f)).
 *   group_score device fp32 [L*H_kv][B][max_seq_len]   F_g[v] for v < n (fp32
 *               sum over the group's heads in head order).
 *   crit_idx    device int32 [L*H_kv][B][max_crit]     ascending positions.
 *   marg_idx    device int32 [L*H_kv][B][max_marg]     ascending positions.
 *   marg_w      device fp32 [L*H_kv][B][max_marg][8]   per-head a'_{f(l,h)}
 *               at marg_idx, head slot h - g*G (slots >= G are 0).
 *   counts      device int32 [L*H_kv][B][2]            (K', M') after clamping.
 *   ws          >= smallkv_select_group_workspace_size bytes.
 * Errors: as smallkv_select, plus H % H_kv != 0 or G > 8 (SMALLKV_ERR_SHAPE).
 * Consumed by smallkv_plan_group / smallkv_attend(... SMALLKV_ATTEND_GROUP_SELECTION).
 */
size_t smallkv_select_group_workspace_size(const smallkv_cache* slm,
                                           const smallkv_batch* batch,
                                           const smallkv_budgets* budgets,
                                           int32_t n_llm_layers,
                                           int32_t llm_kv_heads);
int smallkv_select_group(const uint16_t* slm_q, const smallkv_cache* slm,
                         const smallkv_batch* batch, const int32_t* head_map,
                         int32_t n_llm_layers, int32_t llm_q_heads,
                         int32_t llm_kv_heads, const smallkv_budgets* budgets,
                         float* slm_logits, float* slm_lse, float* group_score,
                         int32_t* crit_idx, int32_t* marg_idx, float* marg_w,
                         int32_t* counts, void* ws, size_t ws_bytes,
                         void* stream);

/* Bytes of the gather plan of n_llm_layers layers (0 on invalid arguments). */
size_t smallkv_plan_size(const smallkv_cache* llm, const smallkv_batch* batch,
                         int32_t n_llm_layers);

/*
 * smallkv_plan — optional, once per decode step after smallkv_select: stages
 * for every LLM layer, sequence and kv-group the first gather batch of
 * smallkv_attend (per entry: row offset in the layer's pool, head mask,
 * marginal weight) so each attend launch starts streaming after one read.
 * Same arguments as smallkv_attend's selection inputs; plan is device memory
 * of >= smallkv_plan_size bytes (16-byte aligned), fully rewritten.  The plan
 * depends on the page tables, head map and selection of this step only.
 * Errors: as smallkv_attend.
 */
int smallkv_plan(const smallkv_cache* llm, const smallkv_batch* batch,
                 const int32_t* head_map, int32_t n_llm_layers,
                 int32_t slm_heads_total, const smallkv_budgets* budgets,
                 const int32_t* crit_idx, const int32_t* marg_idx,
                 const float* marg_w, const int32_t* counts, void* plan,
                 size_t plan_bytes, void* stream);

/*
 * smallkv_plan_group — smallkv_plan for variant f2: the selection inputs are
 * smallkv_select_group's group-indexed outputs (crit_idx / marg_idx / marg_w
 * / counts as documented there); same plan size and buffer rules.  The plan
 * must be consumed by smallkv_attend with SMALLKV_ATTEND_GROUP_SELECTION.
 */
int smallkv_plan_group(const smallkv_cache* llm, const smallkv_batch* batch,
                       const int32_t* head_map, int32_t n_llm_layers,
                       const smallkv_budgets* budgets, const int32_t* crit_idx,
                       const int32_t* marg_idx, const float* marg_w,
                       const int32_t* counts, void* plan, size_t plan_bytes,
                       void* stream);

/* Bytes of workspace smallkv_attend needs (0 on invalid arguments). */
size_t smallkv_attend_workspace_size(const smallkv_cache* llm,
                                     const smallkv_batch* batch);

/*
 * smallkv_attend — compensated decode attention for one LLM layer
 * (Alg. 1 l.11-14; App. D SmallKV_attention_forward P:788-793).
 *
 * For every sequence b and LLM query head h of layer `llm_layer`, with
 * j = head_map[llm_layer*H + h], kv-head g = h / (H/H_kv), the lists written
 * by smallkv_select for (j, b) and R' from n_recent (R2, R10):
 *   l_k = q_h · K_g[k] / sqrt(d)              for k in C ∪ R'
 *   w_k = exp(l_k - max) / Σ_{C∪R'} exp(.)     (O_c = 0 if C ∪ R' is empty)
 *   O_c = Σ w_k V_g[k];  O_m = Σ_{k∈M} a'_j[k] V_g[k];  out = O_c + O_m
 * with a'_j[k] = marg_w[j][b][i] for k = marg_idx[j][b][i] (Eq. 6).
 * Inputs:
 *   llm_layer   index into head_map's layer dimension (0 <= llm_layer < L).
 *   cache_layer layer slot of `llm`'s pools holding this layer's K/V
 *               (lets a caller rotate a resident subset of layers).
 *   q           device bf16 [B][H][d].
 *   n_llm_layers L (head_map has L*H entries).
 *   crit_idx, marg_idx, marg_w, counts: smallkv_select outputs (same batch
 *               and budgets; slm_heads_total = l*H_s rows).
 *   plan        NULL, or the smallkv_plan buffer of this step (then the
 *               kernel skips its own two rounds of list / page-table loads).
 *   out         device fp32 [B][H][d].
 *   flags       0 or a combination of SMALLKV_ATTEND_OVERLAP_PROLOGUE and
 *               SMALLKV_ATTEND_GROUP_SELECTION.  OVERLAP_PROLOGUE: the kernel is always
 *               launched with programmatic dependent launch: it reads q and
 *               writes out only after the previous kernel on `stream` has
 *               completed.  With the flag it may also start BEFORE that, and
 *               then reads the selection outputs, head_map, seq_lens,
 *               budgets, block table and K/V pools during the previous
 *               kernel's tail — so the caller guarantees those (and `plan`)
 *               were complete before the previous kernel started (true when
 *               another kernel, e.g. a previous smallkv_attend, separates this
 *               call from smallkv_select / smallkv_plan and from the K/V
 *               append).  The first attend after smallkv_select or
 *               smallkv_plan must therefore be called without the flag.
 *   ws          device workspace, >= smallkv_attend_workspace_size bytes,
 *               zero-filled once by the caller (smallkv_workspace_init) and
 *               left zeroed by every call: when a group's list is split over
 *               more CTAs than the GPU co-schedules as one thread-block
 *               cluster, or under the stream-K split (long lists over
 *               >= 32 groups that do not divide the SMs: #SMs CTAs take
 *               equal byte shares of all groups end to end), the CTAs merge
 *               their partial states through it (a per-group arrival counter
 *               + partial rows, merged in rank / share order:
 *               deterministic); otherwise it is unused.
 *               SMALLKV_ATTEND_GROUP_SELECTION (variant f2, R16): the
 *               selection inputs are smallkv_select_group's group-indexed
 *               outputs; every head of group g attends over the group's
 *               shared C ∪ R' and weights the shared marginal set with its
 *               own marg_w slot; slm_heads_total is ignored.  The plan (if
 *               any) must come from smallkv_plan_group.
 * Errors: as smallkv_select, plus H/H_kv > 8, unknown flags (SMALLKV_ERR_SHAPE).
 */
#define SMALLKV_ATTEND_OVERLAP_PROLOGUE 1
#define SMALLKV_ATTEND_GROUP_SELECTION 2
int smallkv_attend(int32_t llm_layer, int32_t cache_layer, const uint16_t* q,
                   const smallkv_cache* llm, const smallkv_batch* batch,
                   const int32_t* head_map, int32_t n_llm_layers,
                   int32_t slm_heads_total, const smallkv_budgets* budgets,
                   const int32_t* crit_idx, const int32_t* marg_idx,
                   const float* marg_w, const int32_t* counts, const void* plan,
                   float* out, int32_t flags, void* ws, size_t ws_bytes,
                   void* stream);

/*
 * Variant f4 (R18) — host-tiered KV (the paper's
 * memory-saving mode: the KV cache migrates between GPU HBM
 * and CPU memory, the change being moved each step).  The full paged LLM pool
 * lives in HOST memory (pinned, UVA-addressable: `host_llm.k/v`); each
 * (layer, sequence, kv-group) keeps the rows its current list needs in an HBM
 * hot pool of `capacity` slots:
 *   host_llm       LLM layer l reads layer slot l mod host_llm.num_layers of its
 *                  pools (num_layers = L: every layer; fewer: a rotated subset).
 *   hot_k / hot_v  device bf16 [L][B][H_kv][capacity][d] (caller-owned).
 *   state          device bytes >= smallkv_tier_state_size(): per group the
 *                  position->slot and slot->position maps, residency flags, the
 *                  entries' slots, and two uint64 counters (rows fetched over
 *                  the host link; capacity overflows).  Initialise once with
 *                  smallkv_tier_init.
 * smallkv_tier_update (LLM layers [layer_begin, layer_begin+layer_count) in two
 * launches — the lists' bookkeeping, then the host-link copies — e.g. all of
 * them right after smallkv_select / _select_group, so the refresh of every
 * layer runs ahead of the attends; a group whose list is unchanged
 * since its last refresh only compares it):
 * frees the slots of positions the group's list no longer holds, gives every
 * newly listed position a free slot, and copies from host memory only what is
 * missing — V for every new position, K only where a critical or recent entry
 * needs it (marginal rows stay V-only, R11); rows resident at the previous
 * step are not moved.  capacity must be a multiple of 4 and >= the list size
 * R' + (#distinct rows)·(K' + M') of every group, else the group is skipped
 * and counted as an overflow: its hot pool is left unchanged and
 * smallkv_plan_tiered / smallkv_attend_tiered read nothing for it and write
 * NaN to its heads' outputs.
 * smallkv_plan_tiered: smallkv_plan over the hot-pool slots (after
 * smallkv_tier_update; plan size as smallkv_plan_size).
 * smallkv_attend_tiered: smallkv_attend reading the hot pool (plan: NULL or
 * smallkv_plan_tiered's).
 * flags: SMALLKV_ATTEND_GROUP_SELECTION for variant f2 selections.
 * Errors: as smallkv_attend, plus max_seq_len > 524288 or a capacity that is
 * not a multiple of 4 in [4, 2^24] (SMALLKV_ERR_SHAPE), small state
 * (SMALLKV_ERR_WORKSPACE).
 */
size_t smallkv_tier_state_size(const smallkv_cache* llm, const smallkv_batch* batch,
                               int32_t n_llm_layers, int32_t capacity);
int smallkv_tier_init(void* state, size_t state_bytes, const smallkv_cache* llm,
                      const smallkv_batch* batch, int32_t n_llm_layers, int32_t capacity,
                      void* stream);
int smallkv_tier_update(int32_t layer_begin, int32_t layer_count, const smallkv_cache* host_llm,
                        uint16_t* hot_k, uint16_t* hot_v, int32_t capacity,
                        const smallkv_batch* batch, const int32_t* head_map,
                        int32_t n_llm_layers, int32_t slm_heads_total,
                        const smallkv_budgets* budgets, const int32_t* crit_idx,
                        const int32_t* marg_idx, const float* marg_w, const int32_t* counts,
                        int32_t flags, void* state, size_t state_bytes, void* stream);
int smallkv_plan_tiered(const smallkv_cache* host_llm, int32_t capacity, const void* state,
                        const smallkv_batch* batch, const int32_t* head_map,
                        int32_t n_llm_layers, int32_t slm_heads_total,
                        const smallkv_budgets* budgets, const int32_t* crit_idx,
                        const int32_t* marg_idx, const float* marg_w, const int32_t* counts,
                        int32_t flags, void* plan, size_t plan_bytes, void* stream);
int smallkv_attend_tiered(int32_t llm_layer, const uint16_t* q,
                          const smallkv_cache* host_llm, const uint16_t* hot_k,
                          const uint16_t* hot_v, int32_t capacity, const void* state,
                          const smallkv_batch* batch, const int32_t* head_map,
                          int32_t n_llm_layers, int32_t slm_heads_total,
                          const smallkv_budgets* budgets, const int32_t* crit_idx,
                          const int32_t* marg_idx, const float* marg_w,
                          const int32_t* counts, const void* plan, float* out, int32_t flags,
                          void* ws, size_t ws_bytes, void* stream);

/*
 * Variant f3 (R17) — the prefill side of matching.
 *
 * smallkv_match_window — host helper, the matching window of a prompt of n
 * tokens ("range of 100 to 200 ... delays ... truncate"):
 *   n < w_min  => *len = 0 (DEFER matching and eviction), *start = 0;
 *   otherwise     *len = min(n, w_max), *start = keep_last ? n - *len : 0
 *   (keep_last = 1: the most recent tokens).
 * Errors: NULL outputs (SMALLKV_ERR_NULL); w_min < 1, w_max < w_min or n < 0
 * (SMALLKV_ERR_SHAPE).
 */
int smallkv_match_window(int32_t n, int32_t w_min, int32_t w_max, int32_t keep_last,
                         int32_t* start, int32_t* len);

/*
 * smallkv_prefill_scores — the F vectors of Eq. 2 for one model and one
 * sequence: for every layer l < cache->num_layers and q-head h,
 *   A[u][v] = softmax over v <= start+u of q_{l,u,h} · K_{l,kv(h)}[v] / sqrt(d)
 *   F[l*H + h][v - start] = Σ_{u < len} A[u][v],   v in [start, start+len)
 * (Eq. 1 column sums, of the window's causal prefill attention rows
 * over their full prefix).  Feed the LLM's and the SLM's F to
 * smallkv_match_heads (K0) to build the head map.
 *   q      device bf16 [num_layers][len][H][d]: the window's post-RoPE queries.
 *   cache  the model's paged cache (K used; positions [0, start+len) of
 *          sequence `seq` must be written — the caller's contract).
 *   seq    row of the block table.
 *   F      device fp32 [num_layers * H][len], fully written.
 * Tensor cores (mma.sync) for q·Kᵀ; deterministic.  Errors: NULL pointers,
 * head_dim not in {64,128}, len not in [1,1024], start < 0 or the window past
 * the block table, seq < 0, non-sm_100 device.
 */
int smallkv_prefill_scores(const uint16_t* q, const smallkv_cache* cache, int32_t seq,
                           int32_t start, int32_t len, float* F, void* stream);

/*
 * smallkv_match_heads — prefill similarity matching (Eq. 2-3).
 *   llm_F  device fp32 [n_llm][w]  accumulative scores F(A_i, C) (Eq. 1) of
 *          every LLM head over the matching window (R8).
 *   slm_F  device fp32 [n_slm][w]  same for every SLM head.
 *   k_match TopK size, 1 <= k_match <= w <= 512 (SPEC default
 *          max(16, ceil(0.2 w))).
 *   head_map out, device int32 [n_llm]: argmax_j Jaccard(TopK(F_i), TopK(F'_j)),
 *          ties -> smallest j.  TopK ties -> lower index.
 *   jaccard out, device fp32 [n_llm]: the winning Jaccard value.
 *   ws     device workspace >= smallkv_match_heads_workspace_size(n_llm, n_slm)
 *          bytes (TopK bitsets; no initialisation needed).
 * Errors: NULL pointers, w outside [1,512], k_match outside [1,w], n_llm or
 * n_slm < 1, small workspace, non-sm_100 device.
 */
size_t smallkv_match_heads_workspace_size(int32_t n_llm, int32_t n_slm);
int smallkv_match_heads(const float* llm_F, int32_t n_llm, const float* slm_F,
                        int32_t n_slm, int32_t w, int32_t k_match,
                        int32_t* head_map, float* jaccard, void* ws,
                        size_t ws_bytes, void* stream);

/* Zero-fill `bytes` of device memory at `ws` on `stream` (workspace init). */
int smallkv_workspace_init(void* ws, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SMALLKV_H_ */
