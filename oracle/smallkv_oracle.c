/*
 * smallkv_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU implementation of SmallKV's decode hot path
 * (arXiv 2508.02751), written straight from the paper so that the CUDA path
 * in paper_2508_02751_b200/ can be checked against it.  It shares no code,
 * header, table or helper with the CUDA path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; R1..R15 = the
 * readings listed in DESIGN.md §3.
 *
 * Every step follows the paper's order and notation:
 *   oracle_slm_rows   — A'_{f(i)} for the current decode token: the softmax of
 *                       q'·K'^T/sqrt(d_h) over the full SLM cache C^s_all
 *                       (P:107 A = Softmax(QK^T/sqrt(d_h)); "In
 *                       decoding stage, let the attention be A_i ∈ R^{1×n}").
 *   oracle_split      — Eq. 4 as "retain the top" (R7) with recent window (R10)
 *                       and Eq. 6's TopK / Top(P-K) bands (R4), ties by lower
 *                       index (R3).
 *   oracle_attend     — Eq. 6 / Alg. 1 l.12-14: O_c = FlashAttention over the
 *                       critical ∪ recent K/V (R2),
 *                       O_m = A'_{f(i)}[M]·V[M], O = O_c + O_m (R13,
 *                       P:205).
 *   oracle_match_heads— Eq. 2 Jaccard of TopK sets, Eq. 3 argmax.
 *   oracle_select_acc — variant f1: Eq. 1 running column sums.
 *   oracle_match_window / oracle_prefill_scores — variant f3: matching window
 *                       (R17) and Eq. 1 column sums of the window's causal
 *                       prefill attention rows, the F vectors of Eq. 2.
 *   oracle_select_group / oracle_attend_group — variant f2: one split per LLM
 *                       KV head of the summed proxy rows (R16), per-head
 *                       marginal weights.
 *
 * Precision: bf16 inputs are widened exactly to double; all arithmetic is
 * double.  Sorting uses the C library qsort (a library primitive).
 * Parity pins for each function are in tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- bf16 bits -> double (exact: bf16 is the top half of an IEEE fp32) ---- */
static double bf16_to_double(uint16_t bits) {
  uint32_t u = ((uint32_t)bits) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

/* One model's paged cache, in the layout the caller hands the hot path:
 *   pool[layer][page][kv_head][page_size][head_dim], bf16 bits,
 *   token pos of sequence b in page block_table[b][pos / page_size],
 *   row pos % page_size. */
typedef struct {
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
} oracle_cache;

/* Address of the head_dim-long row of (layer, sequence b, token pos, kv head). */
static const uint16_t* cache_row(const oracle_cache* c, const uint16_t* pool,
                                 int layer, int b, int pos, int kvh) {
  int32_t page = c->block_table[(int64_t)b * c->max_blocks + pos / c->page_size];
  int64_t row = (((int64_t)layer * c->num_pages + page) * c->num_kv_heads + kvh) *
                    c->page_size + pos % c->page_size;
  return pool + row * c->head_dim;
}

/* ------------------------------------------------------------------------- *
 * Step 1: the SLM attention row of flat SLM head j for sequence b.
 * A = Softmax(Q K^T / sqrt(d_h)); in decode Q is the current token's
 * query, so the row is a'_v = exp(s'_v - m') / Σ_u exp(s'_u - m') with
 * s'_v = q'·K'[v] / sqrt(d_s), over every cached token v in [0, n) of the full
 * SLM cache C^s_all (the SLM cache is never compressed, R11).
 * Outputs: s[n] (logits), a[n] (probabilities), *m (max logit), *lse.
 * ------------------------------------------------------------------------- */
void oracle_slm_row(const uint16_t* slm_q, /* [l][B][H_s][d_s] */
                    const oracle_cache* slm, int32_t batch, int32_t j, int32_t b,
                    int32_t n, double* s, double* a, double* m_out,
                    double* lse_out) {
  const int H_s = slm->num_q_heads, d = slm->head_dim;
  const int layer = j / H_s, head = j % H_s;
  const int G_s = H_s / slm->num_kv_heads;
  const int kvh = head / G_s;
  const uint16_t* q = slm_q + (((int64_t)layer * batch + b) * H_s + head) * d;
  const double scale = 1.0 / sqrt((double)d);
  double m = -INFINITY;
  for (int v = 0; v < n; ++v) {
    const uint16_t* kr = cache_row(slm, slm->k, layer, b, v, kvh);
    double dot = 0.0;
    for (int t = 0; t < d; ++t) dot += bf16_to_double(q[t]) * bf16_to_double(kr[t]);
    s[v] = dot * scale;
    if (s[v] > m) m = s[v];
  }
  double z = 0.0;
  for (int v = 0; v < n; ++v) z += exp(s[v] - m);
  for (int v = 0; v < n; ++v) a[v] = exp(s[v] - m) / z;
  if (m_out) *m_out = m;
  if (lse_out) *lse_out = m + log(z);
}

/* ------------------------------------------------------------------------- *
 * Step 2-3: budgets and the three-way split of one score row (Eq. 4, Eq. 6).
 * R5 clamp: R' = min(R, n), K' = min(K, n-R'), M' = min(M, n-R'-K').
 * Recent = [n-R', n) (R10).  Positions v in [0, n-R') are sorted by
 * (score desc, v asc) (R3); critical = the first K' (Eq. 6 TopK),
 * marginal = the next M' (Eq. 6 Top(P-K), R4), evicted = the rest.
 * crit / marg are written in ascending position order.
 * counts[0] = K', counts[1] = M', counts[2] = R'.
 * ------------------------------------------------------------------------- */
typedef struct {
  double score;
  int32_t idx;
} scored_t;

static int cmp_score_desc_idx_asc(const void* pa, const void* pb) {
  const scored_t* x = (const scored_t*)pa;
  const scored_t* y = (const scored_t*)pb;
  if (x->score > y->score) return -1;
  if (x->score < y->score) return 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

static int cmp_int(const void* pa, const void* pb) {
  int32_t x = *(const int32_t*)pa, y = *(const int32_t*)pb;
  return (x > y) - (x < y);
}

void oracle_split(const double* score, int32_t n, int32_t K, int32_t R, int32_t M,
                  int32_t* crit, int32_t* marg, int32_t* counts) {
  int32_t Rc = R < n ? R : n;
  if (Rc < 0) Rc = 0;
  int32_t Kc = K < n - Rc ? K : n - Rc;
  if (Kc < 0) Kc = 0;
  int32_t Mc = M < n - Rc - Kc ? M : n - Rc - Kc;
  if (Mc < 0) Mc = 0;
  const int32_t ranked = n - Rc;
  scored_t* order = (scored_t*)malloc(sizeof(scored_t) * (ranked > 0 ? ranked : 1));
  for (int32_t v = 0; v < ranked; ++v) {
    order[v].score = score[v];
    order[v].idx = v;
  }
  qsort(order, (size_t)ranked, sizeof(scored_t), cmp_score_desc_idx_asc);
  for (int32_t i = 0; i < Kc; ++i) crit[i] = order[i].idx;
  for (int32_t i = 0; i < Mc; ++i) marg[i] = order[Kc + i].idx;
  qsort(crit, (size_t)Kc, sizeof(int32_t), cmp_int);
  qsort(marg, (size_t)Mc, sizeof(int32_t), cmp_int);
  counts[0] = Kc;
  counts[1] = Mc;
  counts[2] = Rc;
  free(order);
}

/* ------------------------------------------------------------------------- *
 * Steps 1-3 for every requested (row j, sequence b).
 * rows[n_rows]: flat SLM heads to process (the image of the head map).
 * Outputs per (r, b), r the index into rows[]:
 *   a_out  [n_rows][B][max_n]  SLM probabilities a'_v (v < n_b)
 *   s_out  [n_rows][B][max_n]  logits s'_v (may be NULL)
 *   stats  [n_rows][B][2]      (m', lse')
 *   crit   [n_rows][B][max_crit], marg [n_rows][B][max_marg]
 *   counts [n_rows][B][3]      (K', M', R')
 * Ranking uses a' (the probabilities, Eq. 6's F(A'_{f(i)}) with F the row
 * itself in decode, R1).
 * ------------------------------------------------------------------------- */
void oracle_select(const uint16_t* slm_q, const oracle_cache* slm,
                   const int32_t* seq_lens, int32_t batch, int32_t max_n,
                   const int32_t* rows, int32_t n_rows, const int32_t* k_crit,
                   const int32_t* n_recent, const int32_t* k_marg,
                   int32_t max_crit, int32_t max_marg, double* a_out,
                   double* s_out, double* stats, int32_t* crit, int32_t* marg,
                   int32_t* counts) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t rb = 0; rb < (int64_t)n_rows * batch; ++rb) {
    const int32_t r = (int32_t)(rb / batch), b = (int32_t)(rb % batch);
    const int32_t n = seq_lens[b];
    double* a = a_out + rb * max_n;
    double* s = s_out ? s_out + rb * max_n : (double*)malloc(sizeof(double) * n);
    oracle_slm_row(slm_q, slm, batch, rows[r], b, n, s, a, &stats[rb * 2],
                   &stats[rb * 2 + 1]);
    oracle_split(a, n, k_crit[b], n_recent[b], k_marg[b], crit + rb * max_crit,
                 marg + rb * max_marg, counts + rb * 3);
    if (!s_out) free(s);
  }
}

/* ------------------------------------------------------------------------- *
 * Variant f1: accumulative score selection.  Eq. 1
 * defines F(A, C) as the column sums s^v = Σ_u A[u, v] of the attention matrix;
 * in decode each step contributes one more row, so the running score of the
 * SLM row j is  F_t[v] = F_{t-1}[v] + a'_t[v]  (positions new at step t start
 * from F_{t-1} = 0, i.e. the caller zero-fills acc once).  The split then ranks
 * by F_t instead of a'_t (Eq. 6 with F over all rows seen so far); the
 * marginal weights stay the current row a'_t (Eq. 6: A'_{f(i)}[k]).
 * acc [n_rows][B][max_n] is read and updated in place; everything else is as
 * oracle_select.
 * ------------------------------------------------------------------------- */
void oracle_select_acc(const uint16_t* slm_q, const oracle_cache* slm,
                       const int32_t* seq_lens, int32_t batch, int32_t max_n,
                       const int32_t* rows, int32_t n_rows, const int32_t* k_crit,
                       const int32_t* n_recent, const int32_t* k_marg,
                       int32_t max_crit, int32_t max_marg, double* acc, double* a_out,
                       double* s_out, double* stats, int32_t* crit, int32_t* marg,
                       int32_t* counts) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t rb = 0; rb < (int64_t)n_rows * batch; ++rb) {
    const int32_t r = (int32_t)(rb / batch), b = (int32_t)(rb % batch);
    const int32_t n = seq_lens[b];
    double* a = a_out + rb * max_n;
    double* f = acc + rb * max_n;
    double* s = s_out ? s_out + rb * max_n : (double*)malloc(sizeof(double) * n);
    oracle_slm_row(slm_q, slm, batch, rows[r], b, n, s, a, &stats[rb * 2],
                   &stats[rb * 2 + 1]);
    for (int32_t v = 0; v < n; ++v) f[v] += a[v];
    oracle_split(f, n, k_crit[b], n_recent[b], k_marg[b], crit + rb * max_crit,
                 marg + rb * max_marg, counts + rb * 3);
    if (!s_out) free(s);
  }
}

/* ------------------------------------------------------------------------- *
 * Step 4: compensated attention of one LLM layer (Alg. 1 l.12-14).
 * For LLM head h of layer `layer` (cache slot `cache_layer`), j = head_map[layer*H+h],
 * kv head g = h / (H/H_kv), and the sets of row r_of_head = row_slot[j]:
 *   l_k = q_h·K_g[k] / sqrt(d)                  k in C ∪ R'
 *   w_k = exp(l_k - max) / Σ exp(l - max)       (FlashAttention over the
 *                                               selected K/V, R2)
 *   O_c = Σ w_k V_g[k]   (0 when C ∪ R' is empty)
 *   O_m = Σ_{k∈M} a'_j[k] V_g[k]                (Eq. 6 second branch)
 *   out = O_c + O_m                              (no renormalisation, R13)
 * a_rows[n_rows][B][max_n] are the SLM probabilities (from oracle_select);
 * crit/marg/counts are the selection lists (the oracle's own or, for output
 * parity, the GPU's verified ones).
 * out: [B][H][d] doubles.  Also writes the critical softmax mass check
 * wsum_out[B][H] = Σ w_k (must be 1 when C ∪ R' is non-empty), may be NULL.
 * ------------------------------------------------------------------------- */
/* One head's compensated output: sets (crit / marg / counts) of selection row
 * `rb_set`, marginal weights a' of SLM row `rb_w` (both [slot][b] indices). */
static void attend_head(const oracle_cache* llm, int32_t cache_layer, const uint16_t* qh, int b,
                        int n, int g, int64_t rb_set, int64_t rb_w, const double* a_rows,
                        int32_t max_n, const int32_t* crit, const int32_t* marg,
                        const int32_t* counts, int32_t max_crit, int32_t max_marg, double* o,
                        double* wsum_out) {
  const int d = llm->head_dim;
  const double scale = 1.0 / sqrt((double)d);
  const int32_t Kc = counts[rb_set * 3], Mc = counts[rb_set * 3 + 1], Rc = counts[rb_set * 3 + 2];
  const int32_t* C = crit + rb_set * max_crit;
  const int32_t* Mset = marg + rb_set * max_marg;
  const double* a = a_rows + rb_w * max_n;
  for (int t = 0; t < d; ++t) o[t] = 0.0;

  /* critical ∪ recent positions */
  const int nsel = Kc + Rc;
  int32_t* sel = (int32_t*)malloc(sizeof(int32_t) * (nsel > 0 ? nsel : 1));
  for (int i = 0; i < Kc; ++i) sel[i] = C[i];
  for (int i = 0; i < Rc; ++i) sel[Kc + i] = n - Rc + i;
  double* logit = (double*)malloc(sizeof(double) * (nsel > 0 ? nsel : 1));
  double mx = -INFINITY;
  for (int i = 0; i < nsel; ++i) {
    const uint16_t* kr = cache_row(llm, llm->k, cache_layer, b, sel[i], g);
    double dot = 0.0;
    for (int t = 0; t < d; ++t) dot += bf16_to_double(qh[t]) * bf16_to_double(kr[t]);
    logit[i] = dot * scale;
    if (logit[i] > mx) mx = logit[i];
  }
  double z = 0.0;
  for (int i = 0; i < nsel; ++i) z += exp(logit[i] - mx);
  double wsum = 0.0;
  for (int i = 0; i < nsel; ++i) {
    const double w = exp(logit[i] - mx) / z;
    wsum += w;
    const uint16_t* vr = cache_row(llm, llm->v, cache_layer, b, sel[i], g);
    for (int t = 0; t < d; ++t) o[t] += w * bf16_to_double(vr[t]);
  }
  /* marginal compensation: SLM weights times LLM V */
  for (int i = 0; i < Mc; ++i) {
    const int k = Mset[i];
    const uint16_t* vr = cache_row(llm, llm->v, cache_layer, b, k, g);
    for (int t = 0; t < d; ++t) o[t] += a[k] * bf16_to_double(vr[t]);
  }
  if (wsum_out) *wsum_out = wsum;
  free(sel);
  free(logit);
}

void oracle_attend(int32_t layer, int32_t cache_layer, const uint16_t* q, /* [B][H][d] */
                   const oracle_cache* llm, const int32_t* seq_lens, int32_t batch,
                   const int32_t* head_map, const int32_t* row_slot,
                   const double* a_rows, int32_t max_n, const int32_t* crit,
                   const int32_t* marg, const int32_t* counts, int32_t max_crit,
                   int32_t max_marg, double* out, double* wsum_out) {
  const int H = llm->num_q_heads, d = llm->head_dim;
  const int G = H / llm->num_kv_heads;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t bh = 0; bh < (int64_t)batch * H; ++bh) {
    const int b = (int)(bh / H), h = (int)(bh % H);
    const int j = head_map[layer * H + h];
    const int64_t rb = (int64_t)row_slot[j] * batch + b;
    attend_head(llm, cache_layer, q + ((int64_t)b * H + h) * d, b, seq_lens[b], h / G, rb, rb,
                a_rows, max_n, crit, marg, counts, max_crit, max_marg, out + bh * d,
                wsum_out ? wsum_out + bh : NULL);
  }
}

/* ------------------------------------------------------------------------- *
 * Variant f2: per-kv-group shared selection (R16).
 * For LLM layer `layer`, kv group g (q heads g·G .. g·G+G-1) and sequence b,
 * the group score sums the SLM proxy rows of the group's heads,
 *     F_g[v] = Σ_{h in group g} a'_{f(layer,h)}[v]
 * (Eq. 6's F(A'_{f(i)}) of each head i, summed over the heads that share one
 * LLM KV head; App. A counts budgets per KV head), and ONE three-way
 * split of F_g (oracle_split: Eq. 4 / Eq. 6, R3-R5, R7, R10) is shared by all
 * heads of the group.  a_rows / row_slot come from oracle_select over the
 * image of the head map.  Outputs per (g, b), gb = g·B + b:
 *   score [H_kv][B][max_n], crit [H_kv][B][max_crit], marg [H_kv][B][max_marg],
 *   counts [H_kv][B][3] = (K', M', R').
 * ------------------------------------------------------------------------- */
void oracle_select_group(int32_t layer, int32_t H, int32_t H_kv, const int32_t* head_map,
                         const int32_t* row_slot, const double* a_rows, int32_t max_n,
                         const int32_t* seq_lens, int32_t batch, const int32_t* k_crit,
                         const int32_t* n_recent, const int32_t* k_marg, int32_t max_crit,
                         int32_t max_marg, double* score, int32_t* crit, int32_t* marg,
                         int32_t* counts) {
  const int G = H / H_kv;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t gb = 0; gb < (int64_t)H_kv * batch; ++gb) {
    const int g = (int)(gb / batch), b = (int)(gb % batch);
    const int n = seq_lens[b];
    double* F = score + gb * max_n;
    for (int v = 0; v < n; ++v) F[v] = 0.0;
    for (int h = 0; h < G; ++h) {
      const int j = head_map[layer * H + g * G + h];
      const double* a = a_rows + ((int64_t)row_slot[j] * batch + b) * max_n;
      for (int v = 0; v < n; ++v) F[v] += a[v];
    }
    oracle_split(F, n, k_crit[b], n_recent[b], k_marg[b], crit + gb * max_crit,
                 marg + gb * max_marg, counts + gb * 3);
  }
}

/* Step 4 for variant f2: head h of group g attends over its group's shared
 * sets (crit / marg / counts of (g, b)); its marginal weights stay its own SLM
 * row a'_{f(layer,h)} (Eq. 6 second branch). */
void oracle_attend_group(int32_t layer, int32_t cache_layer, const uint16_t* q, /* [B][H][d] */
                         const oracle_cache* llm, const int32_t* seq_lens, int32_t batch,
                         const int32_t* head_map, const int32_t* row_slot,
                         const double* a_rows, int32_t max_n, const int32_t* crit,
                         const int32_t* marg, const int32_t* counts, int32_t max_crit,
                         int32_t max_marg, double* out, double* wsum_out) {
  const int H = llm->num_q_heads, d = llm->head_dim;
  const int G = H / llm->num_kv_heads;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t bh = 0; bh < (int64_t)batch * H; ++bh) {
    const int b = (int)(bh / H), h = (int)(bh % H);
    const int j = head_map[layer * H + h];
    const int64_t rb_w = (int64_t)row_slot[j] * batch + b;
    const int64_t rb_set = (int64_t)(h / G) * batch + b;
    attend_head(llm, cache_layer, q + ((int64_t)b * H + h) * d, b, seq_lens[b], h / G, rb_set,
                rb_w, a_rows, max_n, crit, marg, counts, max_crit, max_marg, out + bh * d,
                wsum_out ? wsum_out + bh : NULL);
  }
}

/* ------------------------------------------------------------------------- *
 * Prefill matching (Eq. 2-3).
 * oracle_topk: the k positions with the largest F, ties -> lower index
 * (S:121), returned as a membership mask in_top[w].
 * oracle_match_heads: S(i,j) = |T_i ∩ T'_j| / |T_i ∪ T'_j| (Eq. 2),
 * f(i) = argmax_j S(i,j) with ties -> smallest j (Eq. 3).
 * ------------------------------------------------------------------------- */
void oracle_topk(const double* F, int32_t w, int32_t k, uint8_t* in_top) {
  scored_t* order = (scored_t*)malloc(sizeof(scored_t) * (w > 0 ? w : 1));
  for (int32_t v = 0; v < w; ++v) {
    order[v].score = F[v];
    order[v].idx = v;
    in_top[v] = 0;
  }
  qsort(order, (size_t)w, sizeof(scored_t), cmp_score_desc_idx_asc);
  for (int32_t i = 0; i < k && i < w; ++i) in_top[order[i].idx] = 1;
  free(order);
}

void oracle_match_heads(const double* llm_F, int32_t n_llm, const double* slm_F,
                        int32_t n_slm, int32_t w, int32_t k, int32_t* head_map,
                        double* jaccard) {
  uint8_t* tl = (uint8_t*)malloc((size_t)n_llm * w + 1);
  uint8_t* ts = (uint8_t*)malloc((size_t)n_slm * w + 1);
  for (int32_t i = 0; i < n_llm; ++i) oracle_topk(llm_F + (int64_t)i * w, w, k, tl + (int64_t)i * w);
  for (int32_t j = 0; j < n_slm; ++j) oracle_topk(slm_F + (int64_t)j * w, w, k, ts + (int64_t)j * w);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n_llm; ++i) {
    double best = -1.0;
    int32_t best_j = -1;
    for (int32_t j = 0; j < n_slm; ++j) {
      int32_t inter = 0, uni = 0;
      for (int32_t v = 0; v < w; ++v) {
        const int x = tl[(int64_t)i * w + v], y = ts[(int64_t)j * w + v];
        inter += x & y;
        uni += x | y;
      }
      const double s = uni == 0 ? 1.0 : (double)inter / (double)uni;
      if (s > best) {
        best = s;
        best_j = j;
      }
    }
    head_map[i] = best_j;
    jaccard[i] = best;
  }
  free(tl);
  free(ts);
}

/* Eq. 1 accumulative score F(A, C) of one n×n attention matrix (column sums,
 * s^v = Σ_u A[u, v]); used to build matching inputs and for pins. */
void oracle_accumulate_scores(const double* A, int32_t n, double* F) {
  for (int32_t v = 0; v < n; ++v) {
    double s = 0.0;
    for (int32_t u = 0; u < n; ++u) s += A[(int64_t)u * n + v];
    F[v] = s;
  }
}

/* ------------------------------------------------------------------------- *
 * Variant f3: prefill-side scores for head matching.
 * Matching window ("range of 100 to 200 ... delays ... truncate",
 * R17): n < w_min => DEFER (returns 0); else len = min(n, w_max) and
 * start = keep_last ? n - len : 0 (SPEC S:157-162 keeps the most recent).
 * ------------------------------------------------------------------------- */
int oracle_match_window(int32_t n, int32_t w_min, int32_t w_max, int32_t keep_last,
                        int32_t* start, int32_t* len) {
  if (n < w_min) return 0;
  *len = n < w_max ? n : w_max;
  *start = keep_last ? n - *len : 0;
  return 1;
}

/* F over the window of one sequence (Eq. 1): for every layer l and
 * head h, the causal prefill attention rows of the window's queries
 *   A[u][v] = softmax_{v <= pos(u)} (q_{l,u,h} · k_{l,v,kv(h)} / sqrt(d)),
 *   pos(u) = start + u  (the full causal prefix, P:107 A = Softmax(QK^T/sqrt(d_h)))
 * summed over the window's rows:  F[l*H + h][v - start] = Σ_u A[u][v] for v in
 * the window.  q: bf16 [L][len][H][d] (the window's queries); K from the paged
 * cache of sequence b, layer slots 0..L-1.  F: [L*H][len] doubles. */
void oracle_prefill_scores(const uint16_t* q, const oracle_cache* c, int32_t b, int32_t start,
                           int32_t len, double* F) {
  const int L = c->num_layers, H = c->num_q_heads, d = c->head_dim;
  const int G = H / c->num_kv_heads;
  const double scale = 1.0 / sqrt((double)d);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t lh = 0; lh < (int64_t)L * H; ++lh) {
    const int l = (int)(lh / H), h = (int)(lh % H);
    double* f = F + lh * len;
    for (int v = 0; v < len; ++v) f[v] = 0.0;
    double* s = (double*)malloc(sizeof(double) * (start + len));
    for (int u = 0; u < len; ++u) {
      const int pos = start + u;
      const uint16_t* qu = q + (((int64_t)l * len + u) * H + h) * d;
      double mx = -INFINITY;
      for (int v = 0; v <= pos; ++v) {
        const uint16_t* kr = cache_row(c, c->k, l, b, v, h / G);
        double dot = 0.0;
        for (int t = 0; t < d; ++t) dot += bf16_to_double(qu[t]) * bf16_to_double(kr[t]);
        s[v] = dot * scale;
        if (s[v] > mx) mx = s[v];
      }
      double z = 0.0;
      for (int v = 0; v <= pos; ++v) z += exp(s[v] - mx);
      for (int v = start; v <= pos; ++v) f[v - start] += exp(s[v] - mx) / z;
    }
    free(s);
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
