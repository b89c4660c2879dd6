/*
 * freekv_oracle.h -- plain CPU oracle of FreeKV's per-layer decode-step
 * KV-retrieval path (arXiv 2505.13109).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2505_13109_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * Citations "P:<line>" refer to PAPER.md lines (with section), "CFR-n" to the
 * canonical fp32 recipe written out in DESIGN.md §3.
 *
 * All q/K/V/summaries are bf16 given as raw uint16 bit patterns; every bf16 ->
 * fp32 conversion is exact (CFR-1).  Build flags (CFR-0):
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 */
#ifndef FREEKV_ORACLE_H
#define FREEKV_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* modes (Table tab:abl-tau: tau=0 "No Correction", tau=1 "No Speculation") */
#define FKO_MODE_SPECULATIVE 0
#define FKO_MODE_ALWAYS 1
#define FKO_MODE_NEVER 2

float fko_bf16_to_f32(uint16_t b);
/* round-to-nearest-even fp32 -> bf16 (used only by tests to build inputs) */
uint16_t fko_f32_to_bf16(float x);

/* Page summary, P:231 (§3.2 "min-max pooled keys within each page").
 * keys: [n_tok][d] bf16.  mn/mx: [d] bf16 = channel-wise min / max under the
 * total order of finite values with -0 < +0 (reading R-5). */
void fko_page_summary(const uint16_t* keys, int n_tok, int d, uint16_t* mn, uint16_t* mx);

/* Quest-style channel-wise upper bound, P:231 + reading A-1; CFR-2:
 * u = +0; for c ascending: u = fl(u + (q_c >= 0 ? q_c*mx_c : q_c*mn_c)). */
float fko_page_bound(const uint16_t* q, const uint16_t* mn, const uint16_t* mx, int d);

/* CFR-3: r = fl32(log2(e)/sqrt(d)) (evaluated in double then rounded). */
float fko_score_scale(int d);

/* CFR-5: the canonical exp2 for x <= 0. */
float fko_cexp2(float x);

/* CFR-6: balanced pairwise tree sum of a[0..n), n a power of two. */
float fko_tree_sum(const float* a, int n);

/* MeanS pooling, P:232-234 (§3.2, formula on P:234) with readings A-2..A-4;
 * CFR-4..8.  s: base-2 logits [G][ld] (only columns j in [j_begin, j_end) are
 * read).  Writes pooled[j] for j in [j_begin, j_end) = sum_g softmax_g(s)[j]
 * (un-divided by G, A-4).  n_leaves = next_pow2(j_end) leaves enter the tree. */
void fko_pool_means(const float* s, int G, int ld, int j_begin, int j_end, float* pooled);

/* Top-K, P:101 (§2.1) + A-5/CFR-9: the K largest pooled[j], j in [j_begin,
 * j_end), ties -> lower j; written ascending into sel[K], -1 padded.
 * If j_end - j_begin <= K all candidates are selected (A-11).
 * Returns the number selected. */
int fko_topk(const float* pooled, int j_begin, int j_end, int K, int32_t* sel);

/* Whole selection for one (batch, kv-head) unit, P:231-234 + P:257.
 * q: [G][d]; summ: [n_off][2][d] (index 0 = min, 1 = max; rows < n_sink unused).
 * Candidates J = [n_sink, n_off).  pooled_out (nullable): [n_off] floats
 * (rows outside J untouched).  Returns number selected. */
int fko_select_unit(const uint16_t* q, const uint16_t* summ, int G, int d,
                    int n_sink, int n_off, int K, int32_t* sel, float* pooled_out);

/* Cosine similarity of adjacent queries, P:180 (§3.1), CFR-10, A-14 (zero -> 0). */
float fko_cosine(const uint16_t* a, const uint16_t* b, int d);

/* Group-mean pooling of C and threshold, P:247-250 (§3.3), CFR-10, A-13.
 * Returns flag (1 = corrected); writes the pooled mean to *cbar. */
int fko_pool_correct(const float* C, int G, float tau, int mode, float* cbar);

/* ---- group-consistency variants (exp:abl-g-cons,
 * Table tab:abl-g-cons, Table tab:abl-g-corr).  The paper pools, max or mean over
 * the G heads of a group, (i) the query vectors (Q), (ii) the attention weights between the
 * queries and the page summaries (QK) or (iii) the softmax-normalised weights (S); FreeKV uses
 * MeanS.  CFR for the variants: MeanQ q_c = fl(seq-sum_g q_gc / G) in fp32,
 * MaxQ q_c = max_g q_gc, then CFR-2 with u = fma(q_c, m_c, u) and one softmax (G = 1);
 * MeanQK s_j = fl(seq-sum_g s_gj / G), MaxQK s_j = max_g s_gj, then one softmax; MaxS
 * pooled_j = max_g p_gj.  Ranking as CFR-9. */
#define FKO_POOL_MEAN_S 0
#define FKO_POOL_MAX_S 1
#define FKO_POOL_MEAN_QK 2
#define FKO_POOL_MAX_QK 3
#define FKO_POOL_MEAN_Q 4
#define FKO_POOL_MAX_Q 5
int fko_select_unit_pool(const uint16_t* q, const uint16_t* summ, int G, int d, int n_sink, int n_off, int K,
                         int pool, int32_t* sel, float* pooled_out);
/* Correction pooling (tab:abl-g-corr): cpool 0 = mean of C_g (FreeKV); cpool 1 = the paper's
 * "max pooling over group C_i", read as max pooling of the need to correct, i.e. the unit is
 * corrected when its least similar head is below tau (min_g C_g < tau) -- the paper says it
 * "triggers more corrections" than mean pooling, which max_g C_g would not (reading
 * R-11).  cbar = the pooled value. */
int fko_pool_correct_v(const float* C, int G, float tau, int mode, int cpool, float* cbar);

/* Correction decision for one unit: cosine per head then fko_pool_correct.
 * bootstrap != 0 (no resident selection yet, A-12) -> flagged. */
int fko_correct_unit(const uint16_t* q, const uint16_t* q_prev, int G, int d,
                     float tau, int mode, int bootstrap, float* cbar);

/* Attention over a token subset in fp64, P:95-97 (§2.1):
 * o_h = sum_{t in toks} softmax_t(q_h . k_t / sqrt(d)) v_t.
 * q: [G][d]; Kt/Vt: [*][d] rows indexed by toks[0..n_tok); out: [G][d]. */
void fko_attn_unit(const uint16_t* q, const uint16_t* Kt, const uint16_t* Vt,
                   int G, int d, const int32_t* toks, int n_tok, double* out);

/* Batched helpers (OpenMP across units only; never inside a unit, CFR-0). */
void fko_select_batch(int n_units, const uint16_t* q /*[U][G][d]*/,
                      const uint16_t* const* summ /*U pointers*/, int G, int d,
                      int n_sink, const int32_t* n_off /*[U]*/, int K,
                      int32_t* sel /*[U][K]*/);
void fko_attn_batch(int n_units, const uint16_t* q /*[U][G][d]*/,
                    const uint16_t* const* Kt, const uint16_t* const* Vt,
                    int G, int d, const int32_t* const* toks, const int32_t* n_tok,
                    double* out /*[U][G][d]*/);
int fko_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
