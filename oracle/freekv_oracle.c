/*
 * freekv_oracle.c -- plain, slow, obviously correct CPU oracle of FreeKV's
 * decode-step KV-retrieval path (arXiv 2505.13109).  See freekv_oracle.h.
 *
 * TEST INFRASTRUCTURE ONLY -- never linked by the product path.
 *
 * Every function follows one passage of PAPER.md (cited) and the canonical
 * fp32 recipe (CFR) written out in DESIGN.md §3.  No blocking, fusion or
 * reordering beyond what the recipe states.  Floating point: x86-64 SSE,
 * FLT_EVAL_METHOD == 0, compiled with -ffp-contract=off -fno-fast-math so
 * every float operation below rounds once, in the order written.
 */
#include "freekv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static float f32_from_bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t bits_from_f32(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

float fko_bf16_to_f32(uint16_t b) { return f32_from_bits(((uint32_t)b) << 16); }

uint16_t fko_f32_to_bf16(float x) {
    uint32_t u = bits_from_f32(x);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (uint16_t)((u >> 16) | 0x40); /* NaN */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

/* Total order on finite bf16 values with -0 < +0 (reading R-5). */
static int bf16_less(uint16_t a, uint16_t b) {
    float fa = fko_bf16_to_f32(a), fb = fko_bf16_to_f32(b);
    if (fa < fb) return 1;
    if (fa > fb) return 0;
    /* equal values: only +-0 can differ in bits; -0 (sign set) is smaller */
    return (a & 0x8000u) && !(b & 0x8000u);
}

void fko_page_summary(const uint16_t* keys, int n_tok, int d, uint16_t* mn, uint16_t* mx) {
    for (int c = 0; c < d; ++c) {
        uint16_t lo = keys[c], hi = keys[c];
        for (int t = 1; t < n_tok; ++t) {
            uint16_t k = keys[(size_t)t * d + c];
            if (bf16_less(k, lo)) lo = k;
            if (bf16_less(hi, k)) hi = k;
        }
        mn[c] = lo;
        mx[c] = hi;
    }
}

float fko_page_bound(const uint16_t* q, const uint16_t* mn, const uint16_t* mx, int d) {
    float u = 0.0f;
    for (int c = 0; c < d; ++c) {
        float qc = fko_bf16_to_f32(q[c]);
        float t = (qc >= 0.0f) ? qc * fko_bf16_to_f32(mx[c]) : qc * fko_bf16_to_f32(mn[c]);
        u = u + t;
    }
    return u;
}

float fko_score_scale(int d) { return (float)(1.4426950408889634074 / sqrt((double)d)); }

float fko_cexp2(float x) {
    /* CFR-5 coefficients c_k = fl32(ln2^k / k!), k = 0..7 */
    static const uint32_t C[8] = {0x3F800000u, 0x3F317218u, 0x3E75FDF0u, 0x3D635847u,
                                  0x3C1D955Bu, 0x3AAEC3FFu, 0x39218489u, 0x377FE5FEu};
    if (x < -125.0f) return 0.0f;
    float n = rintf(x);          /* ties-to-even under the default rounding mode */
    float f = x - n;             /* exact, |f| <= 1/2 */
    float P = f32_from_bits(C[7]);
    for (int k = 6; k >= 0; --k) P = fmaf(P, f, f32_from_bits(C[k]));
    int32_t ni = (int32_t)n;
    return f32_from_bits(bits_from_f32(P) + ((uint32_t)ni << 23));
}

float fko_tree_sum(const float* a, int n) {
    if (n == 1) return a[0];
    int h = n / 2;
    float l = fko_tree_sum(a, h);
    float r = fko_tree_sum(a + h, h);
    return l + r;
}

static int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

void fko_pool_means(const float* s, int G, int ld, int j_begin, int j_end, float* pooled) {
    int P2 = next_pow2(j_end > 0 ? j_end : 1);
    float* e = (float*)calloc((size_t)P2, sizeof(float));
    for (int j = j_begin; j < j_end; ++j) pooled[j] = 0.0f;
    for (int g = 0; g < G; ++g) {
        const float* sg = s + (size_t)g * ld;
        /* CFR-4: m = max over candidates */
        float m = sg[j_begin];
        for (int j = j_begin + 1; j < j_end; ++j)
            if (sg[j] > m) m = sg[j];
        /* CFR-5: e_j = cexp2(s_j - m); non-candidate leaves stay +0 */
        memset(e, 0, (size_t)P2 * sizeof(float));
        for (int j = j_begin; j < j_end; ++j) e[j] = fko_cexp2(sg[j] - m);
        /* CFR-6: Z = pairwise tree over leaves 0..P2-1 */
        float Z = fko_tree_sum(e, P2);
        /* CFR-7 normalise, CFR-8 pool sequentially over g */
        for (int j = j_begin; j < j_end; ++j) {
            float p = e[j] / Z;
            pooled[j] = (g == 0) ? p : pooled[j] + p;
        }
    }
    free(e);
}

typedef struct { uint32_t key; int32_t j; } kj_t;

static int cmp_rank(const void* a, const void* b) {
    const kj_t* x = (const kj_t*)a;
    const kj_t* y = (const kj_t*)b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1; /* key descending */
    return x->j < y->j ? -1 : (x->j > y->j ? 1 : 0);        /* id ascending */
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int fko_topk(const float* pooled, int j_begin, int j_end, int K, int32_t* sel) {
    int n = j_end - j_begin;
    if (n < 0) n = 0;
    for (int i = 0; i < K; ++i) sel[i] = -1;
    if (n <= K) {
        for (int i = 0; i < n; ++i) sel[i] = j_begin + i;
        return n;
    }
    kj_t* a = (kj_t*)malloc((size_t)n * sizeof(kj_t));
    for (int i = 0; i < n; ++i) {
        uint32_t k = bits_from_f32(pooled[j_begin + i]);
        if (k == 0x80000000u) k = 0u; /* -0 -> +0 (CFR-9); all pooled >= 0 */
        a[i].key = k;
        a[i].j = j_begin + i;
    }
    qsort(a, (size_t)n, sizeof(kj_t), cmp_rank);
    for (int i = 0; i < K; ++i) sel[i] = a[i].j;
    qsort(sel, (size_t)K, sizeof(int32_t), cmp_i32);
    free(a);
    return K;
}

int fko_select_unit(const uint16_t* q, const uint16_t* summ, int G, int d,
                    int n_sink, int n_off, int K, int32_t* sel, float* pooled_out) {
    int n = n_off - n_sink;
    if (n <= K) return fko_topk(NULL, n_sink, n_off, K, sel); /* A-11: all of J */
    float r = fko_score_scale(d);
    float* s = (float*)calloc((size_t)G * n_off, sizeof(float));
    float* pooled = (float*)calloc((size_t)n_off, sizeof(float));
    for (int g = 0; g < G; ++g)
        for (int j = n_sink; j < n_off; ++j) {
            const uint16_t* mn = summ + (size_t)j * 2 * d;
            const uint16_t* mx = mn + d;
            float u = fko_page_bound(q + (size_t)g * d, mn, mx, d); /* CFR-2 */
            s[(size_t)g * n_off + j] = u * r;                       /* CFR-3 */
        }
    fko_pool_means(s, G, n_off, n_sink, n_off, pooled);
    int cnt = fko_topk(pooled, n_sink, n_off, K, sel);
    if (pooled_out)
        for (int j = n_sink; j < n_off; ++j) pooled_out[j] = pooled[j];
    free(s);
    free(pooled);
    return cnt;
}

/* ---- group-consistency variants (f3), see freekv_oracle.h ---- */

/* CFR-2 with an fp32 query: u = fma(q_c, m_c, u) (exact product, one rounding) */
static float page_bound_f32q(const float* q, const uint16_t* mn, const uint16_t* mx, int d) {
    float u = 0.0f;
    for (int c = 0; c < d; ++c) {
        float m = (q[c] >= 0.0f) ? fko_bf16_to_f32(mx[c]) : fko_bf16_to_f32(mn[c]);
        u = fmaf(q[c], m, u);
    }
    return u;
}

/* softmax over candidates per head g < G (CFR-4..7), then pooled_j = max_g p_gj */
static void pool_max_s(const float* s, int G, int ld, int j_begin, int j_end, float* pooled) {
    float* one = (float*)calloc((size_t)ld, sizeof(float));
    for (int g = 0; g < G; ++g) {
        fko_pool_means(s + (size_t)g * ld, 1, ld, j_begin, j_end, one); /* one head's p */
        for (int j = j_begin; j < j_end; ++j) pooled[j] = (g == 0 || one[j] > pooled[j]) ? one[j] : pooled[j];
    }
    free(one);
}

int fko_select_unit_pool(const uint16_t* q, const uint16_t* summ, int G, int d, int n_sink, int n_off, int K,
                         int pool, int32_t* sel, float* pooled_out) {
    if (pool == FKO_POOL_MEAN_S) return fko_select_unit(q, summ, G, d, n_sink, n_off, K, sel, pooled_out);
    int n = n_off - n_sink;
    if (n <= K) return fko_topk(NULL, n_sink, n_off, K, sel); /* A-11 */
    float r = fko_score_scale(d);
    float* s = (float*)calloc((size_t)G * n_off, sizeof(float));
    float* pooled = (float*)calloc((size_t)n_off, sizeof(float));
    if (pool == FKO_POOL_MEAN_Q || pool == FKO_POOL_MAX_Q) {
        /* (i) pool the queries, score once */
        float* qb = (float*)calloc((size_t)d, sizeof(float));
        for (int c = 0; c < d; ++c) {
            float a = fko_bf16_to_f32(q[c]);
            for (int g = 1; g < G; ++g) {
                float x = fko_bf16_to_f32(q[(size_t)g * d + c]);
                a = (pool == FKO_POOL_MEAN_Q) ? a + x : (x > a ? x : a);
            }
            qb[c] = (pool == FKO_POOL_MEAN_Q) ? a / (float)G : a;
        }
        for (int j = n_sink; j < n_off; ++j) {
            const uint16_t* mn = summ + (size_t)j * 2 * d;
            s[j] = page_bound_f32q(qb, mn, mn + d, d) * r;
        }
        fko_pool_means(s, 1, n_off, n_sink, n_off, pooled);
        free(qb);
    } else {
        for (int g = 0; g < G; ++g)
            for (int j = n_sink; j < n_off; ++j) {
                const uint16_t* mn = summ + (size_t)j * 2 * d;
                s[(size_t)g * n_off + j] = fko_page_bound(q + (size_t)g * d, mn, mn + d, d) * r;
            }
        if (pool == FKO_POOL_MAX_S) {
            pool_max_s(s, G, n_off, n_sink, n_off, pooled);
        } else { /* (ii) pool the scores, one softmax */
            float* sb = (float*)calloc((size_t)n_off, sizeof(float));
            for (int j = n_sink; j < n_off; ++j) {
                float a = s[j];
                for (int g = 1; g < G; ++g) {
                    float x = s[(size_t)g * n_off + j];
                    a = (pool == FKO_POOL_MEAN_QK) ? a + x : (x > a ? x : a);
                }
                sb[j] = (pool == FKO_POOL_MEAN_QK) ? a / (float)G : a;
            }
            fko_pool_means(sb, 1, n_off, n_sink, n_off, pooled);
            free(sb);
        }
    }
    int cnt = fko_topk(pooled, n_sink, n_off, K, sel);
    if (pooled_out)
        for (int j = n_sink; j < n_off; ++j) pooled_out[j] = pooled[j];
    free(s);
    free(pooled);
    return cnt;
}

int fko_pool_correct_v(const float* C, int G, float tau, int mode, int cpool, float* cbar) {
    if (cpool == 0) return fko_pool_correct(C, G, tau, mode, cbar);
    float mn = C[0];
    for (int g = 1; g < G; ++g)
        if (C[g] < mn) mn = C[g];
    if (cbar) *cbar = mn;
    if (mode == FKO_MODE_ALWAYS || tau >= 1.0f) return 1;
    if (mode == FKO_MODE_NEVER || tau <= 0.0f) return 0;
    return mn < tau;
}

float fko_cosine(const uint16_t* a, const uint16_t* b, int d) {
    float dot = 0.0f, n1 = 0.0f, n2 = 0.0f;
    for (int c = 0; c < d; ++c) {
        float x = fko_bf16_to_f32(a[c]), y = fko_bf16_to_f32(b[c]);
        dot = dot + x * y;
        n1 = n1 + x * x;
        n2 = n2 + y * y;
    }
    if (n1 == 0.0f || n2 == 0.0f) return 0.0f; /* A-14 */
    float den = sqrtf(n1) * sqrtf(n2);
    return dot / den;
}

int fko_pool_correct(const float* C, int G, float tau, int mode, float* cbar) {
    float acc = C[0];
    for (int g = 1; g < G; ++g) acc = acc + C[g];
    float mean = acc / (float)G;
    if (cbar) *cbar = mean;
    if (mode == FKO_MODE_ALWAYS || tau >= 1.0f) return 1;
    if (mode == FKO_MODE_NEVER || tau <= 0.0f) return 0;
    return mean < tau;
}

int fko_correct_unit(const uint16_t* q, const uint16_t* q_prev, int G, int d,
                     float tau, int mode, int bootstrap, float* cbar) {
    float C[256];
    for (int g = 0; g < G; ++g) C[g] = fko_cosine(q + (size_t)g * d, q_prev + (size_t)g * d, d);
    int flag = fko_pool_correct(C, G, tau, mode, cbar);
    if (bootstrap) return 1; /* A-12: step 0 is synchronous */
    return flag;
}

void fko_attn_unit(const uint16_t* q, const uint16_t* Kt, const uint16_t* Vt,
                   int G, int d, const int32_t* toks, int n_tok, double* out) {
    double* l = (double*)malloc((size_t)(n_tok > 0 ? n_tok : 1) * sizeof(double));
    double inv = 1.0 / sqrt((double)d);
    for (int g = 0; g < G; ++g) {
        const uint16_t* qg = q + (size_t)g * d;
        double* o = out + (size_t)g * d;
        for (int c = 0; c < d; ++c) o[c] = 0.0;
        if (n_tok == 0) continue;
        double m = -INFINITY;
        for (int i = 0; i < n_tok; ++i) {
            const uint16_t* k = Kt + (size_t)toks[i] * d;
            double dot = 0.0;
            for (int c = 0; c < d; ++c) dot += (double)fko_bf16_to_f32(qg[c]) * (double)fko_bf16_to_f32(k[c]);
            l[i] = dot * inv;
            if (l[i] > m) m = l[i];
        }
        double Z = 0.0;
        for (int i = 0; i < n_tok; ++i) {
            l[i] = exp(l[i] - m);
            Z += l[i];
        }
        for (int i = 0; i < n_tok; ++i) {
            const uint16_t* v = Vt + (size_t)toks[i] * d;
            double w = l[i] / Z;
            for (int c = 0; c < d; ++c) o[c] += w * (double)fko_bf16_to_f32(v[c]);
        }
    }
    free(l);
}

void fko_select_batch(int n_units, const uint16_t* q, const uint16_t* const* summ, int G, int d,
                      int n_sink, const int32_t* n_off, int K, int32_t* sel) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int u = 0; u < n_units; ++u)
        fko_select_unit(q + (size_t)u * G * d, summ[u], G, d, n_sink, n_off[u], K,
                        sel + (size_t)u * K, NULL);
}

void fko_attn_batch(int n_units, const uint16_t* q, const uint16_t* const* Kt,
                    const uint16_t* const* Vt, int G, int d, const int32_t* const* toks,
                    const int32_t* n_tok, double* out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int u = 0; u < n_units; ++u)
        fko_attn_unit(q + (size_t)u * G * d, Kt[u], Vt[u], G, d, toks[u], n_tok[u],
                      out + (size_t)u * G * d);
}

int fko_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
