// select_fused.cu -- rows a9 + a1 + a2 + a3 + a4 in ONE launch: a thread-block
// cluster of C CTAs per unit scores its pages, and the cluster then runs the
// per-head softmax, MeanS pooling and top-K over distributed shared memory.
//
//   a2  PAPER.md P:231: Quest channel-wise bound (reading A-1), CFR-2/3
//   a3  P:232-234: softmax per head over candidates (A-3), mean pool over the group
//   a4  P:100-101: top-K, ties -> lower page id (A-5, CFR-9); P:296 delta + slots
//   a1  P:180: group-mean cosine vs tau (CFR-10)
//   a9  P:317: fused single-token append (append_unit.cuh)
//
// Leaf (page) j of the pairwise tree of CFR-6 belongs to CTA j / ppc, thread
// (j % ppc) / lpt: thread-local trees, xor butterflies in a warp, a pairwise
// tree over the 4 warps and one over the C CTAs (rank order) reproduce the
// balanced tree over C * ppc page ids -- a zero-padded power of two >=
// next_pow2(n_off), which gives the same Z as the recipe's tree.
//
// Scores never leave the SM: each CTA streams its 32-page summary blocks
// through a per-warp ring of 4 KiB cp.async.bulk (TMA engine) chunks into
// shared memory and keeps the G x ppc scores there.  Cross-CTA steps (max, Z,
// 4 radix-select histograms, output offsets) exchange a few bytes per CTA
// through DSMEM, one cluster barrier each.
#include <cooperative_groups.h>

#include <algorithm>

#include "append_unit.cuh"

namespace cg = cooperative_groups;

namespace fkv {

namespace fused {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxK = 256;
constexpr int kChunkBytes = 4096;  // 32 pages x {min,max} x 32 channels, bf16
constexpr int kRing = 3;
constexpr int kMaxC = 16;

__device__ __forceinline__ float cexp2_cfr(float x) {  // CFR-5
    if (x < -125.0f) return 0.0f;
    const float n = rintf(x);
    const float f = __fsub_rn(x, n);
    float P = __uint_as_float(0x377FE5FEu);
    P = __fmaf_rn(P, f, __uint_as_float(0x39218489u));
    P = __fmaf_rn(P, f, __uint_as_float(0x3AAEC3FFu));
    P = __fmaf_rn(P, f, __uint_as_float(0x3C1D955Bu));
    P = __fmaf_rn(P, f, __uint_as_float(0x3D635847u));
    P = __fmaf_rn(P, f, __uint_as_float(0x3E75FDF0u));
    P = __fmaf_rn(P, f, __uint_as_float(0x3F317218u));
    P = __fmaf_rn(P, f, __uint_as_float(0x3F800000u));
    return __uint_as_float(__float_as_uint(P) + ((uint32_t)(int)n << 23));
}

// CFR-2 over 32 channels (chunk c4 of 4) of one page: u = fma(q_c, m_c, u), m_c = max if
// q_c >= 0 else min, channels ascending.  blk: the chunk in shared memory.
template <int GM>
__device__ __forceinline__ void score_chunk(const uint4* blk, int chunk, int lane, const float (*qv)[GM],
                                            const uint32_t (*qm)[GM], int G, float (&acc)[GM]) {
#pragma unroll 2
    for (int c8 = 0; c8 < 4; ++c8) {
        const uint4 mn4 = blk[(c8 * 2 + 0) * 32 + lane];
        const uint4 mx4 = blk[(c8 * 2 + 1) * 32 + lane];
        const uint32_t mnw[4] = {mn4.x, mn4.y, mn4.z, mn4.w};
        const uint32_t mxw[4] = {mx4.x, mx4.y, mx4.z, mx4.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int c = chunk * 32 + c8 * 8 + 2 * w + half;
                const uint32_t mnb = half ? (mnw[w] & 0xffff0000u) : (mnw[w] << 16);
                const uint32_t mxb = half ? (mxw[w] & 0xffff0000u) : (mxw[w] << 16);
#pragma unroll
                for (int h = 0; h < GM; ++h) {
                    if (h < G) {
                        const uint32_t mk = qm[c][h];
                        acc[h] = __fmaf_rn(qv[c][h], __uint_as_float((mxb & mk) | (mnb & ~mk)), acc[h]);
                    }
                }
            }
        }
    }
}

template <typename T>
__device__ __forceinline__ T* peer(cg::cluster_group& cl, T* p, int rank) {
    return cl.map_shared_rank(p, rank);
}

// grid = U * C CTAs, cluster (C, 1, 1); LPTM: max leaves per thread (ppc <= 128 * LPTM)
template <int GM, int LPTM>
__global__ void __launch_bounds__(kThreads) fkv_select_kernel(FkvDims D, FkvLayer L, FkvScratch X,
                                                             const uint16_t* __restrict__ q,
                                                             const uint16_t* __restrict__ k_new,
                                                             const uint16_t* __restrict__ v_new,
                                                             int32_t* __restrict__ pages_out,
                                                             uint8_t* __restrict__ corrected_out) {
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks();
    const int r = (int)cl.block_rank();
    const int u = blockIdx.x / C, b = u / D.n_kv, m = u % D.n_kv, G = D.G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_sink = D.n_sink, K = D.K;

    extern __shared__ __align__(128) uint8_t s_dyn[];
    // dynamic: [warps][kRing][4 KiB] TMA ring | [GM][128 * LPTM] scores | page staging (CTA 0 append)
    uint8_t* s_ring = s_dyn;
    float* s_sc = reinterpret_cast<float*>(s_dyn + kWarps * kRing * kChunkBytes);
    uint4* s_page = reinterpret_cast<uint4*>(s_dyn + kWarps * kRing * kChunkBytes + GM * 128 * LPTM * 4);
    __shared__ __align__(16) float qv[kHeadDim][GM];
    __shared__ __align__(16) uint32_t qm[kHeadDim][GM];
    __shared__ __align__(8) uint64_t bar[kWarps][kRing];
    __shared__ float s_wred[kWarps][GM];
    __shared__ float s_cmax[GM], s_cz[GM];  // this CTA's partials (read by peers)
    __shared__ int s_hist[2][256];           // this CTA's histograms (read by peers)
    __shared__ int s_tot[256];
    __shared__ int s_dig, s_abv;
    __shared__ unsigned s_wsum[kWarps];
    __shared__ unsigned s_ccnt;              // this CTA's packed (gt, eq) count (read by peers)
    __shared__ int s_sel[kMaxK];             // CTA 0: the selection (written by every CTA)
    __shared__ float s_cos[kMaxG];
    __shared__ uint32_t s_qa[kMaxG * kHeadDim / 2], s_qb[kMaxG * kHeadDim / 2];
    __shared__ int s_res[kMaxK], s_res_slot[kMaxK], s_isfetch[kMaxK], s_pslot[kMaxK];
    __shared__ int s_free[2 * kMaxK];
    __shared__ unsigned char s_used[2 * kMaxK];
    __shared__ int s_flag;

    if (tid == 0 && r == 0) trace_stamp(X.trace, 1, u, 0);
    // ---- frontier of this step (the fused append adds the current token)
    const int ctx0 = L.ctx[u];
    const int Lc_now = ctx0 + (k_new ? 1 : 0);
    const int n_off = max(L.n_off[u], frontier_for(D, Lc_now));
    const int n_cand = n_off - n_sink;
    const bool rank_all = n_cand <= K;  // A-11: all candidates selected, no ranking
    int P2 = 1;
    while (P2 < n_off) P2 <<= 1;
    const int ppc = max(kThreads, P2 / C);  // pages per CTA (power of two)
    const int lpt = ppc / kThreads;         // leaves per thread (<= LPTM, checked on the host)
    const int j0 = r * ppc;                 // first page id of this CTA
    const int jb = j0 + tid * lpt;          // first leaf of this thread

    // ---- stage q (+/- masks) of the group; TMA ring prologue
    if (!rank_all) {
        for (int i = tid; i < GM * kHeadDim; i += kThreads) {
            const int h = i / kHeadDim, c = i % kHeadDim;
            float x = 0.0f;
            if (h < G) x = bf16f(q[((size_t)b * D.n_qo + m * G + h) * kHeadDim + c]);
            qv[c][h] = x;
            qm[c][h] = x >= 0.0f ? 0xffffffffu : 0u;  // CFR-2: q_c >= 0 (incl. -0) uses the max
        }
    }
    // candidate 32-page blocks of this CTA, round-robin over warps
    const int blk_lo = max(j0, n_sink) >> 5, blk_hi = (min(j0 + ppc, n_off) + 31) >> 5;
    const int nb_cta = rank_all ? 0 : max(0, blk_hi - blk_lo);
    const int nb_w = nb_cta > warp ? (nb_cta - warp + kWarps - 1) / kWarps : 0;  // blocks of this warp
    const int nch = nb_w * 4;                                                    // chunks of this warp
    uint8_t* ring = s_ring + warp * (kRing * kChunkBytes);
    auto chunk_src = [&](int k) {
        const int blk = blk_lo + warp + (k >> 2) * kWarps;
        return reinterpret_cast<const uint8_t*>(L.summ + summ_chunk_offset(D, u, blk * 32, 0, 0)) +
               (k & 3) * kChunkBytes;
    };
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kRing; ++i) mbar_init(&bar[warp][i], 1);
        fence_mbar_init();
        for (int k = 0; k < kRing && k < nch; ++k) {
            mbar_expect_tx(&bar[warp][k], kChunkBytes);
            bulk_g2s(ring + k * kChunkBytes, chunk_src(k), kChunkBytes, &bar[warp][k]);
        }
    }
    // ---- CTA 0: fused append of this step's token (row a9) and the correction inputs
    if (r == 0) {
        if (k_new) append_unit(D, L, u, ctx0, k_new, v_new, 1, s_page);  // ctx/n_off published at the end
        const uint32_t* qa32 = reinterpret_cast<const uint32_t*>(q + ((size_t)b * D.n_qo + m * G) * kHeadDim);
        const uint32_t* qb32 = reinterpret_cast<const uint32_t*>(L.q_prev + ((size_t)b * D.n_qo + m * G) * kHeadDim);
        for (int i = tid; i < G * kHeadDim / 2; i += kThreads) {
            s_qa[i] = qa32[i];
            s_qb[i] = qb32[i];
        }
    }
    for (int i = tid; i < 256; i += kThreads) s_hist[0][i] = 0;
    __syncthreads();

    // ---- a2: scoring, thread per page, all heads per thread
    for (int bi = 0; bi < nb_w; ++bi) {
        float acc[GM];
#pragma unroll
        for (int h = 0; h < GM; ++h) acc[h] = 0.0f;
        for (int c4 = 0; c4 < 4; ++c4) {
            const int k = bi * 4 + c4, slot = k % kRing;
            mbar_wait(&bar[warp][slot], (uint32_t)(k / kRing) & 1u);
            score_chunk<GM>(reinterpret_cast<const uint4*>(ring + slot * kChunkBytes), c4, lane, qv, qm, G, acc);
            __syncwarp();
            if (lane == 0 && k + kRing < nch) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bar[warp][slot], kChunkBytes);
                bulk_g2s(ring + slot * kChunkBytes, chunk_src(k + kRing), kChunkBytes, &bar[warp][slot]);
            }
        }
        const int j = (blk_lo + warp + bi * kWarps) * 32 + lane;
        if (j >= n_sink && j < n_off) {
#pragma unroll
            for (int h = 0; h < GM; ++h)
                if (h < G) s_sc[h * ppc + (j - j0)] = __fmul_rn(acc[h], D.score_r);  // CFR-3
        }
    }
    __syncthreads();
    if (tid == 0 && r == 0) trace_stamp(X.trace, 1, u, 1);

    // ---- a1: correction (CFR-10), CTA 0 lanes 0..G-1 of the last warp, 4 chunks of 32
    // channels interleaved with the radix passes
    const bool cos_lane = r == 0 && warp == kWarps - 1 && lane < G;
    float c_dot = 0.0f, c_n1 = 0.0f, c_n2 = 0.0f;
    auto cos_chunk = [&](int part) {
        const uint16_t* qa = reinterpret_cast<const uint16_t*>(s_qa) + lane * kHeadDim;
        const uint16_t* qb = reinterpret_cast<const uint16_t*>(s_qb) + lane * kHeadDim;
#pragma unroll 8
        for (int c = part * 32; c < part * 32 + 32; ++c) {
            const float x = bf16f(qa[c]), y = bf16f(qb[c]);
            c_dot = __fmaf_rn(x, y, c_dot);  // exact product, one rounding = fl(dot + x*y)
            c_n1 = __fmaf_rn(x, x, c_n1);
            c_n2 = __fmaf_rn(y, y, c_n2);
        }
        if (part == 3)
            s_cos[lane] = (c_n1 == 0.0f || c_n2 == 0.0f)
                              ? 0.0f
                              : __fdiv_rn(c_dot, __fmul_rn(__fsqrt_rn(c_n1), __fsqrt_rn(c_n2)));
    };

    int cnt = 0;
    if (rank_all) {
        if (r == 0) {
            for (int i = tid; i < K; i += kThreads) s_sel[i] = i < n_cand ? n_sink + i : -1;
            if (cos_lane)
                for (int part = 0; part < 4; ++part) cos_chunk(part);
        }
        cnt = n_cand > 0 ? n_cand : 0;
    } else {
        auto is_cand = [&](int j) { return j >= n_sink && j < n_off; };
        // ---- CFR-4: max per head (order-free): thread -> warp -> CTA -> cluster
        float M[GM];
#pragma unroll
        for (int g = 0; g < GM; ++g) {
            M[g] = -INFINITY;
            for (int l = 0; l < lpt; ++l)
                if (g < G && is_cand(jb + l)) M[g] = fmaxf(M[g], s_sc[g * ppc + tid * lpt + l]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int g = 0; g < GM; ++g) M[g] = fmaxf(M[g], __shfl_xor_sync(0xffffffffu, M[g], o));
        if (lane == 0)
#pragma unroll
            for (int g = 0; g < GM; ++g) s_wred[warp][g] = M[g];
        __syncthreads();
        if (tid < GM) {
            float v = s_wred[0][tid];
            for (int w = 1; w < kWarps; ++w) v = fmaxf(v, s_wred[w][tid]);
            s_cmax[tid] = v;
        }
        cl.sync();
#pragma unroll
        for (int g = 0; g < GM; ++g) {
            float v = -INFINITY;
            for (int rr = 0; rr < C; ++rr) v = fmaxf(v, *peer(cl, &s_cmax[g], rr));
            M[g] = v;
        }
        // ---- CFR-5/6: e = cexp2(s - m); Z = pairwise tree over page ids
        float Z[GM];
#pragma unroll
        for (int g = 0; g < GM; ++g) {
            float e[LPTM];
#pragma unroll
            for (int l = 0; l < LPTM; ++l)
                e[l] = (l < lpt && g < G && is_cand(jb + l)) ? cexp2_cfr(__fsub_rn(s_sc[g * ppc + tid * lpt + l], M[g]))
                                                             : 0.0f;
#pragma unroll
            for (int w = 1; w < LPTM; w <<= 1)
#pragma unroll
                for (int l = 0; l < LPTM; l += 2 * w) e[l] = __fadd_rn(e[l], e[l + w]);  // leaves >= lpt are +0
            Z[g] = e[0];
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
#pragma unroll
            for (int g = 0; g < GM; ++g) Z[g] = __fadd_rn(Z[g], __shfl_xor_sync(0xffffffffu, Z[g], o));
        __syncthreads();  // s_wred reuse
        if (lane == 0)
#pragma unroll
            for (int g = 0; g < GM; ++g) s_wred[warp][g] = Z[g];
        __syncthreads();
        if (tid < GM) s_cz[tid] = __fadd_rn(__fadd_rn(s_wred[0][tid], s_wred[1][tid]),
                                            __fadd_rn(s_wred[2][tid], s_wred[3][tid]));
        cl.sync();
#pragma unroll
        for (int g = 0; g < GM; ++g) {
            float z[kMaxC];
#pragma unroll
            for (int rr = 0; rr < kMaxC; ++rr) z[rr] = rr < C ? *peer(cl, &s_cz[g], rr) : 0.0f;
#pragma unroll
            for (int w = 1; w < kMaxC; w <<= 1)
#pragma unroll
                for (int l = 0; l < kMaxC; l += 2 * w) z[l] = __fadd_rn(z[l], z[l + w]);
            Z[g] = z[0];
        }
        // ---- CFR-7/8/9: p = e / Z, pooled = sequential sum over g, keys
        uint32_t key[LPTM];
        bool cand[LPTM];
#pragma unroll
        for (int l = 0; l < LPTM; ++l) {
            const int j = jb + l;
            cand[l] = l < lpt && is_cand(j);
            float pi = 0.0f;
            if (cand[l]) {
#pragma unroll
                for (int g = 0; g < GM; ++g) {
                    if (g < G) {
                        const float pg = __fdiv_rn(cexp2_cfr(__fsub_rn(s_sc[g * ppc + tid * lpt + l], M[g])), Z[g]);
                        pi = g == 0 ? pg : __fadd_rn(pi, pg);
                    }
                }
            }
            const uint32_t kk = __float_as_uint(pi);
            key[l] = kk == 0x80000000u ? 0u : kk;
        }
        if (tid == 0 && r == 0) trace_stamp(X.trace, 1, u, 2);
        // ---- radix select of the K-th largest key over the cluster (4 x 8-bit passes)
        uint32_t prefix = 0u, mask = 0u;
        int k_rem = K;
#pragma unroll 1
        for (int pass = 0; pass < 4; ++pass) {
            const int shift = 24 - 8 * pass;
            int* H = s_hist[pass & 1];
#pragma unroll
            for (int l = 0; l < LPTM; ++l) {
                const int dg = (cand[l] && (key[l] & mask) == prefix) ? (int)((key[l] >> shift) & 255u) : -1;
                const unsigned grp = __match_any_sync(0xffffffffu, dg);
                if (dg >= 0 && lane == __ffs(grp) - 1) atomicAdd(&H[dg], __popc(grp));
            }
            cl.sync();
            for (int i = tid; i < 256; i += kThreads) {
                int v = 0;
                for (int rr = 0; rr < C; ++rr) v += peer(cl, H, rr)[i];
                s_tot[i] = v;
                s_hist[(pass + 1) & 1][i] = 0;  // peers finished with it before this pass's barrier
            }
            __syncthreads();
            if (cos_lane) cos_chunk(pass);
            if (warp == 0) {
                int bins[8], lsum = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    bins[i] = s_tot[lane * 8 + i];
                    lsum += bins[i];
                }
                int suf = lsum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_down_sync(0xffffffffu, suf, o);
                    if (lane + o < 32) suf += y;
                }
                int above = suf - lsum;
#pragma unroll
                for (int i = 7; i >= 0; --i) {
                    if (above < k_rem && above + bins[i] >= k_rem) {
                        s_dig = lane * 8 + i;
                        s_abv = above;
                    }
                    above += bins[i];
                }
            }
            __syncthreads();
            k_rem -= s_abv;
            prefix |= (uint32_t)s_dig << shift;
            mask |= 0xFFu << shift;
            __syncthreads();  // s_dig / s_abv reuse
        }
        const uint32_t T = prefix;  // K-th largest key; k_rem keys equal to T are taken (lowest ids)
        // ---- output positions: packed (#gt, #eq) scans in page-id order, thread -> CTA -> cluster
        unsigned n_gt = 0, n_eq = 0;
#pragma unroll
        for (int l = 0; l < LPTM; ++l) {
            n_gt += cand[l] && key[l] > T;
            n_eq += cand[l] && key[l] == T;
        }
        const unsigned mine = (n_gt << 16) | n_eq;
        unsigned x = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wsum[warp] = x;
        __syncthreads();
        unsigned woff = 0;
        for (int w = 0; w < warp; ++w) woff += s_wsum[w];
        if (tid == 0) s_ccnt = s_wsum[0] + s_wsum[1] + s_wsum[2] + s_wsum[3];
        cl.sync();
        unsigned coff = 0;
        for (int rr = 0; rr < r; ++rr) coff += *peer(cl, &s_ccnt, rr);
        const unsigned ex = coff + woff + x - mine;
        int gt_before = (int)(ex >> 16), eq_before = (int)(ex & 0xffffu);
        int* sel0 = peer(cl, s_sel, 0);
#pragma unroll
        for (int l = 0; l < LPTM; ++l) {
            if (!cand[l]) continue;
            const bool gt = key[l] > T, eq = key[l] == T;
            if (gt || (eq && eq_before < k_rem)) sel0[gt_before + min(eq_before, k_rem)] = jb + l;
            gt_before += gt;
            eq_before += eq;
        }
        cnt = K;
    }
    cl.sync();  // the selection is complete in CTA 0's s_sel; nobody touches peer memory after this
    if (r != 0) return;
    if (tid == 0) {
        trace_stamp(X.trace, 1, u, 3);
        if (k_new) {  // every CTA of the cluster has read ctx / n_off by now
            L.ctx[u] = Lc_now;
            L.n_off[u] = n_off;
        }
    }

    // ---- CTA 0: flag, delta vs resident, slots, fetch list, page list (as select.cu)
    const int res_valid = D.full_refresh ? 0 : L.res_valid[u];
    const int res_front = L.res_front[u], res_cnt = L.res_cnt[u];
    for (int i = tid; i < K; i += kThreads) {
        s_res[i] = res_valid ? L.res_pages[(size_t)u * K + i] : -1;
        s_res_slot[i] = res_valid ? L.res_slot[(size_t)u * K + i] : -1;
        if (i >= cnt) s_sel[i] = -1;
    }
    for (int i = tid; i < 2 * K; i += kThreads) s_used[i] = 0;
    __syncthreads();
    if (tid == 0) {
        float acc = s_cos[0];
        for (int g = 1; g < G; ++g) acc = __fadd_rn(acc, s_cos[g]);
        const float mean = __fdiv_rn(acc, (float)G);
        int flag;
        if (D.mode == 1 || D.tau >= 1.0f) flag = 1;
        else if (D.mode == 2 || D.tau <= 0.0f) flag = 0;
        else flag = mean < D.tau;
        if (!res_valid) flag = 1;
        s_flag = flag;
        L.flags[u] = (uint8_t)flag;
        L.cbar[u] = mean;
        L.pend_front[u] = n_off;
        if (corrected_out) corrected_out[u] = (uint8_t)flag;
    }
    // membership of S_i in R via a page -> index table in the (now dead) TMA ring, 24 K
    // entries >= n_page_max (checked on the host); entries are validated against s_res
    uint16_t* s_idx = reinterpret_cast<uint16_t*>(s_ring);
    for (int i = tid; i < K; i += kThreads)
        if (s_res[i] >= 0) s_idx[s_res[i]] = (uint16_t)i;
    __syncthreads();
    for (int a = tid; a < K; a += kThreads) {
        int f = 0;
        const int Sa = s_sel[a];
        if (Sa >= 0) {
            f = 1;
            const int i = s_idx[Sa];
            if (i < K && s_res[i] == Sa) {
                f = 0;
                s_pslot[a] = s_res_slot[i];
            }
        } else {
            s_pslot[a] = -1;
        }
        s_isfetch[a] = f;
        if (s_res[a] >= 0) s_used[s_res_slot[a]] = 1;
        L.pend_pages[(size_t)u * K + a] = Sa;
        if (pages_out) pages_out[(size_t)u * K + a] = Sa;
    }
    __syncthreads();
    if (warp == 0) {
        int nfree = 0;
        for (int base = 0; base < 2 * K; base += 32) {
            const int sl = base + lane;
            const bool fr = sl < 2 * K && !s_used[sl];
            const unsigned bal = __ballot_sync(0xffffffffu, fr);
            if (fr) s_free[nfree + __popc(bal & ((1u << lane) - 1u))] = sl;
            nfree += __popc(bal);
        }
        __syncwarp();
        int nf = 0;
        for (int base = 0; base < K; base += 32) {
            const int a = base + lane;
            const bool fe = a < K && s_isfetch[a];
            const unsigned bal = __ballot_sync(0xffffffffu, fe);
            if (fe) {
                const int rr = nf + __popc(bal & ((1u << lane) - 1u));
                const int slot = s_free[rr];
                s_pslot[a] = slot;
                L.fetch_page[(size_t)u * K + rr] = s_sel[a];
                L.fetch_slot[(size_t)u * K + rr] = slot;
            }
            nf += __popc(bal);
        }
        if (lane == 0) {
            L.n_fetch[u] = nf;
            L.pend_cnt[u] = cnt;
        }
    }
    __syncthreads();
    for (int i = tid; i < K; i += kThreads) L.pend_slot[(size_t)u * K + i] = s_pslot[i];
    // this step's attention page list (row a7): sink pages, pages in use (S_i if corrected,
    // the resident set otherwise), local pages [f*p, Lc) (reading A-9)
    {
        const int flag = s_flag;
        const int Lc = Lc_now, p = D.p;
        const int sink_tok = min(D.S_tok, Lc);
        const int n_sp = (sink_tok + p - 1) / p;
        const int n_sel = flag ? cnt : res_cnt;
        const int f = flag ? n_off : res_front;
        const int n_last = (Lc - 1) / p;
        const int n_loc = (Lc > f * p) ? (n_last - f + 1) : 0;
        const size_t pe = page_elems(D);
        const int total = n_sp + n_sel + n_loc;
        for (int i = tid; i < total; i += kThreads) {
            const uint16_t* base;
            int valid;
            if (i < n_sp) {
                base = L.sink + ((size_t)u * D.n_sink + i) * pe;
                valid = min(p, sink_tok - i * p);
            } else if (i < n_sp + n_sel) {
                const int a = i - n_sp;
                const int slot = flag ? s_pslot[a] : s_res_slot[a];
                base = L.slots + ((size_t)u * 2 * K + slot) * pe;
                valid = p;
            } else {
                const int j = f + (i - n_sp - n_sel);
                base = L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe;
                valid = min(p, Lc - j * p);
            }
            X.page_rows[(size_t)u * D.P_max + i] = (int)((base - L.arena) / kHeadDim);
            X.page_valid[(size_t)u * D.P_max + i] = (uint8_t)valid;
        }
        if (tid == 0) X.page_cnt[u] = total;
    }
    if (tid == 0) trace_stamp(X.trace, 1, u, 4);
}

}  // namespace fused

template <int GM, int LPTM>
static cudaError_t launch_sel(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              const uint16_t* k_new, const uint16_t* v_new, int32_t* pages_out,
                              uint8_t* corrected_out, int C, cudaStream_t s) {
    const size_t smem = (size_t)fused::kWarps * fused::kRing * fused::kChunkBytes + (size_t)GM * 128 * LPTM * 4 +
                        page_elems(D) * sizeof(uint16_t);
    auto kern = fused::fkv_select_kernel<GM, LPTM>;
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.U * C, 1, 1);
    cfg.blockDim = dim3(fused::kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, D, L, X, q, k_new, v_new, pages_out, corrected_out);
}

// cluster = C CTAs per unit; lptm >= max(128, P2max / C) / 128 for the handle's largest frontier.
cudaError_t launch_select_fused(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                const uint16_t* k_new, const uint16_t* v_new, int32_t* pages_out,
                                uint8_t* corrected_out, int cluster, int lptm, cudaStream_t s) {
    const int gm = D.G <= 1 ? 1 : (D.G <= 2 ? 2 : (D.G <= 4 ? 4 : 8));
#define FKV_SEL(GMV, LV)                                                                                     \
    if (gm == GMV && lptm == LV)                                                                             \
        return launch_sel<GMV, LV>(D, L, X, q, k_new, v_new, pages_out, corrected_out, cluster, s);
    FKV_SEL(1, 1) FKV_SEL(1, 2) FKV_SEL(1, 4) FKV_SEL(1, 8)
    FKV_SEL(2, 1) FKV_SEL(2, 2) FKV_SEL(2, 4) FKV_SEL(2, 8)
    FKV_SEL(4, 1) FKV_SEL(4, 2) FKV_SEL(4, 4) FKV_SEL(4, 8)
    FKV_SEL(8, 1) FKV_SEL(8, 2) FKV_SEL(8, 4) FKV_SEL(8, 8)
#undef FKV_SEL
    return cudaErrorInvalidValue;
}

}  // namespace fkv
