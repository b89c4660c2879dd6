// select.cu -- rows a1-a4: correction check, page scoring, MeanS pooling,
// top-K and delta vs the resident set.
//
//   fkv_score_kernel          a2  PAPER.md P:231 (Quest-style min-max summaries,
//                                 reading A-1); CFR-2/3
//   fkv_select_finalize_kernel a1  P:180, P:247-250 (group-mean cosine vs tau; CFR-10)
//                              a3  P:232-234 (softmax per head over candidates,
//                                 mean pooling over the group; CFR-4..8)
//                              a4  P:100-101 (top-K, ties -> lower id; CFR-9),
//                                 P:296 (cache of selected pages: delta + slots)
//
// Every floating-point step that decides an index follows the canonical fp32
// recipe with explicit round-to-nearest intrinsics, so the page
// indices are bit-identical to the CPU oracle.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "append_unit.cuh"

namespace cg = cooperative_groups;

namespace fkv {

// ---------------------------------------------------------------- CFR-5
__device__ __forceinline__ float cexp2_cfr(float x) {
    if (x < -125.0f) return 0.0f;
    const float n = rintf(x);          // ties-to-even
    const float f = __fsub_rn(x, n);   // exact
    float P = __uint_as_float(0x377FE5FEu);
    P = __fmaf_rn(P, f, __uint_as_float(0x39218489u));
    P = __fmaf_rn(P, f, __uint_as_float(0x3AAEC3FFu));
    P = __fmaf_rn(P, f, __uint_as_float(0x3C1D955Bu));
    P = __fmaf_rn(P, f, __uint_as_float(0x3D635847u));
    P = __fmaf_rn(P, f, __uint_as_float(0x3E75FDF0u));
    P = __fmaf_rn(P, f, __uint_as_float(0x3F317218u));
    P = __fmaf_rn(P, f, __uint_as_float(0x3F800000u));
    const int ni = (int)n;
    return __uint_as_float(__float_as_uint(P) + ((uint32_t)ni << 23));
}

// Group pooling of the heads' cosines (CFR-10): 0 = mean (sequential sum / G, FreeKV);
// 1 = minimum, the "max pooling over group C_i" of tab:abl-g-corr (reading R-11)
__device__ __forceinline__ float pool_cos(const float* c, int G, int corr_pool) {
    float acc = c[0];
    for (int g = 1; g < G; ++g) acc = corr_pool ? (c[g] < acc ? c[g] : acc) : __fadd_rn(acc, c[g]);
    return corr_pool ? acc : __fdiv_rn(acc, (float)G);
}

// ----------------------------------------------------------- a2: scoring
constexpr int kScoreWarps = 4;
constexpr int kSummBlockBytes = 32 * 2 * kHeadDim * 2;  // 16 KiB: 32 pages x {min,max} x 128 ch

// CFR-2 per channel c and head h: u = fma(q_c, m_c, u) with m_c = mx_c if q_c >= 0 else
// mn_c (exact product, one rounding -- exactly the recipe's fl(u + t)).  The select is a
// LOP3 on a precomputed sign mask, so each head's dependent chain is one FMA per channel.
template <int G>
__device__ __forceinline__ void score_channels(const uint4* blk, int c8_begin, int lane,
                                               const float (*qv)[(G + 3) / 4 * 4],
                                               const uint32_t (*qm)[(G + 3) / 4 * 4], float (&acc)[G]) {
    constexpr int GP = (G + 3) / 4 * 4;
#pragma unroll 2
    for (int c8 = c8_begin; c8 < c8_begin + 4; ++c8) {
        const uint4 mn4 = blk[(c8 * 2 + 0) * 32 + lane];
        const uint4 mx4 = blk[(c8 * 2 + 1) * 32 + lane];
        const uint32_t mnw[4] = {mn4.x, mn4.y, mn4.z, mn4.w};
        const uint32_t mxw[4] = {mx4.x, mx4.y, mx4.z, mx4.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int c = c8 * 8 + 2 * w + half;
                const uint32_t mnb = half ? (mnw[w] & 0xffff0000u) : (mnw[w] << 16);
                const uint32_t mxb = half ? (mxw[w] & 0xffff0000u) : (mxw[w] << 16);
#pragma unroll
                for (int h4 = 0; h4 < GP; h4 += 4) {
                    const float4 q4 = *reinterpret_cast<const float4*>(&qv[c][h4]);
                    const uint4 m4 = *reinterpret_cast<const uint4*>(&qm[c][h4]);
                    const float qq[4] = {q4.x, q4.y, q4.z, q4.w};
                    const uint32_t mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (h4 + e < G) {
                            const float sel = __uint_as_float((mxb & mm[e]) | (mnb & ~mm[e]));
                            acc[h4 + e] = __fmaf_rn(qq[e], sel, acc[h4 + e]);
                        }
                    }
                }
            }
        }
    }
}

// Even G: the same recipe with the select folded into the arithmetic and two heads per
// instruction.  With q+ = max(q, 0), q- = min(q, 0): u = fma(q-_c, mn_c, fma(q+_c, mx_c, u)) --
// one product is a signed zero, so each step is CFR-2's single rounding (equal up to the sign
// of zero, which CFR-2 allows) -- evaluated for heads (h, h+1) at once with FFMA2
// (fma.rn.f32x2, sm_100a).  qp/qn hold q+ / q- per channel and head.
template <int G>
__device__ __forceinline__ void score_channels_x2(const uint4* blk, int c8_begin, int lane,
                                                  const float (*qp)[(G + 3) / 4 * 4],
                                                  const float (*qn)[(G + 3) / 4 * 4],
                                                  unsigned long long (&acc2)[G / 2]) {
#pragma unroll 2
    for (int c8 = c8_begin; c8 < c8_begin + 4; ++c8) {
        const uint4 mn4 = blk[(c8 * 2 + 0) * 32 + lane];
        const uint4 mx4 = blk[(c8 * 2 + 1) * 32 + lane];
        const uint32_t mnw[4] = {mn4.x, mn4.y, mn4.z, mn4.w};
        const uint32_t mxw[4] = {mx4.x, mx4.y, mx4.z, mx4.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int c = c8 * 8 + 2 * w + half;
                const uint32_t mnb = half ? (mnw[w] & 0xffff0000u) : (mnw[w] << 16);
                const uint32_t mxb = half ? (mxw[w] & 0xffff0000u) : (mxw[w] << 16);
                unsigned long long mx2, mn2;
                asm("mov.b64 %0, {%1, %1};" : "=l"(mx2) : "r"(mxb));
                asm("mov.b64 %0, {%1, %1};" : "=l"(mn2) : "r"(mnb));
#pragma unroll
                for (int k = 0; k < G / 2; ++k) {
                    const unsigned long long p2 = *reinterpret_cast<const unsigned long long*>(&qp[c][2 * k]);
                    const unsigned long long n2 = *reinterpret_cast<const unsigned long long*>(&qn[c][2 * k]);
                    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[k]) : "l"(p2), "l"(mx2));
                    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[k]) : "l"(n2), "l"(mn2));
                }
            }
        }
    }
}

// Thread per page, warp per 32-page summary block, CTA = 4 consecutive blocks of
// one unit (so q is staged once per CTA).  Each warp streams its 16 KiB block
// through a 3-slot ring of 4 KiB chunks (4 channel-groups of 32 channels) filled
// by cp.async.bulk (TMA engine) with mbarrier completion: chunks k+1, k+2 are in
// flight while chunk k is scored.  12 KiB per warp keeps 4 CTAs (16 warps) per
// SM resident, so the dependent FMA chains of many warps interleave.
constexpr int kChunkBytes = kSummBlockBytes / 4;  // channels [32k, 32k+32) of 32 pages, {min,max}
constexpr int kRing = 3;

// pending = 1 when this step's token is appended later in the step (fused into the
// finalize kernel): the frontier is then that of ctx + 1.  Offload at page
// completion (append_unit.cuh) guarantees the candidate summaries already exist.
template <int G>
__global__ void __launch_bounds__(kScoreWarps * 32, 4) fkv_score_kernel(FkvDims D, FkvLayer L,
                                                                        float* __restrict__ scores,
                                                                        const uint16_t* __restrict__ q, int pending,
                                                                        unsigned long long* __restrict__ trace,
                                                                        int which, int gy,
                                                                        const uint16_t* __restrict__ k_new,
                                                                        const uint16_t* __restrict__ v_new,
                                                                        float* __restrict__ cosv) {
    // k_new != NULL: the unit's last-scoring CTA also appends this step's token (row a9) and
    // runs the correction check (row a1, CFR-10 -> cosv[u][g]) after its scoring, so the
    // select kernel starts on the scores directly; ctx / n_off are published by the select
    constexpr int GP = (G + 3) / 4 * 4;
    extern __shared__ __align__(128) uint8_t s_raw[];
    __shared__ __align__(16) float qv[kHeadDim][GP];      // q_c per head
    __shared__ __align__(16) uint32_t qm[kHeadDim][GP];   // ~0 if q_c >= 0 (take max) else 0 (take min)
    __shared__ __align__(8) uint64_t bar[kScoreWarps][kRing];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tcls = 0;  // trace class
    uint8_t* ring = s_raw + warp * (kRing * kChunkBytes);
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < kRing; ++r) mbar_init(&bar[warp][r], 1);
        fence_mbar_init();
    }
    uint32_t ph = 0u;  // per-slot parity of this warp's next completion (slots are reused across items)
    // items (unit, 128-page block): one per CTA, or a grid-stride loop over all of them when the
    // grid is smaller (the background score runs on a bounded number of CTAs)
    for (int item = blockIdx.x; item < D.U * gy; item += gridDim.x) {
        const int u = item / gy, yb = item - u * gy, b = u / D.n_kv, m = u % D.n_kv;
        const int ctx0 = L.ctx[u];
        const int n_off = max(L.n_off[u], frontier_for(D, ctx0 + pending));
        // with k_new the grid has one extra CTA per unit (yb == gy - 1), which only does a1 + a9
        const bool pre_cta = k_new && yb == gy - 1;
        if (yb * kScoreWarps * 32 >= n_off && !pre_cta) continue;  // uniform: no candidate in this item
        __syncthreads();  // the previous item's q staging is no longer read
        const int blk = yb * kScoreWarps + warp;
        const bool active = !pre_cta && blk * 32 < n_off && blk * 32 + 31 >= D.n_sink;
        const int tent = item;
        if (threadIdx.x == 0) trace_stamp(trace, tcls, tent, 0);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(L.summ + summ_chunk_offset(D, u, blk * 32, 0, 0));
        if (lane == 0 && active) {
#pragma unroll
            for (int k = 0; k < kRing; ++k) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bar[warp][k], kChunkBytes);
                bulk_g2s(ring + k * kChunkBytes, src + k * kChunkBytes, kChunkBytes, &bar[warp][k]);
            }
        }
        // q_i is this layer's input: with PDL the kernel may start while the previous layer's
        // last kernel drains; everything above (state and summaries of this layer) is independent
        pdl_wait();
        pdl_trigger();  // dependents launch once the previous layer is complete (see the select)
        for (int i = threadIdx.x; i < GP * kHeadDim; i += blockDim.x) {
            const int h = i / kHeadDim, c = i % kHeadDim;
            float x = 0.0f;
            if (h < G) {
                const uint16_t* qc = q + ((size_t)b * D.n_qo + m * G) * kHeadDim + c;
                if (D.pool >= 4) {  // MeanQ / MaxQ (f3): every head scores the group's pooled query
                    float a = bf16f(qc[0]);
                    for (int g = 1; g < G; ++g) {
                        const float y = bf16f(qc[(size_t)g * kHeadDim]);
                        a = D.pool == 4 ? __fadd_rn(a, y) : (y > a ? y : a);
                    }
                    x = D.pool == 4 ? __fdiv_rn(a, (float)G) : a;
                } else {
                    x = bf16f(qc[(size_t)h * kHeadDim]);
                }
            }
            if (G % 2 == 0) {  // FFMA2 form: q+ / q- (qm holds q- as float bits)
                qv[c][h] = x >= 0.0f ? x : 0.0f;
                qm[c][h] = __float_as_uint(x >= 0.0f ? 0.0f : x);
            } else {
                qv[c][h] = x;
                qm[c][h] = x >= 0.0f ? 0xffffffffu : 0u;  // CFR-2: q_c >= 0 (incl. -0) uses the max
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) trace_stamp(trace, tcls, tent, 1);
        if (active) {
        float acc[G];
#pragma unroll
        for (int h = 0; h < G; ++h) acc[h] = 0.0f;
        unsigned long long acc2[G / 2 > 0 ? G / 2 : 1];
#pragma unroll
        for (int k = 0; k < (G / 2 > 0 ? G / 2 : 1); ++k) acc2[k] = 0ull;
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
            const int slot = k % kRing;
            mbar_wait(&bar[warp][slot], (ph >> slot) & 1u);
            ph ^= 1u << slot;
            if (k == 0 && threadIdx.x == 0) trace_stamp(trace, tcls, tent, 2);
            if constexpr (G % 2 == 0)
                score_channels_x2<G>(reinterpret_cast<const uint4*>(ring + slot * kChunkBytes) - (k * 4) * 2 * 32,
                                     k * 4, lane, qv, reinterpret_cast<const float(*)[(G + 3) / 4 * 4]>(qm), acc2);
            else
                score_channels<G>(reinterpret_cast<const uint4*>(ring + slot * kChunkBytes) - (k * 4) * 2 * 32, k * 4,
                                  lane, qv, qm, acc);
            if (k + kRing < 4) {
                __syncwarp();  // all lanes are done with this slot
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&bar[warp][slot], kChunkBytes);
                    bulk_g2s(ring + slot * kChunkBytes, src + (k + kRing) * kChunkBytes, kChunkBytes,
                             &bar[warp][slot]);
                }
            }
        }
        __syncwarp();  // every lane is done with the ring before the next item refills it
        if constexpr (G % 2 == 0) {
#pragma unroll
            for (int k2 = 0; k2 < G / 2; ++k2) {
                uint32_t lo, hi;
                asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(acc2[k2]));
                acc[2 * k2] = __uint_as_float(lo);
                acc[2 * k2 + 1] = __uint_as_float(hi);
            }
        }
        const int j = blk * 32 + lane;
        if (j >= D.n_sink && j < n_off) {
#pragma unroll
            for (int h = 0; h < G; ++h)
                scores[((size_t)u * G + h) * D.n_page_max + j] = __fmul_rn(acc[h], D.score_r);  // CFR-3
        }
        }  // active
        if (pre_cta) {
            // rows a1 + a9 for the unit, on this CTA's now idle ring as the page staging
            if (threadIdx.x < G) {
                const size_t row = ((size_t)b * D.n_qo + m * G + threadIdx.x) * kHeadDim;
                cosv[(size_t)u * kMaxG + threadIdx.x] = cos_cfr10(q + row, L.q_prev + row);
            }
            __syncthreads();  // every warp is done with the ring
            append_unit(D, L, u, ctx0, k_new, v_new, 1, reinterpret_cast<uint4*>(s_raw));
        }
        if (threadIdx.x == 0) trace_stamp(trace, tcls, tent, 3);
    }
}

// ------------------------------------------------------ a9 + a1 + a3 + a4
// One 512-thread CTA per unit.  Leaf (page) j of the pairwise tree (CFR-6) is
// owned by thread j / LPT, so thread-local trees + an xor butterfly inside a warp
// + the same butterfly over the 32 warp partials reproduce the balanced tree
// over page ids exactly.  Cross-warp reductions are re-done redundantly by every
// warp from shared memory (no second barrier); the radix select double-buffers
// its histogram (2 barriers per 8-bit pass) with warp-aggregated atomics; one
// packed (gt, eq) block scan places the selected ids in ascending order.
constexpr int kMaxK = 256;
constexpr int kHistBins = 4096;

// The resident set of unit u as one thread (tid < K: entry tid) loaded it earlier, e.g. in the
// fused select's prologue before the PDL wait (R is state, untouched by this step's kernels).
struct ResPre {
    int have = 0;
    int valid = 0, front = 0, cnt = 0, page = -1, slot = -1;
};

template <int LPT, int GM, int NT>
__device__ __forceinline__ void finalize_unit(const int u, const FkvDims& D, const FkvLayer& L,
                                              int32_t* __restrict__ page_rows, uint8_t* __restrict__ page_valid,
                                              int32_t* __restrict__ page_dst, int32_t* __restrict__ page_cnt,
                                              unsigned long long* __restrict__ trace,
                                              const float* __restrict__ scores, const uint16_t* __restrict__ q,
                                              const uint16_t* __restrict__ k_new,
                                              const uint16_t* __restrict__ v_new, int32_t* __restrict__ pages_out,
                                              uint8_t* __restrict__ corrected_out, int which,
                                              const float* ssc = nullptr, const float* cos_in = nullptr,
                                              uint64_t* cos_bar = nullptr, int lc_in = -1, int noff_in = -1,
                                              ResPre pre = ResPre(), int appended = 0) {
    // appended: the score kernel has appended this step's token and written the cosines
    // (cos_in, global); this kernel publishes ctx / n_off
    // cos_bar != NULL: cos_in is written later by the helper CTA; wait on this mbarrier
    // (phase 0) before reading it.  lc_in / noff_in >= 0: this step's context and frontier
    // (the helper publishes them to global memory after its append, possibly later)
    // ssc != NULL: the scores are already in shared memory ([G][n_page_max], fused select);
    // cos_in != NULL (fused select, which == 0): the helper CTA has done the correction check
    // (cos_in = per-head cosines in this CTA's shared memory) and the append of this step's token
    constexpr int kThreads = NT, kWarps = NT / 32;
    const int b = u / D.n_kv, m = u % D.n_kv, G = D.G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_sink = D.n_sink, K = D.K;

    __shared__ float s_redm[kWarps][kMaxG], s_redz[kWarps][kMaxG];
    __shared__ float s_cos[kMaxG];
    __shared__ __align__(16) int s_h[kHistBins];           // radix histogram
    __shared__ __align__(16) int s_sup[kHistBins / 32];    // its sums over 32-bin groups
    __shared__ int s_dig[4], s_abv[4];
    __shared__ uint32_t s_bk[32];  // boundary-bin keys and ids
    __shared__ int s_bid[32], s_bn;
    __shared__ unsigned s_wsum[kWarps];
    __shared__ int s_sel[kMaxK];
    __shared__ int s_res[kMaxK], s_res_slot[kMaxK];
    __shared__ int s_isfetch[kMaxK];
    __shared__ int s_pslot[kMaxK];
    __shared__ int s_flag;
    __shared__ int s_free[2 * kMaxK];
    __shared__ unsigned char s_used[2 * kMaxK];
    __shared__ __align__(16) uint32_t s_qa[kMaxG * kHeadDim / 2], s_qb[kMaxG * kHeadDim / 2];
    extern __shared__ __align__(16) uint8_t s_dyn[];
    uint4* s_page = reinterpret_cast<uint4*>(s_dyn);                                   // append staging
    uint16_t* s_idx = reinterpret_cast<uint16_t*>(s_dyn + page_elems(D) * sizeof(uint16_t));  // [n_page_max]

    // which: 0 = flags computed here (primitive API / sequential step); 3 = flags from the prep
    // kernel (overlapped step: the page lists of the units that attend their resident set were
    // built by the prep kernel and are being read while this kernel runs -- only the corrected
    // units' lists are written here)
    const int tcls = 1;  // trace class
    if (tid == 0) trace_stamp(trace, tcls, u, 0);
    const int pre_flag = which ? (int)L.flags[u] : 0;
    int n_off = noff_in >= 0 ? noff_in : L.n_off[u];
    const int ctx0 = lc_in >= 0 ? lc_in : L.ctx[u];
    const int Lc_now = ctx0 + ((k_new || appended) ? 1 : 0);
    if (k_new || appended) n_off = max(n_off, frontier_for(D, Lc_now));
    const int n_cand = n_off - n_sink;
    const bool rank_all = n_cand <= K;  // A-11: all candidates selected, no ranking
    if (tid == 0) trace_stamp(trace, tcls, u, 1);

    // ---- a1: correction (CFR-10), which == 0 only: lanes 0..G-1 of the last warp run the
    // sequential channel sums before the scores arrive
    const bool cos_lane = which == 0 && warp == kWarps - 1 && lane < G && !(D.dbg & 1);
    auto cos_all = [&]() {
        s_cos[lane] = cos_cfr10(reinterpret_cast<const uint16_t*>(s_qa) + lane * kHeadDim,
                                reinterpret_cast<const uint16_t*>(s_qb) + lane * kHeadDim);
    };

    // ---- stage the state this CTA reads (one round trip): resident set.  Step inputs (q_i,
    // the new token) are read only after pdl_wait(): with PDL this kernel may start before
    // the previous layer's last kernel has completed (its prologue overlaps it)
    // debug mode 3 (FREEKV_DEBUG_FULL_REFRESH): forget the resident set every step, so every
    // unit re-fetches all K pages synchronously -- the GEN-X recall-bandwidth stress case
    const int res_valid = pre.have ? pre.valid : (D.full_refresh ? 0 : L.res_valid[u]);
    const int res_front = pre.have ? pre.front : L.res_front[u];  // hoisted: used by the page list at the end
    const int res_cnt = pre.have ? pre.cnt : L.res_cnt[u];
    for (int i = tid; i < K; i += kThreads) {
        const bool mine = pre.have && i == tid;
        s_res[i] = res_valid ? (mine ? pre.page : L.res_pages[(size_t)u * K + i]) : -1;
        s_res_slot[i] = res_valid ? (mine ? pre.slot : L.res_slot[(size_t)u * K + i]) : -1;
    }
    for (int i = tid; i < 2 * K; i += kThreads) s_used[i] = 0;
    for (int i = tid; i < kHistBins; i += kThreads) s_h[i] = 0;
    for (int i = tid; i < kHistBins / 32; i += kThreads) s_sup[i] = 0;
    if (tid == 0) s_bn = 0;
    const size_t srow = (size_t)D.n_page_max;
    __syncthreads();  // staging visible
    // the resident set's page -> index table and used-slot map (no scores needed)
    if (tid < K && s_res[tid] >= 0) {
        s_idx[s_res[tid]] = (uint16_t)tid;
        s_used[s_res_slot[tid]] = 1;
    }
    pdl_wait();  // the previous kernel (score) has completed: scores and step inputs are ready
    pdl_trigger();  // the attention may launch (and read q_i, attend speculatively) from here on
    // ---- step inputs: q_i, q_{i-1} (correction check), and the fused append (row a9) of this
    // step's token -- it only touches the ring / the page completing now (not a candidate of
    // this step) / the host pool
    if (cos_in) {
        if (!cos_bar && tid < G) s_cos[tid] = cos_in[tid];  // visible to warp 0 after the barriers below
        if (appended && tid == 0) {
            L.ctx[u] = Lc_now;
            L.n_off[u] = n_off;
        }
    } else {
        if (which == 0) {
            const uint32_t* qa32 = reinterpret_cast<const uint32_t*>(q + ((size_t)b * D.n_qo + m * G) * kHeadDim);
            const uint32_t* qb32 =
                reinterpret_cast<const uint32_t*>(L.q_prev + ((size_t)b * D.n_qo + m * G) * kHeadDim);
            for (int i = tid; i < G * kHeadDim / 2; i += kThreads) {
                s_qa[i] = qa32[i];
                s_qb[i] = qb32[i];
            }
        }
        if (k_new) {
            append_unit(D, L, u, ctx0, k_new, v_new, 1, s_page);
            if (tid == 0) {
                L.ctx[u] = Lc_now;
                L.n_off[u] = n_off;
            }
        }
        if (which == 0) {
            __syncthreads();  // s_qa / s_qb staged
            if (cos_lane) cos_all();
        }
    }
    // ---- work of the last warp that needs no selection, done in the shadow of the ranking:
    // the correction flag (CFR-10 pooling, A-12, A-13) and the free-slot list (slots of R are
    // used, the others free; slot double-buffering)
    __shared__ int s_nfree;
    const int cnt_final = rank_all ? (n_cand > 0 ? n_cand : 0) : K;
    auto early_tail = [&]() {
        if (lane == 0) {
            if (which) {
                s_flag = pre_flag;  // decided by the prep kernel (same CFR-10 arithmetic)
            } else {
                if (cos_bar) {  // the helper's cosines arrive over DSMEM with a remote mbarrier arrive
                    asm volatile(
                        "{\n.reg .pred P1;\nWAIT_C_%=:\n"
                        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], 0;\n"
                        "@!P1 bra WAIT_C_%=;\n}\n" ::"r"(smem_u32(cos_bar))
                        : "memory");
                    for (int g = 0; g < G; ++g) s_cos[g] = cos_in[g];
                }
                const float mean = pool_cos(s_cos, G, D.corr_pool);
                int flag;
                if (D.mode == 1 || D.tau >= 1.0f) flag = 1;
                else if (D.mode == 2 || D.tau <= 0.0f) flag = 0;
                else flag = mean < D.tau;
                if (!res_valid) flag = 1;
                s_flag = flag;
                L.flags[u] = (uint8_t)flag;
                L.cbar[u] = mean;
                if (corrected_out) corrected_out[u] = (uint8_t)flag;
            }
            L.pend_front[u] = n_off;
            L.pend_cnt[u] = cnt_final;
        }
        int nfree = 0;
        for (int base = 0; base < 2 * K; base += 32) {
            const int sl = base + lane;
            const bool fr = sl < 2 * K && !s_used[sl];
            const unsigned bal = __ballot_sync(0xffffffffu, fr);
            if (fr) s_free[nfree + __popc(bal & ((1u << lane) - 1u))] = sl;
            nfree += __popc(bal);
        }
        if (lane == 0) s_nfree = nfree;
    };
    int cnt;
    if (rank_all) {
        for (int i = tid; i < K; i += kThreads) s_sel[i] = i < n_cand ? n_sink + i : -1;
        cnt = n_cand > 0 ? n_cand : 0;
        __syncthreads();
        if (warp == kWarps - 1) early_tail();
        __syncthreads();  // s_free / s_flag ready for warp 0's delta
    } else {
        if (tid == 0) trace_stamp(trace, tcls, u, 2);
        const int jb = tid * LPT;
        // this thread's leaves, straight from global memory into registers (no staging pass)
        const float* sg = scores + (size_t)u * G * srow;
        bool cand[LPT];
        float sv[GM][LPT];
#pragma unroll
        for (int l = 0; l < LPT; ++l) cand[l] = jb + l >= n_sink && jb + l < n_off;
#pragma unroll
        for (int g = 0; g < GM; ++g)
#pragma unroll
            for (int l = 0; l < LPT; ++l)
                sv[g][l] = (g < G && cand[l]) ? (ssc ? ssc[g * srow + jb + l] : sg[g * srow + jb + l]) : -INFINITY;
        // group-consistency variants (f3): QK pools the heads' scores into head 0; Q pools
        // the queries before scoring (every head then holds the same scores); both use one softmax
        const int Gs = D.pool >= 2 ? 1 : G;
        if (D.pool == 2 || D.pool == 3) {
#pragma unroll
            for (int l = 0; l < LPT; ++l) {
                float a = sv[0][l];
#pragma unroll
                for (int g = 1; g < GM; ++g)
                    if (g < G) a = D.pool == 2 ? __fadd_rn(a, sv[g][l]) : (sv[g][l] > a ? sv[g][l] : a);
                if (cand[l]) sv[0][l] = D.pool == 2 ? __fdiv_rn(a, (float)G) : a;
            }
        }
        // ---- CFR-4: max per head (exact, order-free): one warp-wide redux per head, twice
        float M[GM];
#pragma unroll
        for (int g = 0; g < GM; ++g) {
            M[g] = sv[g][0];
#pragma unroll
            for (int l = 1; l < LPT; ++l) M[g] = fmaxf(M[g], sv[g][l]);
            M[g] = warp_max_f32(M[g]);
        }
        if (lane == 0)
#pragma unroll
            for (int g = 0; g < GM; ++g) s_redm[warp][g] = M[g];
        __syncthreads();
        if (warp == kWarps - 1) early_tail();
#pragma unroll
        for (int g = 0; g < GM; ++g) M[g] = warp_max_f32(lane < kWarps ? s_redm[lane][g] : -INFINITY);
        // ---- CFR-5/6: e = cexp2(s - m); Z = pairwise tree in page-id order: thread-local tree over
        // its LPT contiguous leaves, xor butterfly over the 32 lanes, butterfly over the warp
        // partials (lanes >= kWarps hold +0 leaves, which leave a pairwise tree's value unchanged)
        float Z[GM];
#pragma unroll
        for (int g = 0; g < GM; ++g) {
#pragma unroll
            for (int l = 0; l < LPT; ++l)
                sv[g][l] = (g < Gs && cand[l]) ? cexp2_cfr(__fsub_rn(sv[g][l], M[g])) : 0.0f;  // sv := e
            float t[LPT];
#pragma unroll
            for (int l = 0; l < LPT; ++l) t[l] = sv[g][l];
#pragma unroll
            for (int w = 1; w < LPT; w <<= 1)
#pragma unroll
                for (int l = 0; l < LPT; l += 2 * w) t[l] = __fadd_rn(t[l], t[l + w]);
            Z[g] = t[0];
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
#pragma unroll
            for (int g = 0; g < GM; ++g) Z[g] = __fadd_rn(Z[g], __shfl_xor_sync(0xffffffffu, Z[g], o));
        if (lane == 0)
#pragma unroll
            for (int g = 0; g < GM; ++g) s_redz[warp][g] = Z[g];
        __syncthreads();
#pragma unroll
        for (int g = 0; g < GM; ++g) Z[g] = lane < kWarps ? s_redz[lane][g] : 0.0f;
        // the warp partials occupy lanes [0, kWarps): log2(kWarps) butterfly levels build their
        // pairwise tree (the padded lanes would only add +0)
#pragma unroll
        for (int o = 1; o < kWarps; o <<= 1)
#pragma unroll
            for (int g = 0; g < GM; ++g) Z[g] = __fadd_rn(Z[g], __shfl_xor_sync(0xffffffffu, Z[g], o));
        if (kWarps < 32)
#pragma unroll
            for (int g = 0; g < GM; ++g) Z[g] = __shfl_sync(0xffffffffu, Z[g], 0);
        if (tid == 0) trace_stamp(trace, tcls, u, 3);
        // ---- CFR-7/8: p = e / Z; pooled = sequential sum over g; CFR-9 keys
        uint32_t key[LPT];
#pragma unroll
        for (int l = 0; l < LPT; ++l) {
            float pi = 0.0f;
            if (cand[l]) {
#pragma unroll
                for (int g = 0; g < GM; ++g) {
                    if (g < Gs) {
                        const float pg = (D.dbg & 4) ? sv[g][l] * (1.0f / Z[g]) : __fdiv_rn(sv[g][l], Z[g]);
                        // CFR-8 (MeanS: sequential sum) or MaxS
                        pi = g == 0 ? pg : (D.pool == 1 ? (pg > pi ? pg : pi) : __fadd_rn(pi, pg));
                    }
                }
            }
            const uint32_t kk = __float_as_uint(pi);
            key[l] = kk == 0x80000000u ? 0u : kk;
        }
        // ---- exact K-th largest key: radix passes of 12, 12 and 8 bits; as soon as the boundary
        // bin holds <= 32 keys, one warp ranks them directly (usually after the first pass)
        uint32_t prefix = 0u, mask = 0u;
        int k_rem = K;
        uint32_t T = 0u;
        bool resolved = false;
#pragma unroll 1
        for (int pass = 0; pass < 3; ++pass) {
            const int shift = pass == 0 ? 20 : (pass == 1 ? 8 : 0);
            const int nbits = pass == 2 ? 8 : 12;
            const uint32_t dmask = (1u << nbits) - 1u;
            if (tid == 0) trace_stamp(trace, 11, u, pass);  // diagnostics: radix passes taken
            if (pass > 0) {  // fallback passes (rare): clear the histogram first
                __syncthreads();
                for (int i = tid; i < kHistBins; i += kThreads) s_h[i] = 0;
                for (int i = tid; i < kHistBins / 32; i += kThreads) s_sup[i] = 0;
                __syncthreads();
            }
            // plain shared atomics (match.any aggregation measured ~18x slower on B200)
#pragma unroll
            for (int l = 0; l < LPT; ++l) {
                if (cand[l] && (key[l] & mask) == prefix) {
                    const int dg = (int)((key[l] >> shift) & dmask);
                    atomicAdd(&s_h[dg], 1);
                    atomicAdd(&s_sup[dg >> 5], 1);
                }
            }
            __syncthreads();
            if (warp == 0) {
                // level 1: 32-bin groups (lane owns up to 4 contiguous groups, one conflict-free
                // 16-byte load); level 2: the 32 bins of the boundary group, one per lane
                const int nsup = (int)(dmask + 1u) >> 5;  // 128 or 8
                int4 c4 = make_int4(0, 0, 0, 0);
                if (nsup == 128) {
                    c4 = *reinterpret_cast<const int4*>(&s_sup[lane * 4]);
                } else if (lane < nsup) {
                    c4.x = s_sup[lane];  // one group per lane, in c4.x
                }
                const int s4 = c4.x + c4.y + c4.z + c4.w;
                int suf = s4;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_down_sync(0xffffffffu, suf, o);
                    if (lane + o < 32) suf += y;
                }
                int a = suf - s4;  // keys in groups of higher lanes
                int grp = 0;
                if (a < k_rem && a + s4 >= k_rem) {  // exactly one lane
                    if (nsup == 128) {
                        if (a + c4.w >= k_rem) {
                            grp = 3;
                        } else if ((a += c4.w) + c4.z >= k_rem) {
                            grp = 2;
                        } else if ((a += c4.z) + c4.y >= k_rem) {
                            grp = 1;
                        } else {
                            a += c4.y;
                            grp = 0;
                        }
                        grp += lane * 4;
                    } else {
                        grp = lane;
                    }
                }
                const unsigned hit = __ballot_sync(0xffffffffu, a < k_rem && a + s4 >= k_rem);
                const int hl = __ffs(hit) - 1;
                grp = __shfl_sync(0xffffffffu, grp, hl);
                const int above_g = __shfl_sync(0xffffffffu, a, hl);
                const int cb = s_h[grp * 32 + lane];
                int suf2 = cb;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_down_sync(0xffffffffu, suf2, o);
                    if (lane + o < 32) suf2 += y;
                }
                const int ab = above_g + suf2 - cb;  // keys in higher bins
                if (ab < k_rem && ab + cb >= k_rem) {
                    s_dig[0] = grp * 32 + lane;
                    s_abv[0] = ab;
                    s_dig[1] = cb;
                }
            }
            __syncthreads();
            k_rem -= s_abv[0];
            prefix |= (uint32_t)s_dig[0] << shift;
            mask |= dmask << shift;
            if (pass == 2) {  // every bit fixed: T = prefix, take k_rem of the keys equal to it
                T = prefix;
                resolved = true;
                break;
            }
            if (s_dig[1] <= 32) break;
        }
        if (tid == 0) trace_stamp(trace, tcls, u, 4);
        if (!resolved) {
            // the boundary bin's (key, id) pairs (<= 32) -> one warp ranks them exactly (ties -> lower id)
#pragma unroll
            for (int l = 0; l < LPT; ++l) {
                if (cand[l] && (key[l] & mask) == prefix) {
                    const int at = atomicAdd(&s_bn, 1);
                    s_bk[at] = key[l];
                    s_bid[at] = jb + l;
                }
            }
            __syncthreads();
            if (warp == 0) {
                const int n = s_bn;
                const uint32_t mk = lane < n ? s_bk[lane] : 0u;
                const int mi = lane < n ? s_bid[lane] : 0x7fffffff;
                int rank = 0, gt = 0;
                for (int i = 0; i < n; ++i) {
                    const uint32_t ok = __shfl_sync(0xffffffffu, mk, i);
                    const int oi = __shfl_sync(0xffffffffu, mi, i);
                    rank += (ok > mk || (ok == mk && oi < mi)) ? 1 : 0;
                    gt += ok > mk ? 1 : 0;
                }
                // the k_rem-th largest of the bin is the threshold; keys above it in the bin are taken
                if (lane < n && rank == k_rem - 1) {
                    s_dig[2] = (int)mk;
                    s_abv[2] = k_rem - gt;
                }
            }
            __syncthreads();
            T = (uint32_t)s_dig[2];
            k_rem = s_abv[2];
        }
        // ---- one packed block scan of (#gt, #eq) in page-id order
        unsigned n_gt = 0, n_eq = 0;
#pragma unroll
        for (int l = 0; l < LPT; ++l) {
            n_gt += cand[l] && key[l] > T;
            n_eq += cand[l] && key[l] == T;
        }
        unsigned x = (n_gt << 16) | n_eq;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wsum[warp] = x;
        __syncthreads();
        unsigned woff = 0;
        {
            const unsigned ws = lane < warp ? s_wsum[lane] : 0u;
            woff = ws;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) woff += __shfl_xor_sync(0xffffffffu, woff, o);
        }
        const unsigned ex = woff + x - ((n_gt << 16) | n_eq);
        int gt_before = (int)(ex >> 16), eq_before = (int)(ex & 0xffffu);
#pragma unroll
        for (int l = 0; l < LPT; ++l) {
            if (!cand[l]) continue;
            const bool gt = key[l] > T, eq = key[l] == T;
            if (gt || (eq && eq_before < k_rem)) s_sel[gt_before + min(eq_before, k_rem)] = jb + l;
            gt_before += gt;
            eq_before += eq;
        }
        for (int i = tid + K; i < kMaxK; i += kThreads) s_sel[i] = -1;
        cnt = K;
        __syncthreads();
    }

    // ---- flag (CFR-10 pooling, A-12, A-13) and a4: delta vs resident (A-18) + slot assignment
    // (slot double-buffering), warp-synchronous in warp 0: membership of S_i's pages in R via
    // the page -> index table built before the scores arrived (entries validated against s_res)
    if (tid == 0) trace_stamp(trace, tcls, u, 5);
    if (warp == 0) {
        int nf = 0;
        for (int base = 0; base < K; base += 32) {
            const int a = base + lane;
            int fe = 0, slot = -1;
            const int Sa = (a < K && a < cnt) ? s_sel[a] : -1;
            if (Sa >= 0) {
                fe = 1;
                const int i = s_idx[Sa];
                if (i < K && s_res[i] == Sa) {
                    fe = 0;
                    slot = s_res_slot[i];
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, fe);
            if (fe) {
                const int r = nf + __popc(bal & ((1u << lane) - 1u));
                slot = s_free[r];
                L.fetch_page[(size_t)u * K + r] = Sa;
                L.fetch_slot[(size_t)u * K + r] = slot;
            }
            nf += __popc(bal);
            if (a < K) {
                s_isfetch[a] = fe;
                s_pslot[a] = slot;
                L.pend_pages[(size_t)u * K + a] = Sa;
                L.pend_slot[(size_t)u * K + a] = slot;
                if (pages_out) pages_out[(size_t)u * K + a] = Sa;
            }
        }
        if (lane == 0) L.n_fetch[u] = nf;
    }
    __syncthreads();
    if (tid == 0) trace_stamp(trace, tcls, u, 7);
    // ---- this step's attention page list (row a7), one entry per page: arena row of the
    // page's K block and its valid tokens -- sink pages, the pages in use (S_i if corrected,
    // the resident set otherwise), local pages [f*p, Lc) (reading A-9)
    if (which == 0 || s_flag) {
        const int flag = s_flag;
        const int Lc = Lc_now;
        const int p = D.p;
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
                if (flag && D.direct && s_isfetch[a]) {
                    // direct mode: the attention reads this page from the host pool and writes it
                    // back into its slot (bit 7 of page_valid marks a host row)
                    const int j = s_sel[a];
                    page_rows[(size_t)u * D.P_max + i] =
                        L.host_row0 + (int)((((size_t)b * D.n_page_host + j) * D.n_kv + m) * 2 * p);
                    page_valid[(size_t)u * D.P_max + i] = (uint8_t)(p | 0x80);
                    page_dst[(size_t)u * D.P_max + i] = (int)((base - L.arena) / kHeadDim);
                    continue;
                }
            } else {
                const int j = f + (i - n_sp - n_sel);
                base = L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe;
                valid = min(p, Lc - j * p);
            }
            const int row = (int)((base - L.arena) / kHeadDim);
            page_rows[(size_t)u * D.P_max + i] = row;
            page_valid[(size_t)u * D.P_max + i] = (uint8_t)valid;
        }
        if (tid == 0) page_cnt[u] = total;
    }
    if (tid == 0) trace_stamp(trace, tcls, u, 6);
}

// One unit per CTA (the loop also serves smaller grids).
template <int LPT, int GM, int NT>
__global__ void __launch_bounds__(NT) fkv_select_finalize_kernel(FkvDims D, FkvLayer L,
                                                                       int32_t* __restrict__ page_rows,
                                                                       uint8_t* __restrict__ page_valid,
                                                                       int32_t* __restrict__ page_dst,
                                                                       int32_t* __restrict__ page_cnt,
                                                                       unsigned long long* __restrict__ trace,
                                                                       const float* __restrict__ scores,
                                                                       const uint16_t* __restrict__ q,
                                                                       const uint16_t* __restrict__ k_new,
                                                                       const uint16_t* __restrict__ v_new,
                                                                       int32_t* __restrict__ pages_out,
                                                                       uint8_t* __restrict__ corrected_out,
                                                                       int which, const float* __restrict__ cosv) {
    // cosv != NULL: the score kernel appended the token and wrote the cosines ([U][kMaxG])
    for (int u = blockIdx.x; u < D.U; u += gridDim.x) {
        finalize_unit<LPT, GM, NT>(u, D, L, page_rows, page_valid, page_dst, page_cnt, trace, scores, q,
                                   cosv ? nullptr : k_new, cosv ? nullptr : v_new, pages_out, corrected_out, which,
                                   nullptr, cosv ? cosv + (size_t)u * kMaxG : nullptr, nullptr, -1, -1, ResPre(),
                                   cosv ? 1 : 0);
        __syncthreads();  // shared state of this unit is dead before the next unit reuses it
    }
}

// ------------------------------------------------- pipelined step prologue
// One CTA per unit, first kernel of a layer's decode step in the pipelined mode
// (DESIGN.md §5): append this step's token (row a9), the correction check (row
// a1, CFR-10 -- the same arithmetic as the select kernel's), and, for units that
// are not corrected, this step's attention page list over the resident set R
// (speculative units attend the pages selected at step i-1).  The
// selection of step i then runs off the critical path for those units.
constexpr int kPrepThreads = 256;

__global__ void __launch_bounds__(kPrepThreads) fkv_prep_kernel(FkvDims D, FkvLayer L, FkvScratch X,
                                                                const uint16_t* __restrict__ q,
                                                                const uint16_t* __restrict__ k_new,
                                                                const uint16_t* __restrict__ v_new,
                                                                uint8_t* __restrict__ corrected_out) {
    extern __shared__ __align__(16) uint8_t s_dyn[];  // append staging: one (2, p, d) page
    __shared__ __align__(16) uint32_t s_qa[kMaxG * kHeadDim / 2], s_qb[kMaxG * kHeadDim / 2];
    __shared__ float s_cos[kMaxG];
    __shared__ int s_flag;
    const int u = blockIdx.x, b = u / D.n_kv, m = u % D.n_kv, G = D.G, tid = threadIdx.x;
    if (tid == 0) trace_stamp(X.trace, 8, u, 0);
    // state loads first (with PDL they overlap the previous layer's last kernel) ...
    const int L0 = L.ctx[u];
    int n_off = L.n_off[u];
    const int res_valid = D.full_refresh ? 0 : L.res_valid[u];
    const int res_front = L.res_front[u], res_cnt = L.res_cnt[u];
    const int my_slot = tid < D.K ? L.res_slot[(size_t)u * D.K + tid] : 0;
    pdl_wait();  // ... step inputs (q_i, the new token) only after the previous layer has completed
    pdl_trigger();
    {
        const uint32_t* qa32 = reinterpret_cast<const uint32_t*>(q + ((size_t)b * D.n_qo + m * G) * kHeadDim);
        const uint32_t* qb32 = reinterpret_cast<const uint32_t*>(L.q_prev + ((size_t)b * D.n_qo + m * G) * kHeadDim);
        for (int i = tid; i < G * kHeadDim / 2; i += kPrepThreads) {
            s_qa[i] = qa32[i];
            s_qb[i] = qb32[i];
        }
    }
    if (k_new) append_unit(D, L, u, L0, k_new, v_new, 1, reinterpret_cast<uint4*>(s_dyn));
    const int Lc = L0 + (k_new ? 1 : 0);
    n_off = max(n_off, frontier_for(D, Lc));
    __syncthreads();
    // ---- a1 (CFR-10): head g's cosine, sequential channel sums by thread g
    if (tid < G)
        s_cos[tid] = cos_cfr10(reinterpret_cast<const uint16_t*>(s_qa) + tid * kHeadDim,
                               reinterpret_cast<const uint16_t*>(s_qb) + tid * kHeadDim);
    __syncthreads();
    // q_prev := q_i now (q_prev is read only by this check): the background select
    // of this step reads q_i from here, so the caller's q buffer may be reused at once
    {
        uint32_t* qp = reinterpret_cast<uint32_t*>(L.q_prev + ((size_t)b * D.n_qo + m * G) * kHeadDim);
        for (int i = tid; i < G * kHeadDim / 2; i += kPrepThreads) qp[i] = s_qa[i];
    }
    if (tid == 0) {
        const float mean = pool_cos(s_cos, G, D.corr_pool);
        int flag;
        if (D.mode == 1 || D.tau >= 1.0f) flag = 1;
        else if (D.mode == 2 || D.tau <= 0.0f) flag = 0;
        else flag = mean < D.tau;
        if (!res_valid) flag = 1;
        s_flag = flag;
        L.flags[u] = (uint8_t)flag;
        L.cbar[u] = mean;
        if (corrected_out) corrected_out[u] = (uint8_t)flag;
        L.ctx[u] = Lc;
        L.n_off[u] = n_off;
    }
    __syncthreads();
    if (s_flag) {  // corrected: the page list is built by the select kernel from S_i
        if (tid == 0) trace_stamp(X.trace, 8, u, 1);
        return;
    }
    // ---- page list over R: sink pages, R's slots, local pages [f_R * p, Lc) (reading A-9)
    const int p = D.p;
    const int sink_tok = min(D.S_tok, Lc);
    const int n_sp = (sink_tok + p - 1) / p;
    const int n_last = (Lc - 1) / p;
    const int n_loc = (Lc > res_front * p) ? (n_last - res_front + 1) : 0;
    const int total = n_sp + res_cnt + n_loc;
    const size_t pe = page_elems(D);
    if (tid < res_cnt) {  // R's slots (K <= 256 <= kPrepThreads)
        const uint16_t* base = L.slots + ((size_t)u * 2 * D.K + my_slot) * pe;
        X.page_rows[(size_t)u * D.P_max + n_sp + tid] = (int)((base - L.arena) / kHeadDim);
        X.page_valid[(size_t)u * D.P_max + n_sp + tid] = (uint8_t)p;
    }
    for (int i = tid; i < total; i += kPrepThreads) {
        const uint16_t* base;
        int valid;
        if (i < n_sp) {
            base = L.sink + ((size_t)u * D.n_sink + i) * pe;
            valid = min(p, sink_tok - i * p);
        } else if (i < n_sp + res_cnt) {
            continue;
        } else {
            const int j = res_front + (i - n_sp - res_cnt);
            base = L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe;
            valid = min(p, Lc - j * p);
        }
        X.page_rows[(size_t)u * D.P_max + i] = (int)((base - L.arena) / kHeadDim);
        X.page_valid[(size_t)u * D.P_max + i] = (uint8_t)valid;
    }
    if (tid == 0) {
        X.page_cnt[u] = total;
        trace_stamp(X.trace, 8, u, 1);
    }
}

cudaError_t launch_prep(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                        const uint16_t* k_new, const uint16_t* v_new, uint8_t* corrected_out, bool pdl,
                        cudaStream_t s) {
    const size_t smem = page_elems(D) * sizeof(uint16_t);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(fkv_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(fkv_prep_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    return launch_ex(fkv_prep_kernel, dim3(D.U), dim3(kPrepThreads), smem, s, pdl, D, L, X, q, k_new, v_new,
                     corrected_out);
}

template <int G>
static void launch_score_g(const FkvDims& D, const FkvLayer& L, float* scores, const uint16_t* q, int max_n_off,
                           int pending, unsigned long long* trace, int which, bool pdl, cudaStream_t s,
                           const uint16_t* k_new, const uint16_t* v_new, float* cosv) {
    const int per_cta = kScoreWarps * 32;
    const int gy = (max_n_off + per_cta - 1) / per_cta;
    if (gy <= 0 && !k_new) return;  // (with k_new the append + correction CTA still runs)
    const int smem = kScoreWarps * kRing * kChunkBytes;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(fkv_score_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(fkv_score_kernel<G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        configured = true;
    }
    const int gyl = std::max(gy, 0) + (k_new ? 1 : 0);  // + one CTA per unit for the append + correction check
    const int grid = D.U * gyl;             // one (unit, 128-page block) item per CTA
    launch_ex(fkv_score_kernel<G>, dim3(grid), dim3(per_cta), smem, s, pdl, D, L, scores, q, pending, trace, which, gyl,
              k_new, v_new, cosv);
}

cudaError_t launch_score(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                         int max_n_off, int pending, int which, bool pdl, cudaStream_t s,
                         const uint16_t* k_new, const uint16_t* v_new) {
    switch (D.G) {
        case 1: launch_score_g<1>(D, L, X.scores, q, max_n_off, pending, X.trace, which, pdl, s, k_new, v_new, X.cosv); break;
        case 2: launch_score_g<2>(D, L, X.scores, q, max_n_off, pending, X.trace, which, pdl, s, k_new, v_new, X.cosv); break;
        case 3: launch_score_g<3>(D, L, X.scores, q, max_n_off, pending, X.trace, which, pdl, s, k_new, v_new, X.cosv); break;
        case 4: launch_score_g<4>(D, L, X.scores, q, max_n_off, pending, X.trace, which, pdl, s, k_new, v_new, X.cosv); break;
        case 5: launch_score_g<5>(D, L, X.scores, q, max_n_off, pending, X.trace, which, pdl, s, k_new, v_new, X.cosv); break;
        case 6: launch_score_g<6>(D, L, X.scores, q, max_n_off, pending, X.trace, which, pdl, s, k_new, v_new, X.cosv); break;
        case 7: launch_score_g<7>(D, L, X.scores, q, max_n_off, pending, X.trace, which, pdl, s, k_new, v_new, X.cosv); break;
        case 8: launch_score_g<8>(D, L, X.scores, q, max_n_off, pending, X.trace, which, pdl, s, k_new, v_new, X.cosv); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------- fused select: score + select, 2-CTA cluster
// One cluster of two 1024-thread CTAs per unit.  Both CTAs stream half of the unit's
// candidate summary blocks through a 2-deep ring of 4 KiB chunks (16 scoring warps, chunks
// of this step in flight before the previous kernel has finished -- summaries are state,
// not step input) and score them (CFR-2/3, the same arithmetic as fkv_score_kernel) into
// the leader CTA's shared memory (DSMEM stores); after one cluster barrier the helper
// exits and the leader runs the select on the scores in shared memory.  Removes the
// score kernel's launch, its global score round trip and the score -> select boundary.
constexpr int kFusedScoreWarps = 16;
constexpr int kFusedRing = 2;

__host__ __device__ inline size_t fused_off_sc(const FkvDims& D) {
    return (page_elems(D) * 2 + (size_t)D.n_page_max * 2 + 15) / 16 * 16;
}
__host__ __device__ inline size_t fused_off_ring(const FkvDims& D) {
    return (fused_off_sc(D) + (size_t)D.G * D.n_page_max * 4 + 127) / 128 * 128;
}
__host__ __device__ inline size_t fused_smem_bytes(const FkvDims& D) {  // + kMaxG floats (helper cosines)
    return fused_off_ring(D) + (size_t)kFusedScoreWarps * kFusedRing * kChunkBytes;
}

template <int LPT, int GM, int NT, int CL>
__global__ void __launch_bounds__(NT)
    fkv_select_c2_kernel(FkvDims D, FkvLayer L, int32_t* __restrict__ page_rows, uint8_t* __restrict__ page_valid,
                         int32_t* __restrict__ page_dst, int32_t* __restrict__ page_cnt,
                         unsigned long long* __restrict__ trace, const uint16_t* __restrict__ q,
                         const uint16_t* __restrict__ k_new, const uint16_t* __restrict__ v_new,
                         int32_t* __restrict__ pages_out, uint8_t* __restrict__ corrected_out, int which) {
    constexpr int GP = (GM + 3) / 4 * 4;
    extern __shared__ __align__(16) uint8_t s_dyn[];
    __shared__ __align__(16) float qv[kHeadDim][GP];
    __shared__ __align__(16) uint32_t qm[kHeadDim][GP];
    __shared__ __align__(8) uint64_t bar[kFusedScoreWarps][kFusedRing];
    const int rank = CL == 2 ? (int)cg::this_cluster().block_rank() : 0;
    const int u = CL == 2 ? (blockIdx.x >> 1) : blockIdx.x, b = u / D.n_kv, m = u % D.n_kv, G = D.G;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    float* s_sc = reinterpret_cast<float*>(s_dyn + fused_off_sc(D));
    uint8_t* ring = s_dyn + fused_off_ring(D) + (size_t)warp * kFusedRing * kChunkBytes;
    if (tid == 0) trace_stamp(trace, 0, blockIdx.x, 0);
    // ---- this CTA's summary blocks (state: readable before pdl_wait)
    const int ctx0 = L.ctx[u];
    const int n_off = max(L.n_off[u], frontier_for(D, ctx0 + (k_new ? 1 : 0)));
    const int blk_lo = D.n_sink >> 5;
    const int nblk = n_off > D.n_sink ? ((n_off - 1) >> 5) - blk_lo + 1 : 0;
    const int half = CL == 2 ? (nblk + 1) >> 1 : nblk;
    const int my0 = rank ? half : 0, my1 = rank ? nblk : half;
    const int nmine = my1 - my0;
    // chunk c (0..) of warp w: block my0 + w + 16 * (c >> 2), channel group c & 3
    constexpr int kSW = NT / 32 < kFusedScoreWarps ? NT / 32 : kFusedScoreWarps;  // scoring warps
    const bool scorer = warp < kSW && warp < nmine;
    const int nchunks = scorer ? ((nmine - warp + kSW - 1) / kSW) * 4 : 0;
    auto chunk_src = [&](int c) {
        const int blk = blk_lo + my0 + warp + kSW * (c >> 2);
        return reinterpret_cast<const uint8_t*>(L.summ + summ_chunk_offset(D, u, blk * 32, 0, 0)) +
               (size_t)(c & 3) * kChunkBytes;
    };
    if (scorer && lane == 0) {
#pragma unroll
        for (int r = 0; r < kFusedRing; ++r) mbar_init(&bar[warp][r], 1);
        fence_mbar_init();
        for (int c = 0; c < kFusedRing && c < nchunks; ++c) {
            mbar_expect_tx(&bar[warp][c], kChunkBytes);
            bulk_g2s(ring + c * kChunkBytes, chunk_src(c), kChunkBytes, &bar[warp][c]);
        }
    }
    ResPre pre;  // the leader's resident set, loaded while the previous kernel drains
    if (rank == 0) {
        pre.have = 1;
        pre.valid = D.full_refresh ? 0 : L.res_valid[u];
        pre.front = L.res_front[u];
        pre.cnt = L.res_cnt[u];
        if (tid < D.K) {
            pre.page = L.res_pages[(size_t)u * D.K + tid];
            pre.slot = L.res_slot[(size_t)u * D.K + tid];
        }
    }
    pdl_wait();  // step inputs (q_i) are ready
    // dependents (the attention) launch only once every CTA of this kernel is past its wait:
    // the previous layer is then complete, so they may read q_i (and attend speculatively)
    pdl_trigger();
    if (tid == 0) trace_stamp(trace, 0, blockIdx.x, 1);
    float* s_cosx = reinterpret_cast<float*>(s_dyn + fused_smem_bytes(D));  // [kMaxG] helper -> leader
    // the helper CTA takes the leader's prologue work -- the correction check (CFR-10) and
    // the append of this step's token (row a9) -- after its share of the scoring, while the
    // leader runs the select; the cosines reach the leader over DSMEM with a remote arrive
    // on an mbarrier in the leader's shared memory, which it waits on just before the flag
    const bool helped = CL == 2 && which == 0 && !(D.dbg & 2);  // FREEKV_DEBUG_EXP bit 1: off (A/B)
    __shared__ __align__(8) uint64_t s_cosbar;
    if (helped && rank == 0 && tid == 0) {
        mbar_init(&s_cosbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < GP * kHeadDim; i += blockDim.x) {
        const int h = i / kHeadDim, c = i % kHeadDim;
        float x = 0.0f;
        if (h < G) x = bf16f(q[((size_t)b * D.n_qo + m * G + h) * kHeadDim + c]);
        qv[c][h] = x;
        qm[c][h] = x >= 0.0f ? 0xffffffffu : 0u;  // CFR-2: q_c >= 0 (incl. -0) uses the max
    }
    __syncthreads();
    if (tid == 0) trace_stamp(trace, 0, blockIdx.x, 2);
    float* dst_sc = s_sc;  // scores land in the leader
    if (CL == 2 && rank) dst_sc = cg::this_cluster().map_shared_rank(s_sc, 0);
    if (scorer) {
        float acc[GM];
        int cur_blk = -1;
        for (int c = 0; c < nchunks; ++c) {
            const int slot = c % kFusedRing;
            if ((c & 3) == 0) {
#pragma unroll
                for (int h = 0; h < GM; ++h) acc[h] = 0.0f;
                cur_blk = blk_lo + my0 + warp + kSW * (c >> 2);
            }
            mbar_wait(&bar[warp][slot], (uint32_t)(c / kFusedRing) & 1u);
            score_channels<GM>(reinterpret_cast<const uint4*>(ring + slot * kChunkBytes) - ((c & 3) * 4) * 2 * 32,
                               (c & 3) * 4, lane, qv, qm, acc);
            __syncwarp();  // every lane is done with this slot
            if (c + kFusedRing < nchunks && lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bar[warp][slot], kChunkBytes);
                bulk_g2s(ring + slot * kChunkBytes, chunk_src(c + kFusedRing), kChunkBytes, &bar[warp][slot]);
            }
            if ((c & 3) == 3) {
                const int j = cur_blk * 32 + lane;
                if (j >= D.n_sink && j < n_off) {
#pragma unroll
                    for (int h = 0; h < GM; ++h)
                        if (h < G) dst_sc[(size_t)h * D.n_page_max + j] = __fmul_rn(acc[h], D.score_r);  // CFR-3
                }
            }
        }
    }
    if (tid == 0) trace_stamp(trace, 0, blockIdx.x, 3);
    if (CL == 2) {
        cg::this_cluster().sync();  // every score is in the leader's shared memory
        if (tid == 0) trace_stamp(trace, 0, blockIdx.x, 4);
        if (rank) {
            if (helped) {
                if (warp == NT / 32 - 1 && lane < G) {
                    const size_t row = ((size_t)b * D.n_qo + m * G + lane) * kHeadDim;
                    *cg::this_cluster().map_shared_rank(&s_cosx[lane], 0) = cos_cfr10(q + row, L.q_prev + row);
                }
                __syncwarp();
                if (warp == NT / 32 - 1 && lane == 0) {
                    // release the DSMEM stores above, then arrive on the leader's barrier
                    const uint32_t rb = (uint32_t)__cvta_generic_to_shared(cg::this_cluster().map_shared_rank(&s_cosbar, 0));
                    asm volatile(
                        "{\n.reg .b32 ra;\n"
                        "mapa.shared::cluster.u32 ra, %0, 0;\n"
                        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(smem_u32(&s_cosbar))
                        : "memory");
                    (void)rb;
                }
                if (k_new) {
                    append_unit(D, L, u, ctx0, k_new, v_new, 1, reinterpret_cast<uint4*>(s_dyn));
                    if (tid == 0) {
                        L.ctx[u] = ctx0 + 1;
                        L.n_off[u] = n_off;
                    }
                }
            }
            return;
        }
    } else {
        __syncthreads();
    }
    // helped: the append (ctx / n_off already published, visible after the cluster barrier)
    // and the correction check were done by the helper CTA
    finalize_unit<LPT, GM, NT>(u, D, L, page_rows, page_valid, page_dst, page_cnt, trace, nullptr, q,
                               helped ? nullptr : k_new, helped ? nullptr : v_new, pages_out, corrected_out, which,
                               s_sc, helped ? s_cosx : nullptr, helped ? &s_cosbar : nullptr,
                               helped ? ctx0 + (k_new ? 1 : 0) : -1, helped ? n_off : -1, pre);
}

template <int LPT, int GM, int NT, int CL>
static cudaError_t launch_c2_g(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                               const uint16_t* k_new, const uint16_t* v_new, int32_t* pages_out,
                               uint8_t* corrected_out, bool pdl, int which, cudaStream_t s) {
    auto kern = fkv_select_c2_kernel<LPT, GM, NT, CL>;
    const size_t smem = fused_smem_bytes(D) + kMaxG * sizeof(float);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * D.U);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (CL > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CL;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, D, L, X.page_rows, X.page_valid, X.page_dst, X.page_cnt, X.trace, q, k_new,
                              v_new, pages_out, corrected_out, which);
}

// Fused score + select (2-CTA clusters).  Returns cudaErrorNotSupported when the handle's
// shapes do not fit (caller falls back to score + select).
bool select_c2_fits(const FkvDims& D, int lpt, int nt) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t static_est = 40 * 1024;  // finalize_unit + scoring statics (upper bound)
    const bool lpt_ok = nt == 1024 ? lpt <= 2 : (nt == 512 ? lpt <= 4 : (nt == 256 && lpt >= 2 && lpt <= 8));
    return lpt_ok && fused_smem_bytes(D) + static_est <= (size_t)optin;
}

// lpt = leaves per thread for nt threads (nt * lpt >= the tree size); nt in {256, 512, 1024}
cudaError_t launch_select_c2(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                             const uint16_t* k_new, const uint16_t* v_new, int32_t* pages_out,
                             uint8_t* corrected_out, int lpt, int nt, int cl, bool pdl, int which, cudaStream_t s) {
#define FKV_C2C(LP, GMV, N)                                                                                       \
    do {                                                                                                         \
        if (cl == 1)                                                                                             \
            return launch_c2_g<LP, GMV, N, 1>(D, L, X, q, k_new, v_new, pages_out, corrected_out, pdl, which, s); \
        return launch_c2_g<LP, GMV, N, 2>(D, L, X, q, k_new, v_new, pages_out, corrected_out, pdl, which, s);     \
    } while (0)
#define FKV_C2G(LP, N)                       \
    do {                                     \
        if (D.G <= 1) FKV_C2C(LP, 1, N);     \
        if (D.G <= 2) FKV_C2C(LP, 2, N);     \
        if (D.G <= 4) FKV_C2C(LP, 4, N);     \
        FKV_C2C(LP, 8, N);                   \
    } while (0)
    if (nt == 1024) {
        if (lpt == 1) FKV_C2G(1, 1024);
        if (lpt == 2) FKV_C2G(2, 1024);
    } else if (nt == 512) {
        if (lpt == 1) FKV_C2G(1, 512);
        if (lpt == 2) FKV_C2G(2, 512);
        if (lpt == 4) FKV_C2G(4, 512);
    } else if (nt == 256) {
        if (lpt == 2) FKV_C2G(2, 256);
        if (lpt == 4) FKV_C2G(4, 256);
        if (lpt == 8) FKV_C2G(8, 256);
    }
#undef FKV_C2G
#undef FKV_C2C
    return cudaErrorNotSupported;
}

// GM = group-size bucket (1, 2, 4, 8) >= G: the per-head loops and shuffles run GM wide
template <int LPT, int GM, int NT>
static cudaError_t launch_fin_g(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                const uint16_t* k_new, const uint16_t* v_new, int32_t* pages_out,
                                uint8_t* corrected_out, size_t smem, bool pdl, int which, cudaStream_t s,
                                int appended) {
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(fkv_select_finalize_kernel<LPT, GM, NT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(fkv_select_finalize_kernel<LPT, GM, NT>,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    const int grid = D.U;
    return launch_ex(fkv_select_finalize_kernel<LPT, GM, NT>, dim3(grid), dim3(NT), smem, s, pdl, D, L, X.page_rows,
                     X.page_valid, X.page_dst, X.page_cnt, X.trace, (const float*)X.scores, q, k_new, v_new, pages_out,
                     corrected_out, which, (const float*)(appended ? X.cosv : nullptr));
}

template <int LPT, int NT>
static cudaError_t launch_fin(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              const uint16_t* k_new, const uint16_t* v_new, int32_t* pages_out,
                              uint8_t* corrected_out, size_t smem, bool pdl, int which, cudaStream_t s,
                              int appended) {
    if (D.G <= 1) return launch_fin_g<LPT, 1, NT>(D, L, X, q, k_new, v_new, pages_out, corrected_out, smem, pdl, which, s, appended);
    if (D.G <= 2) return launch_fin_g<LPT, 2, NT>(D, L, X, q, k_new, v_new, pages_out, corrected_out, smem, pdl, which, s, appended);
    if (D.G <= 4) return launch_fin_g<LPT, 4, NT>(D, L, X, q, k_new, v_new, pages_out, corrected_out, smem, pdl, which, s, appended);
    return launch_fin_g<LPT, 8, NT>(D, L, X, q, k_new, v_new, pages_out, corrected_out, smem, pdl, which, s, appended);
}

// nt = threads per CTA (512 or 1024); lpt = leaves per thread: nt * lpt >= next_pow2(n_off) for every
// n_off the handle can reach (a larger zero-padded tree gives the same Z, CFR-6).  k_new/v_new non-NULL
// fuses this step's single-token append (row a9) into the kernel.
cudaError_t launch_finalize(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                            const uint16_t* k_new, const uint16_t* v_new, int32_t* pages_out,
                            uint8_t* corrected_out, int lpt, int nt, bool pdl, int which, cudaStream_t s,
                            int appended) {
    const size_t smem = page_elems(D) * sizeof(uint16_t) + (size_t)D.n_page_max * sizeof(uint16_t);
#define FKV_FIN(LP, N) \
    return launch_fin<LP, N>(D, L, X, q, k_new, v_new, pages_out, corrected_out, smem, pdl, which, s, appended)
    if (nt == 1024) {
        switch (lpt) {
            case 1: FKV_FIN(1, 1024);
            case 2: FKV_FIN(2, 1024);
            case 4: FKV_FIN(4, 1024);
            case 8: FKV_FIN(8, 1024);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (lpt) {
        case 1: FKV_FIN(1, 512);
        case 2: FKV_FIN(2, 512);
        case 4: FKV_FIN(4, 512);
        case 8: FKV_FIN(8, 512);
        case 16: FKV_FIN(16, 512);
        default: return cudaErrorInvalidValue;
    }
#undef FKV_FIN
}

}  // namespace fkv
