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
#include <algorithm>

#include "fkv_internal.cuh"

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

// ----------------------------------------------------------- a2: scoring
// Thread per page, warp per 32-page summary block.  Each warp pulls its whole
// 16 KiB block (32 pages x {min,max} x 128 channels, bf16) into shared memory
// with ONE cp.async.bulk (TMA engine, mbarrier completion), so every warp has
// its full working set in flight at once; q is staged meanwhile.  Lanes then
// read their page's 16-byte channel chunks conflict-free.
// CFR-2 in the two-FMA form: for c ascending,
//   u = fma(max(q_c,0), mx_c, u); u = fma(min(q_c,0), mn_c, u)
// -- exactly one of the two changes u, by fl(u + q_c * m_c) with an exact
// product, so u equals the recipe's sequential sum up to the sign of zero.
constexpr int kScoreWarps = 4;
constexpr int kSummBlockBytes = 32 * 2 * kHeadDim * 2;  // 16 KiB: 32 pages x {min,max} x 128 ch

// Heads of a group are split over the 4 warps of a CTA (warp w scores heads
// w, w+4 for every page of the block), so all 4 warps share one 16 KiB summary
// block in shared memory.  Each CTA takes a contiguous range of the flattened
// (unit-major) list of active 32-page blocks and streams it through a 2-stage
// ring of cp.async.bulk (TMA) copies with mbarrier completion: block i+1 lands
// while block i is scored.  ~6 CTAs (24 warps) per SM hide the FMA latency.

template <int G>
__global__ void __launch_bounds__(kScoreWarps * 32) fkv_score_kernel(FkvDims D, FkvLayer L,
                                                                     float* __restrict__ scores,
                                                                     const uint16_t* __restrict__ q, int blk_lo,
                                                                     int nb_act) {
    constexpr int NH = (G + kScoreWarps - 1) / kScoreWarps;  // heads of this warp (<= 2)
    extern __shared__ __align__(128) uint8_t s_raw[];
    uint4* buf = reinterpret_cast<uint4*>(s_raw);                                   // [2][16 KiB]
    float4* qpn = reinterpret_cast<float4*>(s_raw + 2 * kSummBlockBytes);          // [G][64]: (q+,q-) x 2 ch
    __shared__ __align__(8) uint64_t bar[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long N = (long long)D.U * nb_act;
    const long long i0 = (long long)blockIdx.x * N / gridDim.x, i1 = (long long)(blockIdx.x + 1) * N / gridDim.x;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto active = [&](long long i) {
        const int u = (int)(i / nb_act), blk = blk_lo + (int)(i % nb_act);
        const int n_off = L.n_off[u];
        return blk * 32 < n_off && blk * 32 + 31 >= D.n_sink;
    };
    auto issue = [&](long long i, int sb) {  // thread 0 only
        const int u = (int)(i / nb_act), blk = blk_lo + (int)(i % nb_act);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[sb], kSummBlockBytes);
        bulk_g2s(buf + sb * (kSummBlockBytes / 16), L.summ + summ_chunk_offset(D, u, blk * 32, 0, 0),
                 kSummBlockBytes, &bar[sb]);
    };
    if (threadIdx.x == 0) {
        if (i0 < i1 && active(i0)) issue(i0, 0);
        if (i0 + 1 < i1 && active(i0 + 1)) issue(i0 + 1, 1);
    }
    uint32_t phase_bits = 0u;
    int q_unit = -1;
    for (long long i = i0; i < i1; ++i) {
        const int sb = (int)((i - i0) & 1);
        const int u = (int)(i / nb_act), blk = blk_lo + (int)(i % nb_act);
        const bool act = active(i);
        if (act && u != q_unit) {  // stage (q+, q-) of this unit, two channels per float4
            const int b = u / D.n_kv, m = u % D.n_kv;
            for (int e = threadIdx.x; e < G * kHeadDim / 2; e += blockDim.x) {
                const int h = e / (kHeadDim / 2), c2 = e % (kHeadDim / 2);
                const uint32_t w2 = *reinterpret_cast<const uint32_t*>(
                    q + ((size_t)b * D.n_qo + m * G + h) * kHeadDim + 2 * c2);
                const float x0 = bf16_lo(w2), x1 = bf16_hi(w2);
                qpn[h * (kHeadDim / 2) + c2] = make_float4(fmaxf(x0, 0.0f), fminf(x0, 0.0f), fmaxf(x1, 0.0f),
                                                           fminf(x1, 0.0f));
            }
            __syncthreads();
            q_unit = u;
        }
        if (act) {
            mbar_wait(&bar[sb], (phase_bits >> sb) & 1u);
            phase_bits ^= 1u << sb;
            const uint4* blkp = buf + sb * (kSummBlockBytes / 16);
            float acc[NH];
#pragma unroll
            for (int k = 0; k < NH; ++k) acc[k] = 0.0f;
#pragma unroll 2
            for (int c8 = 0; c8 < kHeadDim / 8; ++c8) {
                const uint4 mn4 = blkp[(c8 * 2 + 0) * 32 + lane];
                const uint4 mx4 = blkp[(c8 * 2 + 1) * 32 + lane];
                const uint32_t mnw[4] = {mn4.x, mn4.y, mn4.z, mn4.w};
                const uint32_t mxw[4] = {mx4.x, mx4.y, mx4.z, mx4.w};
#pragma unroll
                for (int wd = 0; wd < 4; ++wd) {
                    const float mn0 = bf16_lo(mnw[wd]), mn1 = bf16_hi(mnw[wd]);
                    const float mx0 = bf16_lo(mxw[wd]), mx1 = bf16_hi(mxw[wd]);
#pragma unroll
                    for (int k = 0; k < NH; ++k) {
                        const int h = warp + k * kScoreWarps;
                        if (h < G) {
                            const float4 qq = qpn[h * (kHeadDim / 2) + c8 * 4 + wd];
                            // channel 2*wd (ascending), then channel 2*wd+1 -- CFR-2 order
                            acc[k] = __fmaf_rn(qq.x, mx0, acc[k]);
                            acc[k] = __fmaf_rn(qq.y, mn0, acc[k]);
                            acc[k] = __fmaf_rn(qq.z, mx1, acc[k]);
                            acc[k] = __fmaf_rn(qq.w, mn1, acc[k]);
                        }
                    }
                }
            }
            const int j = blk * 32 + lane;
            const int n_off = L.n_off[u];
            if (j >= D.n_sink && j < n_off) {
#pragma unroll
                for (int k = 0; k < NH; ++k) {
                    const int h = warp + k * kScoreWarps;
                    if (h < G) scores[((size_t)u * G + h) * D.n_page_max + j] = __fmul_rn(acc[k], D.score_r);  // CFR-3
                }
            }
        }
        __syncthreads();  // every warp is done with buffer sb (and with q) before it is refilled
        if (threadIdx.x == 0 && i + 2 < i1 && active(i + 2)) issue(i + 2, sb);
    }
}

// ------------------------------------------------------- block utilities
// Exclusive scan of one int per thread over a 1024-thread block (thread order).
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = s_warp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_warp[lane] = w;  // inclusive
    }
    __syncthreads();
    const int warp_off = warp ? s_warp[warp - 1] : 0;
    *total = s_warp[31];
    __syncthreads();
    return warp_off + x - v;
}

constexpr int kMaxK = 256;

// ------------------------------------------------------ a1 + a3 + a4
template <int LPT>
__global__ void __launch_bounds__(1024) fkv_select_finalize_kernel(FkvDims D, FkvLayer L,
                                                                   const float* __restrict__ scores,
                                                                   const uint16_t* __restrict__ q,
                                                                   int32_t* __restrict__ pages_out,
                                                                   uint8_t* __restrict__ corrected_out) {
    const int u = blockIdx.x, b = u / D.n_kv, m = u % D.n_kv, G = D.G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_off = L.n_off[u], n_sink = D.n_sink, K = D.K;

    __shared__ float s_red[32][kMaxG];
    __shared__ float s_M[kMaxG], s_Z[kMaxG], s_cos[kMaxG];
    __shared__ int s_hist[256];
    __shared__ int s_warp[32];
    __shared__ int s_digit, s_above;
    __shared__ int s_sel[kMaxK], s_cnt;
    __shared__ int s_res[kMaxK], s_res_slot[kMaxK];
    __shared__ int s_isfetch[kMaxK];
    __shared__ int s_free[2 * kMaxK];
    __shared__ unsigned char s_used[2 * kMaxK];
    __shared__ uint32_t s_qa[kMaxG * kHeadDim / 2], s_qb[kMaxG * kHeadDim / 2];
    extern __shared__ float s_sc[];  // [G][n_page_max] scores of this unit (candidates only)

    // ---- a1: correction (CFR-10).  q_i and q_{i-1} of the group are staged in shared
    // memory with coalesced loads; threads 0..G-1 then run the sequential channel sums.
    {
        const uint32_t* qa32 = reinterpret_cast<const uint32_t*>(q + ((size_t)b * D.n_qo + m * G) * kHeadDim);
        const uint32_t* qb32 = reinterpret_cast<const uint32_t*>(L.q_prev + ((size_t)b * D.n_qo + m * G) * kHeadDim);
        for (int i = tid; i < G * kHeadDim / 2; i += blockDim.x) {
            s_qa[i] = qa32[i];
            s_qb[i] = qb32[i];
        }
    }
    __syncthreads();
    if (tid < G) {
        const uint16_t* qa = reinterpret_cast<const uint16_t*>(s_qa) + tid * kHeadDim;
        const uint16_t* qb = reinterpret_cast<const uint16_t*>(s_qb) + tid * kHeadDim;
        float dot = 0.0f, n1 = 0.0f, n2 = 0.0f;
#pragma unroll 16
        for (int c = 0; c < kHeadDim; ++c) {
            const float x = bf16f(qa[c]), y = bf16f(qb[c]);
            dot = __fmaf_rn(x, y, dot);  // exact product, one rounding = fl(dot + x*y)
            n1 = __fmaf_rn(x, x, n1);
            n2 = __fmaf_rn(y, y, n2);
        }
        s_cos[tid] = (n1 == 0.0f || n2 == 0.0f) ? 0.0f : __fdiv_rn(dot, __fmul_rn(__fsqrt_rn(n1), __fsqrt_rn(n2)));
    }
    // resident set into smem
    const int res_valid = L.res_valid[u];
    for (int i = tid; i < K; i += blockDim.x) {
        s_res[i] = res_valid ? L.res_pages[(size_t)u * K + i] : -1;
        s_res_slot[i] = res_valid ? L.res_slot[(size_t)u * K + i] : -1;
    }
    for (int i = tid; i < 2 * K; i += blockDim.x) s_used[i] = 0;

    const int n_cand = n_off - n_sink;
    if (n_cand <= K) {
        // A-11: all candidates selected
        for (int i = tid; i < K; i += blockDim.x) s_sel[i] = i < n_cand ? n_sink + i : -1;
        if (tid == 0) s_cnt = n_cand > 0 ? n_cand : 0;
        __syncthreads();
    } else {
        const size_t srow = (size_t)D.n_page_max;
        {
            const float* sg = scores + (size_t)u * G * srow;
            for (int j = n_sink + tid; j < n_off; j += blockDim.x) {
                float v[kMaxG];  // all heads' loads in flight together
#pragma unroll
                for (int g = 0; g < kMaxG; ++g)
                    if (g < G) v[g] = sg[g * srow + j];
#pragma unroll
                for (int g = 0; g < kMaxG; ++g)
                    if (g < G) s_sc[g * srow + j] = v[g];
            }
        }
        __syncthreads();
        const float* su = s_sc;
        const int jb = tid * LPT;
        // ---- CFR-4: max per head
        float mx[kMaxG];
#pragma unroll
        for (int g = 0; g < kMaxG; ++g) mx[g] = -INFINITY;
#pragma unroll
        for (int g = 0; g < kMaxG; ++g) {
            if (g < G) {
#pragma unroll
                for (int l = 0; l < LPT; ++l) {
                    const int j = jb + l;
                    if (j >= n_sink && j < n_off) mx[g] = fmaxf(mx[g], su[g * srow + j]);
                }
                float v = mx[g];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
                if (lane == 0) s_red[warp][g] = v;
            }
        }
        __syncthreads();
        if (warp == 0) {
            for (int g = 0; g < G; ++g) {
                float v = s_red[lane][g];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
                if (lane == 0) s_M[g] = v;
            }
        }
        __syncthreads();
        // ---- CFR-5/6: e = cexp2(s - m); Z = pairwise tree over leaves in page-id order
        for (int g = 0; g < G; ++g) {
            float e[LPT];
            const float M = s_M[g];
#pragma unroll
            for (int l = 0; l < LPT; ++l) {
                const int j = jb + l;
                e[l] = (j >= n_sink && j < n_off) ? cexp2_cfr(__fsub_rn(su[g * srow + j], M)) : 0.0f;
            }
#pragma unroll
            for (int w = 1; w < LPT; w <<= 1)
#pragma unroll
                for (int l = 0; l < LPT; l += 2 * w) e[l] = __fadd_rn(e[l], e[l + w]);
            float v = e[0];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (lane == 0) s_red[warp][g] = v;
        }
        __syncthreads();
        if (warp == 0) {
            for (int g = 0; g < G; ++g) {
                float v = s_red[lane][g];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
                if (lane == 0) s_Z[g] = v;
            }
        }
        __syncthreads();
        // ---- CFR-7/8: p = e / Z; pooled = sequential sum over g
        float pi[LPT];
#pragma unroll
        for (int l = 0; l < LPT; ++l) pi[l] = 0.0f;
        for (int g = 0; g < G; ++g) {
            const float M = s_M[g], Z = s_Z[g];
#pragma unroll
            for (int l = 0; l < LPT; ++l) {
                const int j = jb + l;
                if (j >= n_sink && j < n_off) {
                    const float p = __fdiv_rn(cexp2_cfr(__fsub_rn(su[g * srow + j], M)), Z);
                    pi[l] = g == 0 ? p : __fadd_rn(pi[l], p);
                }
            }
        }
        // ---- CFR-9: radix select of the K-th largest key
        uint32_t key[LPT];
        bool cand[LPT];
#pragma unroll
        for (int l = 0; l < LPT; ++l) {
            const int j = jb + l;
            cand[l] = j >= n_sink && j < n_off;
            uint32_t kk = __float_as_uint(pi[l]);
            key[l] = kk == 0x80000000u ? 0u : kk;
        }
        uint32_t prefix = 0u, mask = 0u;
        int k_rem = K;
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int i = tid; i < 256; i += blockDim.x) s_hist[i] = 0;
            __syncthreads();
#pragma unroll
            for (int l = 0; l < LPT; ++l)
                if (cand[l] && (key[l] & mask) == prefix) atomicAdd(&s_hist[(key[l] >> shift) & 255u], 1);
            __syncthreads();
            if (warp == 0) {
                int bins[8], lsum = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    bins[i] = s_hist[lane * 8 + i];
                    lsum += bins[i];
                }
                // inclusive suffix scan over lanes (from high lanes down)
                int suf = lsum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_down_sync(0xffffffffu, suf, o);
                    if (lane + o < 32) suf += y;
                }
                int above = suf - lsum;  // count in bins of higher lanes
#pragma unroll
                for (int i = 7; i >= 0; --i) {
                    if (above < k_rem && above + bins[i] >= k_rem) {
                        s_digit = lane * 8 + i;
                        s_above = above;
                    }
                    above += bins[i];
                }
            }
            __syncthreads();
            const int Dg = s_digit;
            k_rem -= s_above;
            prefix |= (uint32_t)Dg << shift;
            mask |= 0xFFu << shift;
            __syncthreads();
        }
        const uint32_t T = prefix;  // K-th largest key; take k_rem of the keys equal to T (lowest ids)
        int n_eq = 0;
#pragma unroll
        for (int l = 0; l < LPT; ++l) n_eq += (cand[l] && key[l] == T);
        int tot;
        int eq_rank = block_excl_scan(n_eq, s_warp, &tot);
        bool take[LPT];
        int n_take = 0;
#pragma unroll
        for (int l = 0; l < LPT; ++l) {
            bool t = false;
            if (cand[l]) {
                if (key[l] > T) t = true;
                else if (key[l] == T) { t = eq_rank < k_rem; ++eq_rank; }
            }
            take[l] = t;
            n_take += t;
        }
        int pos = block_excl_scan(n_take, s_warp, &tot);
#pragma unroll
        for (int l = 0; l < LPT; ++l)
            if (take[l]) s_sel[pos++] = jb + l;
        for (int i = tid + K; i < kMaxK; i += blockDim.x) s_sel[i] = -1;  // harmless pad
        if (tid == 0) s_cnt = K;
        __syncthreads();
    }

    // ---- flag (CFR-10 pooling, A-12, A-13)
    if (tid == 0) {
        float acc = s_cos[0];
        for (int g = 1; g < G; ++g) acc = __fadd_rn(acc, s_cos[g]);
        const float mean = __fdiv_rn(acc, (float)G);
        int flag;
        if (D.mode == 1 || D.tau >= 1.0f) flag = 1;
        else if (D.mode == 2 || D.tau <= 0.0f) flag = 0;
        else flag = mean < D.tau;
        if (!res_valid) flag = 1;
        L.flags[u] = (uint8_t)flag;
        L.cbar[u] = mean;
        L.pend_front[u] = n_off;
        if (corrected_out) corrected_out[u] = (uint8_t)flag;
    }
    // ---- a4: delta vs resident (A-18) and slot assignment
    const int cnt = s_cnt;
    if (tid < K) {
        int f = 0;
        const int Sa = tid < cnt ? s_sel[tid] : -1;
        if (Sa >= 0) {
            f = 1;
            for (int i = 0; i < K; ++i)
                if (s_res[i] == Sa) { f = 0; L.pend_slot[(size_t)u * K + tid] = s_res_slot[i]; }
        }
        s_isfetch[tid] = f;
        if (s_res[tid] >= 0) s_used[s_res_slot[tid]] = 1;
        L.pend_pages[(size_t)u * K + tid] = Sa;
        if (pages_out) pages_out[(size_t)u * K + tid] = Sa;
        if (Sa < 0) L.pend_slot[(size_t)u * K + tid] = -1;
    }
    __syncthreads();
    if (warp == 0) {
        // free slots ascending
        int nfree = 0;
        for (int base = 0; base < 2 * K; base += 32) {
            const int s = base + lane;
            const bool fr = s < 2 * K && !s_used[s];
            const unsigned bal = __ballot_sync(0xffffffffu, fr);
            if (fr) s_free[nfree + __popc(bal & ((1u << lane) - 1u))] = s;
            nfree += __popc(bal);
        }
        __syncwarp();
        int nf = 0;
        for (int base = 0; base < K; base += 32) {
            const int a = base + lane;
            const bool fe = a < K && s_isfetch[a];
            const unsigned bal = __ballot_sync(0xffffffffu, fe);
            if (fe) {
                const int r = nf + __popc(bal & ((1u << lane) - 1u));
                const int slot = s_free[r];
                L.pend_slot[(size_t)u * K + a] = slot;
                L.fetch_page[(size_t)u * K + r] = s_sel[a];
                L.fetch_slot[(size_t)u * K + r] = slot;
            }
            nf += __popc(bal);
        }
        if (lane == 0) {
            L.n_fetch[u] = nf;
            L.pend_cnt[u] = cnt;
        }
    }
}

template <int G>
static void launch_score_g(const FkvDims& D, const FkvLayer& L, float* scores, const uint16_t* q, int max_n_off,
                           cudaStream_t s) {
    const int blk_lo = D.n_sink / 32;
    const int nb_act = (max_n_off + 31) / 32 - blk_lo;
    if (nb_act <= 0) return;
    const int smem = 2 * kSummBlockBytes + G * kHeadDim * 2 * 4;
    static int max_ctas = 0;
    if (!max_ctas) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(fkv_score_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fkv_score_kernel<G>, kScoreWarps * 32, smem);
        max_ctas = sms * (per_sm > 0 ? per_sm : 1);
    }
    const long long n = (long long)D.U * nb_act;
    const int grid = (int)std::min<long long>(max_ctas, n);
    fkv_score_kernel<G><<<grid, kScoreWarps * 32, smem, s>>>(D, L, scores, q, blk_lo, nb_act);
}

cudaError_t launch_score(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                         int max_n_off, cudaStream_t s) {
    switch (D.G) {
        case 1: launch_score_g<1>(D, L, X.scores, q, max_n_off, s); break;
        case 2: launch_score_g<2>(D, L, X.scores, q, max_n_off, s); break;
        case 3: launch_score_g<3>(D, L, X.scores, q, max_n_off, s); break;
        case 4: launch_score_g<4>(D, L, X.scores, q, max_n_off, s); break;
        case 5: launch_score_g<5>(D, L, X.scores, q, max_n_off, s); break;
        case 6: launch_score_g<6>(D, L, X.scores, q, max_n_off, s); break;
        case 7: launch_score_g<7>(D, L, X.scores, q, max_n_off, s); break;
        case 8: launch_score_g<8>(D, L, X.scores, q, max_n_off, s); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int LPT>
static cudaError_t launch_fin(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              int32_t* pages_out, uint8_t* corrected_out, size_t smem, cudaStream_t s) {
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(fkv_select_finalize_kernel<LPT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    fkv_select_finalize_kernel<LPT><<<D.U, 1024, smem, s>>>(D, L, X.scores, q, pages_out, corrected_out);
    return cudaGetLastError();
}

// lpt = leaves per thread of the 1024-thread tree; 1024 * lpt >= next_pow2(n_off) for every n_off the
// handle can reach (a larger zero-padded tree gives the same Z, CFR-6).
cudaError_t launch_finalize(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                            int32_t* pages_out, uint8_t* corrected_out, int lpt, cudaStream_t s) {
    const size_t smem = (size_t)D.G * D.n_page_max * sizeof(float);
    switch (lpt) {
        case 1: return launch_fin<1>(D, L, X, q, pages_out, corrected_out, smem, s);
        case 2: return launch_fin<2>(D, L, X, q, pages_out, corrected_out, smem, s);
        case 4: return launch_fin<4>(D, L, X, q, pages_out, corrected_out, smem, s);
        case 8: return launch_fin<8>(D, L, X, q, pages_out, corrected_out, smem, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fkv
