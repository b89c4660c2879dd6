// score.cu -- row a2, page scoring (PAPER.md P:231 Quest-style min/max summaries, reading A-1;
// P:133-134; CFR-2/3), plus one extra CTA per unit for rows a1 (correction check, P:247-250;
// CFR-10) and a9 (append of this step's token).
//
// Thread-per-page: CFR-2 fixes each (page, head) score as a sequential fp32 chain over the
// channels c = 0..127, so a page's chain cannot be split across threads.  Each thread owns
// kScPPT = 4 pages and evaluates the chains of two heads at once with packed FFMA2
// (fma.rn.f32x2): u_pair = fma({q-_h, q-_h'}, {mn, mn}, fma({q+_h, q+_h'}, {mx, mx}, u_pair)),
// with q+ = max(q, 0), q- = min(q, 0) -- one of the two products is a signed zero, so every step
// is CFR-2's single rounding of u + q_c * (q_c >= 0 ? mx_c : mn_c) (equal up to the sign of zero,
// which CFR-2 allows).  Odd G pads the last pair with a zero head.
//
// Why head pairs and 4 pages per thread (measured, tools/iso_bench.py --trace): the broadcast
// 16-byte shared loads of q cost 4 MIO cycles each (512 B of register writes per warp), and with
// page pairs ({q, q} per head) they bounded the loop at ~7 us on c2.  A head pair's {q+_h, q+_h',
// q-_h, q-_h'} is one load and feeds 8 FFMA2 (4 pages x 2 terms): 4x fewer q loads per page.
//
// Summaries are channel-group-major (fkv_internal.cuh summ_off): the {min, max} of 8 channels
// of a warp's 128 consecutive pages are two contiguous 2 KiB runs, streamed per warp through a
// ring of kScStages 4 KiB stages filled by cp.async.bulk (TMA engine, SASS UBLKCP) with mbarrier
// completion.  The first stages are issued before the PDL wait: summaries are layer state, not
// step input.
#include "append_unit.cuh"

namespace fkv {

constexpr int kScWarps = FKV_SC_WARPS;  // warps per CTA of the speculative step's parts 0/1
template <int PPT, int W, int S = 4> struct ScGeom {            // PPT pages/thread, W warps/CTA, S stages/warp
    static constexpr int WarpPages = 32 * PPT;
    static constexpr int CtaPages = W * WarpPages;              // a power of two
    static constexpr int StageBytes = 2 * WarpPages * 16;       // {min, max} x pages x 8 channels
    static constexpr int Smem = W * S * StageBytes;
};
static_assert(ScGeom<4, kScWarps>::CtaPages == kScoreCtaPages, "score CTA page count (the select waits per item)");
static_assert(ScGeom<1, kScWarps>::CtaPages == kScoreCtaPagesFast, "score CTA page count (the select waits per item)");

__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void ffma2(unsigned long long& acc, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ float pk_lo(unsigned long long v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float pk_hi(unsigned long long v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t u4w(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// ---- decode-step prologue of one layer, one CTA per unit (rows a8 deferred, a1, a9):
//  * deferred commit R := S_{i-1} of a unit whose previous selection ran in the background (P:225:
//    the pages selected with q_{i-1} are the ones used at step i) -- its side chain (select + recall)
//    was joined before this kernel;
//  * q_cur := q_i (the side chain's scoring and selection read it after the caller's buffer may be
//    reused);
//  * correction check (CFR-10): per-head cosine of q_i and q_{i-1}, group decision
//    (readings A-12, A-13, R-11) published in L.flags / L.cbar;
//  * append of this step's token (offload + summary when its page completes) and the new
//    context length / frontier (every later kernel of the layer-step runs after this one);
//  * ordered: the unit's slot in L.order (corrected units from the front, the others from the
//    back) -- the side chain scores and selects the corrected units first.
constexpr int kPreThreads = 128;

// full = 1: the pre kernel (every duty above).  full = 0: the extra CTAs of the serial step's score
// grid -- correction flag and append only; the context length stays unpublished until the
// attention's commit (the scoring CTAs of the same grid read it: the token is "pending").
__device__ __forceinline__ void pre_unit(const FkvDims& D, const FkvLayer& L, int u, const uint16_t* __restrict__ q,
                                         const uint16_t* __restrict__ k_new, const uint16_t* __restrict__ v_new,
                                         int ordered, int full, uint4* s_page) {
    __shared__ float s_cos[kMaxG];
    const int b = u / D.n_kv, m = u % D.n_kv, G = D.G, tid = threadIdx.x, nt = blockDim.x;
    // state only before the PDL wait (the previous kernel is the previous layer's attention)
    const int pv = full ? L.pend_valid[u] : 0;
    if (pv) {
        for (int i = tid; i < D.K; i += nt) {
            L.res_pages[(size_t)u * D.K + i] = L.pend_pages[(size_t)u * D.K + i];
            L.res_slot[(size_t)u * D.K + i] = L.pend_slot[(size_t)u * D.K + i];
        }
        if (tid == 0) {
            L.res_front[u] = L.pend_front[u];
            L.res_cnt[u] = L.pend_cnt[u];
            L.res_valid[u] = 1;
            L.pend_valid[u] = 0;
        }
    }
    const int res_valid = D.full_refresh ? 0 : (pv ? 1 : L.res_valid[u]);
    const int ctx0 = L.ctx[u];
    if (tid == 0) trace_stamp(L.trace, 8, u, 0);
    pdl_wait();  // q_i and the new token are this layer's inputs
    pdl_trigger();
    const size_t row0 = ((size_t)b * D.n_qo + m * G) * kHeadDim;
    if (full)
        for (int i = tid; i < G * (kHeadDim / 8); i += nt)
            reinterpret_cast<uint4*>(L.q_cur + row0)[i] = reinterpret_cast<const uint4*>(q + row0)[i];
    if (tid < G) s_cos[tid] = cos_cfr10(q + row0 + (size_t)tid * kHeadDim, L.q_prev + row0 + (size_t)tid * kHeadDim);
    __syncthreads();
    if (tid == 0) {
        const float pooled = pool_cos(s_cos, G, D.corr_pool);
        const int flag = correction_flag(D, pooled, res_valid);
        L.flags[u] = (uint8_t)flag;
        L.cbar[u] = pooled;
        L.score_done[u] = 0;
        if (ordered) {
            // this step's parity is that of the new context length; the other parity's counters were
            // last used by the previous step (joined), so they are reset here for the next one
            const int par = (ctx0 + 1) & 1;
            int32_t* cnt = L.ord_cnt + par * 2;
            const int slot = flag ? atomicAdd(cnt, 1) : D.U - 1 - atomicAdd(cnt + 1, 1);
            L.order[slot] = u;
            L.ord_cnt[(par ^ 1) * 2] = 0;
            L.ord_cnt[(par ^ 1) * 2 + 1] = 0;
        }
    }
    append_unit(D, L, u, ctx0, k_new, v_new, 1, s_page);
    if (full && tid == 0) {
        L.ctx[u] = ctx0 + 1;
        L.n_off[u] = max(L.n_off[u], frontier_for(D, ctx0 + 1));
    }
    if (tid == 0) trace_stamp(L.trace, 8, u, 1);
}

__global__ void __launch_bounds__(kPreThreads) fkv_pre_kernel(FkvDims D, FkvLayer L, const uint16_t* __restrict__ q,
                                                              const uint16_t* __restrict__ k_new,
                                                              const uint16_t* __restrict__ v_new, int ordered) {
    extern __shared__ __align__(16) uint4 s_page[];  // append staging: one (2, p, d) page
    pre_unit(D, L, blockIdx.x, q, k_new, v_new, ordered, 1, s_page);
}

cudaError_t launch_pre(const FkvDims& D, const FkvLayer& L, const uint16_t* q, const uint16_t* k_new,
                       const uint16_t* v_new, int ordered, bool pdl, int prio, cudaStream_t s) {
    const size_t smem = page_elems(D) * sizeof(uint16_t);
    cudaError_t e = func_smem((const void*)fkv_pre_kernel, smem);
    if (e != cudaSuccess) return e;
    return launch_ex(fkv_pre_kernel, dim3(D.U), dim3(kPreThreads), smem, s, pdl, prio, D, L, q, k_new, v_new, ordered);
}

// grid: U * items_per_unit CTAs; item r of a unit scores pages [CP r, CP r + CP) n [n_sink, n_off)
// (CP = 512 for PPT = 4, 128 for PPT = 1).  part >= 0 (speculative step): the unit of CTA i is
// part_unit(i / items_per_unit) and every CTA counts itself done in L.score_done[u] (release),
// which the select kernel acquires per unit instead of waiting for the whole grid.
template <int G, int PPT, int W, int S>
__global__ void __launch_bounds__(W * 32) fkv_score_kernel(FkvDims D, FkvLayer L, const uint16_t* __restrict__ q,
                                                               int items_per_unit, int part,
                                                               const uint16_t* __restrict__ k_new,
                                                               const uint16_t* __restrict__ v_new) {
    constexpr int GP = (G + 1) / 2;  // head pairs
    constexpr int kScPPT = PPT, kScWarpPages = ScGeom<PPT, W>::WarpPages, kScCtaPages = ScGeom<PPT, W>::CtaPages;
    constexpr int kScStageBytes = ScGeom<PPT, W>::StageBytes, kScStages = S;  // ring depth per warp
    const int ordered = part >= 0;
    extern __shared__ __align__(128) uint8_t s_raw[];
    __shared__ __align__(16) float4 s_q[kHeadDim][GP];  // {q+_h, q+_h', q-_h, q-_h'} of pair (h, h') at c
    __shared__ __align__(8) uint64_t bar[W][kScStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* trace = L.trace;
    // part -2 (serial step): U extra CTAs first, each the correction check and append of one unit
    // (the token is pending: the scoring CTAs take the frontier of ctx + 1)
    const int n_pre = part == -2 ? D.U : 0;
    if ((int)blockIdx.x < n_pre) {
        pre_unit(D, L, blockIdx.x, q, k_new, v_new, 0, 0, reinterpret_cast<uint4*>(s_raw));
        return;
    }
    const int item = blockIdx.x - n_pre;
    const int ui = item / items_per_unit, r = item - ui * items_per_unit;
    // part 0 runs on the critical path right after the pre kernel, which writes the unit order
    if (part == 0) pdl_wait();
    const int u = part_unit(D, L, part == -2 ? -1 : part, ui);
    if (u < 0) return;  // CTA-uniform: no unit at this index in this part
    const int b = u / D.n_kv, m = u % D.n_kv;
    // the frontier only grows; the pre kernel (possibly this grid's predecessor) may still raise it,
    // so the summaries issued before the PDL wait are those of the pages below the state's value
    const int pending = part == -2 ? 1 : 0;
    const int n_lo = pending ? max(L.n_off[u], frontier_for(D, L.ctx[u] + 1)) : L.n_off[u];
    if (threadIdx.x == 0) trace_stamp(trace, 0, item, 0);
    const int j0 = r * kScCtaPages + warp * kScWarpPages;
    // (with W = 0 the pre kernel's append may complete a page that is a candidate at once: its
    // summary is written by the predecessor, so nothing is issued before the wait)
    const bool pre_active = D.n_win >= 1 && j0 < n_lo && j0 + kScWarpPages > D.n_sink;
    uint8_t* ring = s_raw + warp * (kScStages * kScStageBytes);
    auto issue = [&](int slot, int c8) {
        mbar_expect_tx(&bar[warp][slot], kScStageBytes);
        bulk_g2s(ring + slot * kScStageBytes, L.summ + summ_off(D, u, c8, 0, j0), kScStageBytes / 2, &bar[warp][slot]);
        bulk_g2s(ring + slot * kScStageBytes + kScStageBytes / 2, L.summ + summ_off(D, u, c8, 1, j0),
                 kScStageBytes / 2, &bar[warp][slot]);
    };
    if (lane == 0) {
#pragma unroll
        for (int s2 = 0; s2 < kScStages; ++s2) mbar_init(&bar[warp][s2], 1);
        fence_mbar_init();
        if (pre_active)
#pragma unroll
            for (int s2 = 0; s2 < kScStages; ++s2) issue(s2, s2);  // state: before the PDL wait
    }
    // q_i is this layer's input: read only after the previous kernel (the previous layer) is done
    pdl_wait();
    pdl_trigger();
    const int n_off = pending ? n_lo : L.n_off[u];  // final for this step
    if (r * kScCtaPages >= n_off) return;  // CTA-uniform: no candidate page (nothing was issued)
    const bool active = j0 < n_off && j0 + kScWarpPages > D.n_sink;
    if (active && !pre_active && lane == 0)
#pragma unroll
        for (int s2 = 0; s2 < kScStages; ++s2) issue(s2, s2);
    // staging: thread (pair hp, channel group c8) loads 16 bytes of each head of the pair
    for (int i = threadIdx.x; i < GP * (kHeadDim / 8); i += blockDim.x) {
        const int hp = i / (kHeadDim / 8), c8 = i % (kHeadDim / 8);
        const uint16_t* qg = q + ((size_t)b * D.n_qo + m * G) * kHeadDim + c8 * 8;
        float x[2][8];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int h = 2 * hp + t;
#pragma unroll
            for (int e = 0; e < 8; ++e) x[t][e] = 0.0f;
            if (h >= G) continue;  // the zero head of an odd group
            if (D.pool >= 4) {  // MeanQ / MaxQ (f3, reading R-12): every head scores the pooled query
                uint4 w = *reinterpret_cast<const uint4*>(qg);
#pragma unroll
                for (int e = 0; e < 8; ++e) x[t][e] = (e & 1) ? bf16_hi(u4w(w, e >> 1)) : bf16_lo(u4w(w, e >> 1));
                for (int g = 1; g < G; ++g) {
                    w = *reinterpret_cast<const uint4*>(qg + (size_t)g * kHeadDim);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float y = (e & 1) ? bf16_hi(u4w(w, e >> 1)) : bf16_lo(u4w(w, e >> 1));
                        x[t][e] = D.pool == 4 ? __fadd_rn(x[t][e], y) : (y > x[t][e] ? y : x[t][e]);
                    }
                }
                if (D.pool == 4)
#pragma unroll
                    for (int e = 0; e < 8; ++e) x[t][e] = __fdiv_rn(x[t][e], (float)G);
            } else {
                const uint4 w = *reinterpret_cast<const uint4*>(qg + (size_t)h * kHeadDim);
#pragma unroll
                for (int e = 0; e < 8; ++e) x[t][e] = (e & 1) ? bf16_hi(u4w(w, e >> 1)) : bf16_lo(u4w(w, e >> 1));
            }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float a = x[0][e], c = x[1][e];
            s_q[c8 * 8 + e][hp] = make_float4(a >= 0.0f ? a : 0.0f, c >= 0.0f ? c : 0.0f, a >= 0.0f ? 0.0f : a,
                                              c >= 0.0f ? 0.0f : c);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) trace_stamp(trace, 0, item, 1);
    if (!active) {
        if (ordered) {
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(L.score_done + u, 1);
            }
        }
        return;
    }
    unsigned long long acc[kScPPT][GP];  // [page i][head pair]
#pragma unroll
    for (int i = 0; i < kScPPT; ++i)
#pragma unroll
        for (int hp = 0; hp < GP; ++hp) acc[i][hp] = 0ull;
#pragma unroll 1
    for (int c8 = 0; c8 < kHeadDim / 8; ++c8) {
        const int slot = c8 % kScStages;
        mbar_wait(&bar[warp][slot], (uint32_t)(c8 / kScStages) & 1u);
        const uint4* st = reinterpret_cast<const uint4*>(ring + slot * kScStageBytes);
        uint4 mn[kScPPT], mx[kScPPT];
#pragma unroll
        for (int i = 0; i < kScPPT; ++i) {
            mn[i] = st[i * 32 + lane];
            mx[i] = st[kScWarpPages + i * 32 + lane];
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int c = c8 * 8 + e;
            unsigned long long mx2[kScPPT], mn2[kScPPT];
#pragma unroll
            for (int i = 0; i < kScPPT; ++i) {
                const float fx = (e & 1) ? bf16_hi(u4w(mx[i], e >> 1)) : bf16_lo(u4w(mx[i], e >> 1));
                const float fn = (e & 1) ? bf16_hi(u4w(mn[i], e >> 1)) : bf16_lo(u4w(mn[i], e >> 1));
                mx2[i] = pk2(fx, fx);
                mn2[i] = pk2(fn, fn);
            }
#pragma unroll
            for (int hp = 0; hp < GP; ++hp) {
                const float4 qq = s_q[c][hp];
                const unsigned long long qp = pk2(qq.x, qq.y), qm = pk2(qq.z, qq.w);
#pragma unroll
                for (int i = 0; i < kScPPT; ++i) {
                    ffma2(acc[i][hp], qp, mx2[i]);
                    ffma2(acc[i][hp], qm, mn2[i]);
                }
            }
        }
        __syncwarp();  // every lane is done with this stage
        if (lane == 0 && c8 + kScStages < kHeadDim / 8) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(slot, c8 + kScStages);
        }
    }
#pragma unroll
    for (int i = 0; i < kScPPT; ++i) {
        const int j = j0 + i * 32 + lane;
        if (j >= D.n_sink && j < n_off) {
#pragma unroll
            for (int h = 0; h < G; ++h) {
                const float uu = (h & 1) ? pk_hi(acc[i][h >> 1]) : pk_lo(acc[i][h >> 1]);
                L.scores[((size_t)u * G + h) * D.n_page_max + j] = __fmul_rn(uu, D.score_r);  // CFR-3
            }
        }
    }
    if (ordered) {  // this item's scores are written: count it (release, cumulative over the CTA barrier)
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(L.score_done + u, 1);
        }
    }
    if (threadIdx.x == 0) trace_stamp(trace, 0, item, 2);
}

template <int G, int PPT, int W, int S = 4>
static cudaError_t launch_score_gp(const FkvDims& D, const FkvLayer& L, const uint16_t* q, int max_n_off, int part,
                                   bool pdl, int prio, cudaStream_t s, const uint16_t* k_new, const uint16_t* v_new) {
    constexpr int CP = ScGeom<PPT, W>::CtaPages;
    const int SM = std::max<int>(ScGeom<PPT, W, S>::Smem, (int)(page_elems(D) * sizeof(uint16_t)));
    const int ipu = std::max(0, (max_n_off + CP - 1) / CP);
    if (ipu == 0 && part != -2) return cudaSuccess;
    cudaError_t e = func_smem((const void*)fkv_score_kernel<G, PPT, W, S>, SM);
    if (e != cudaSuccess) return e;
    const int grid = (part == -2 ? D.U : 0) + D.U * ipu;
    return launch_ex(fkv_score_kernel<G, PPT, W, S>, dim3(grid), dim3(W * 32), SM, s, pdl, prio, D, L, q,
                     std::max(ipu, 1), part, k_new, v_new);
}

template <int G>
static cudaError_t launch_score_g(const FkvDims& D, const FkvLayer& L, const uint16_t* q, int max_n_off, int part,
                                  bool pdl, int prio, cudaStream_t s, const uint16_t* k_new, const uint16_t* v_new) {
    if (part == 0) return launch_score_gp<G, 1, kScWarps>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
    if (part < 0 && D.score_warps == 8)
        return launch_score_gp<G, 4, 8>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
    if (part < 0 && D.score_stages == 6)
        return launch_score_gp<G, 4, kScWarps, 6>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
    if (part < 0 && D.score_stages == 8)
        return launch_score_gp<G, 4, kScWarps, 8>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
    return launch_score_gp<G, 4, kScWarps>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
}

cudaError_t launch_score(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q, int max_n_off,
                         int part, bool pdl, int prio, cudaStream_t s, const uint16_t* k_new, const uint16_t* v_new) {
    (void)X;
    switch (D.G) {
        case 1: return launch_score_g<1>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
        case 2: return launch_score_g<2>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
        case 3: return launch_score_g<3>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
        case 4: return launch_score_g<4>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
        case 5: return launch_score_g<5>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
        case 6: return launch_score_g<6>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
        case 7: return launch_score_g<7>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
        case 8: return launch_score_g<8>(D, L, q, max_n_off, part, pdl, prio, s, k_new, v_new);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fkv
