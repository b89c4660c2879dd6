// select.cu -- rows a1, a3, a4: correction flag (when the score kernel did not decide it),
// per-head softmax + MeanS pooling, top-K, delta vs the resident set, slot assignment and the
// corrected units' attention page lists.
//
//   a1  P:180, P:247-250 (group-mean cosine vs tau; CFR-10)
//   a3  P:232-234 (softmax per head over the candidate pages, mean pooling over the group;
//       CFR-4..8)
//   a4  P:100-101 (top-K, ties -> lower id; CFR-9), P:296 (cache of selected pages: delta +
//       slots)
//
// One cluster of NC CTAs (256 threads each) per unit.  CTA r owns the leaves (page ids)
// [r P2/NC, (r+1) P2/NC) of the pairwise tree of CFR-6 (P2 = NC * 256 * LPT >= next_pow2(n_off),
// zero-padded), thread t of it LPT contiguous leaves -- a power-of-two-aligned partition, so
// thread-local trees, xor butterflies over the lanes, over the warps and finally over the NC
// CTA partials reproduce the balanced tree over page ids exactly.  The cluster exchanges, over
// DSMEM, the per-head maxima, the CTA subtree sums, the radix histograms (every CTA's warp 0
// sums them redundantly, so all CTAs reach the same boundary without another round), the
// <= 32 boundary-bin keys and the (#gt, #eq) totals; each CTA then scatters its selected page
// ids into the leader's list in ascending order and the leader finishes the unit (delta, slots,
// page list) and publishes X.ready[u] (release) for the attention kernel, which runs
// concurrently and waits on it only for corrected units and for the commit.
//
// The CTA is small on purpose (256 threads, <= 64 registers, ~17 KiB of shared memory: packed
// 16-bit histogram bins, membership in R by binary search over R's sorted page list): it shares
// an SM with two attention CTAs, so the attention of the units that are not corrected is never
// held back by the selection.
//
// Every floating-point step that decides an index follows the canonical fp32 recipe (DESIGN.md
// §3) with explicit round-to-nearest intrinsics, so page indices are bit-identical to the CPU
// oracle.
#include <algorithm>
#include <cstdlib>

#include "select_core.cuh"

namespace fkv {

constexpr int kSelThreads = 256;
constexpr int kSelWarps = kSelThreads / 32;

// flag_src: 1 = the pre kernel decided the correction flag (L.flags), 0 = decided here (CFR-10 over
// q_i and q_{i-1}).  list_all: 1 = write the attention page list of every unit (primitive API,
// paper-order recall mode), 0 = of the corrected units only (the others attend their resident set).
// part >= 0 (speculative step): the unit of cluster i is part_unit(part, i) -- part 0 the corrected
// units, part 1 the others; instead of waiting for the whole score grid (PDL), each unit waits for
// its own score items.
template <int LPT, int GM, int NC, int NT>
__global__ void __launch_bounds__(NT, NT == kSelThreads && LPT * GM <= 16 ? 4 : 1)
    fkv_select_kernel(FkvDims D, FkvLayer L, FkvScratch X, const uint16_t* __restrict__ q,
                      int32_t* __restrict__ pages_out, uint8_t* __restrict__ corrected_out, int flag_src,
                      int list_all, int part, int pending) {
    constexpr int W = NT / 32;
    const int rank = NC > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int u = part_unit(D, L, part, (int)blockIdx.x / NC);
    if (u < 0) return;  // cluster-uniform: no unit at this index in this part
    const int b = u / D.n_kv, m = u % D.n_kv, G = D.G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool leader = rank == 0;
    __shared__ SelSmem<W, GM, NC> S;
    __shared__ UnitSmem U;
    if (tid == 0) trace_stamp(X.trace, 1, blockIdx.x, 0);
    // ---- state (the resident set R of the previous step): before the PDL wait
    const int res_valid = D.full_refresh ? 0 : L.res_valid[u];
    const int res_front = L.res_front[u];
    int n_res = 0;
    if (leader) n_res = stage_resident<NT>(D, L, u, res_valid, U);
    rank_clear<NT>(S);
    if (tid == 0) trace_stamp(X.trace, 1, blockIdx.x, 4);
    if constexpr (NC > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    // the context as published before the scores (pre kernel / append kernel), or with the token the
    // score grid appended (pending)
    const int Lc = L.ctx[u] + pending;
    const int n_off = pending ? max(L.n_off[u], frontier_for(D, Lc)) : L.n_off[u];
    const int n_cand = n_off - D.n_sink;
    const bool rank_all = n_cand <= D.K;  // A-11: every candidate selected, no ranking (cluster-uniform)
    if (part >= 0) {  // this unit's score items are written (acquire)
        pdl_trigger();
        if (!rank_all && tid == 0) {
            const int cp = part == 0 ? kScoreCtaPagesFast : kScoreCtaPages;
            spin_until_ge(L.score_done + u, (n_off + cp - 1) / cp);
        }
    } else {
        pdl_wait();  // the scores (previous kernel) are complete; q_i is ready
        pdl_trigger();
    }
    if (tid == 0) trace_stamp(X.trace, 1, blockIdx.x, 5);
    if constexpr (NC > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every CTA started
    __syncthreads();
    if (tid == 0) trace_stamp(X.trace, 1, blockIdx.x, 6);
    // the flag decided before this kernel (score grid / pre kernel, complete here): its load
    // latency overlaps the ranking instead of sitting between the ranking and finish_unit
    const int flag_pre = (flag_src != 0 && tid == 0) ? (int)__ldcg(L.flags + u) : 0;
    int cnt;
    if (rank_all) {
        if (!leader) return;
        for (int i = tid; i < D.K; i += NT) S.sel[i] = i < n_cand ? D.n_sink + i : -1;
        cnt = n_cand > 0 ? n_cand : 0;
        __syncthreads();
    } else {
        const int jb = (rank * NT + tid) * LPT;
        const float* sg = L.scores + (size_t)u * G * D.n_page_max;
        float sv[GM][LPT];
#pragma unroll
        for (int g = 0; g < GM; ++g)
#pragma unroll
            for (int l = 0; l < LPT; ++l) {
                const int j = jb + l;
                sv[g][l] = (g < G && j >= D.n_sink && j < n_off) ? __ldcg(sg + (size_t)g * D.n_page_max + j)
                                                                  : -INFINITY;
            }
        if (tid == 0) trace_stamp(X.trace, 1, blockIdx.x, 1);
        rank_unit<LPT, GM, NC, NT>(D, rank, n_off, sv, S, X.trace, blockIdx.x);
        if (!leader) return;
        cnt = D.K;
    }
    if (tid == 0) trace_stamp(X.trace, 1, blockIdx.x, 2);
    // ---- leader: a1 flag (when not decided by the pre kernel), a4 delta + page list
    if (flag_src == 0 && warp == W - 1 && lane < G) {
        const size_t row = ((size_t)b * D.n_qo + m * G + lane) * kHeadDim;
        U.cos[lane] = cos_cfr10(q + row, L.q_prev + row);
    }
    __syncthreads();
    if (tid == 0) {
        int flag;
        if (flag_src == 0) {
            const float pooled = pool_cos(U.cos, G, D.corr_pool);
            flag = correction_flag(D, pooled, res_valid);
            L.flags[u] = (uint8_t)flag;
            L.cbar[u] = pooled;
        } else {
            flag = flag_pre;
        }
        U.flag = flag;
        if (corrected_out) corrected_out[u] = (uint8_t)flag;
    }
    __syncthreads();
    const int flag = U.flag;
    finish_unit<NT>(D, L, X, u, Lc, n_off, S.sel, cnt, U, n_res, res_front, flag, list_all, pages_out);
    // ---- publish (corrected units, or every unit when list_all -- the mode-0 attention and the
    // combine kernel reset it): the CTA barrier (end of finish_unit) orders every thread's writes
    // before thread 0's release (cumulative).  A unit that is not corrected must not leave ready
    // set: its flag may be set at the next step, before that step's select rewrote its page list.
    if (tid == 0) {
        if (list_all || flag) st_release(X.ready + u, 1);
        trace_stamp(X.trace, 1, blockIdx.x, 3);
    }
}

template <int LPT, int GM, int NC, int NT>
static cudaError_t launch_sel(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              int32_t* pages_out, uint8_t* corrected_out, int flag_src, int list_all, int part,
                              bool pdl, int prio, cudaStream_t s, int pending) {
    auto kern = fkv_select_kernel<LPT, GM, NC, NT>;
    const size_t smem = 0;
    cudaError_t e = func_smem((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.U * NC);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[3];
    int na = 0;
    if (prio) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na].val.priority = prio;
        ++na;
    }
    if (NC > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = NC;
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
    return cudaLaunchKernelEx(&cfg, kern, D, L, X, q, pages_out, corrected_out, flag_src, list_all, part, pending);
}

template <int LPT, int NC, int NT = kSelThreads>
static cudaError_t launch_sel_g(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                int32_t* pages_out, uint8_t* corrected_out, int flag_src, int list_all, int part,
                                bool pdl, int prio, cudaStream_t s, int pending) {
    if (D.G <= 1) return launch_sel<LPT, 1, NC, NT>(D, L, X, q, pages_out, corrected_out, flag_src, list_all, part, pdl, prio, s, pending);
    if (D.G <= 2) return launch_sel<LPT, 2, NC, NT>(D, L, X, q, pages_out, corrected_out, flag_src, list_all, part, pdl, prio, s, pending);
    if (D.G <= 4) return launch_sel<LPT, 4, NC, NT>(D, L, X, q, pages_out, corrected_out, flag_src, list_all, part, pdl, prio, s, pending);
    return launch_sel<LPT, 8, NC, NT>(D, L, X, q, pages_out, corrected_out, flag_src, list_all, part, pdl, prio, s, pending);
}

// nc = CTAs per unit (1, 2, 4, 8), lpt = leaves per thread: nc * 256 * lpt >= next_pow2(n_off) for
// every n_off the handle can reach (a larger zero-padded tree gives the same Z, CFR-6)
cudaError_t launch_select(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                          int32_t* pages_out, uint8_t* corrected_out, int flag_src, int list_all, int part,
                          int nc, int lpt, bool pdl, int prio, cudaStream_t s, int pending, int nt) {
#define FKV_SEL(LP, N) \
    return launch_sel_g<LP, N>(D, L, X, q, pages_out, corrected_out, flag_src, list_all, part, pdl, prio, s, pending)
#define FKV_SELW(LP) \
    return launch_sel_g<LP, 1, 1024>(D, L, X, q, pages_out, corrected_out, flag_src, list_all, part, pdl, prio, s, \
                                     pending)
#define FKV_SELM(LP) \
    return launch_sel_g<LP, 1, 512>(D, L, X, q, pages_out, corrected_out, flag_src, list_all, part, pdl, prio, s, \
                                    pending)
    if (nc == 1 && nt == 512) {
        switch (lpt) {
            case 1: FKV_SELM(1);
            case 2: FKV_SELM(2);
            case 4: FKV_SELM(4);
            case 8: FKV_SELM(8);
            default: return cudaErrorInvalidValue;
        }
    }
    if (nc == 1 && nt == 1024) {  // one wide CTA per unit (few, short per-thread chains)
        switch (lpt) {
            case 1: FKV_SELW(1);
            case 2: FKV_SELW(2);
            case 4: FKV_SELW(4);
            case 8: FKV_SELW(8);
            default: return cudaErrorInvalidValue;
        }
    }
    if (nc == 1) {
        switch (lpt) {
            case 1: FKV_SEL(1, 1);
            case 2: FKV_SEL(2, 1);
            case 4: FKV_SEL(4, 1);
            case 8: FKV_SEL(8, 1);
            case 16: FKV_SEL(16, 1);
            case 32: FKV_SEL(32, 1);
            default: return cudaErrorInvalidValue;
        }
    }
    if (nc == 2) {
        switch (lpt) {
            case 1: FKV_SEL(1, 2);
            case 2: FKV_SEL(2, 2);
            case 4: FKV_SEL(4, 2);
            default: return cudaErrorInvalidValue;
        }
    }
    if (nc == 4) {
        switch (lpt) {
            case 1: FKV_SEL(1, 4);
            case 2: FKV_SEL(2, 4);
            case 4: FKV_SEL(4, 4);
            default: return cudaErrorInvalidValue;
        }
    }
    if (nc == 8) {
        switch (lpt) {
            case 1: FKV_SEL(1, 8);
            case 2: FKV_SEL(2, 8);
            case 4: FKV_SEL(4, 8);
            default: return cudaErrorInvalidValue;
        }
    }
#undef FKV_SEL
#undef FKV_SELW
#undef FKV_SELM
    return cudaErrorInvalidValue;
}

}  // namespace fkv
