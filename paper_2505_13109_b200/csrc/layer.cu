// layer.cu -- the fused decode step of one layer: every row of SURVEY §8(a) for one unit in one
// cluster of C CTAs (4 warps each), one launch per layer.
//
//   a1  correction check (CFR-10) and a9 append: the leader CTA, first
//   a7  sparse decode attention over
//         the resident set R = S_{i-1} when the unit is not corrected (speculative
//         retrieval -- the pages selected with q_{i-1} are used at step i), at once;
//         S_i when it is corrected, after a2-a4 below; its missing pages are read
//         from the pinned host pool and written back to their slots in the same pass (direct mode)
//   a2  page scoring (CFR-2/3): each thread scores the LPT contiguous pages it owns as
//       leaves of the selection tree -- the scores never leave its registers
//   a3  per-head softmax + MeanS pooling (CFR-4..8) and a4 top-K + delta + slots
//       (P:100-101): rank_unit / finish_unit over the cluster (select_core.cuh)
//   a8  R := S_i, q_prev := q_i and the new context length, at the end
//
// A unit that is not corrected attends R first and selects S_i (for step i+1) afterwards, so the
// selection is off its critical path; a corrected unit selects first.  There is no other kernel
// between layers: no score -> select -> attention hand-offs, no co-residency of a select grid with
// the attention grid (both measured costly on B200).  The background recall of
// S_i minus R (row a5) follows on the recall stream.
//
// Shared memory: the 96 KiB attention ring region of the CTA is reused phase by phase -- the
// leader's append staging, the attention slabs (and then the partial records), the scoring rings
// and the q pairs, and the selection's histogram / resident-set state.
#include <cooperative_groups.h>

#include <algorithm>

#include "append_unit.cuh"
#include "attn_core.cuh"
#include "select_core.cuh"

namespace fkv {

constexpr int kLyWarps = 4;
constexpr int kLyThreads = kLyWarps * 32;
constexpr int kLyNst = 3;                                        // attention slab stages per warp
constexpr int kLyWarpBytes = kLyNst * kSlabBytes;                 // 24 KiB per warp
constexpr int kLySmem = kLyWarps * kLyWarpBytes;                  // 96 KiB
constexpr int kLyScoreRing = 20 * 1024;                           // score ring bytes per warp
constexpr int kLyQOff = kLyWarps * kLyScoreRing;                  // q pairs of the scoring (8 KiB)
constexpr int kLyKeyOff = 40 * 1024;                              // the leader's key buffer (select phase)
static_assert(kLyQOff + 8 * 1024 <= kLySmem, "score phase layout");

__device__ __forceinline__ unsigned long long ly_pk2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void ly_ffma2(unsigned long long& acc, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ uint32_t ly_u4w(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// a2 for this thread's leaves jb .. jb + LPT - 1 (the pages its warp streams: 32 * LPT consecutive
// pages), every head of the group: sv[g][l] = fl(u * r) (CFR-2/3) or -inf outside [n_sink, n_off).
// Head pairs share one FFMA2 (u_pair = fma({q-_h, q-_h'}, {mn, mn}, fma({q+_h, q+_h'}, {mx, mx}, u))),
// one of the two products a signed zero: CFR-2's single rounding per channel.  region: this warp's
// 24 KiB (ring: first 16 KiB); q pairs staged in CTA warp 0's region tail.
template <int GM, int LPT>
__device__ __forceinline__ void score_leaves(const FkvDims& D, const FkvLayer& L, int u, int jb, int n_off,
                                             const uint16_t* __restrict__ q, uint8_t* s_stage, uint64_t* sbar,
                                             float (&sv)[GM][LPT]) {
    constexpr int GP = GM >= 2 ? GM / 2 : 1;                      // head pairs
    constexpr int SB = 2 * 32 * LPT * 16;                         // stage: {min, max} x 32 LPT pages x 8 ch
    constexpr int NS = kLyScoreRing / SB < 8 ? kLyScoreRing / SB : 8;  // ring depth (bytes in flight)
    static_assert(NS >= 2, "score ring");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, G = D.G;
    const int b = u / D.n_kv, m = u % D.n_kv;
    float4* s_q = reinterpret_cast<float4*>(s_stage + kLyQOff);  // [128][GP]
    uint8_t* ring = s_stage + warp * kLyScoreRing;
    const int jw = jb - lane * LPT;                               // first page of this warp
    const bool active = jw < n_off && jw + 32 * LPT > D.n_sink;
    auto issue = [&](int slot, int c8) {
        mbar_expect_tx(&sbar[slot], SB);
        bulk_g2s(ring + slot * SB, L.summ + summ_off(D, u, c8, 0, jw), SB / 2, &sbar[slot]);
        bulk_g2s(ring + slot * SB + SB / 2, L.summ + summ_off(D, u, c8, 1, jw), SB / 2, &sbar[slot]);
    };
    __syncthreads();  // the region's previous contents (records, slabs) are dead in every warp
    if (active && lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
        for (int s2 = 0; s2 < NS; ++s2) issue(s2, s2);
    }
    // q pairs: thread (pair hp, channel group c8)
    for (int i = threadIdx.x; i < GP * (kHeadDim / 8); i += blockDim.x) {
        const int hp = i / (kHeadDim / 8), c8 = i % (kHeadDim / 8);
        const uint16_t* qg = q + ((size_t)b * D.n_qo + m * G) * kHeadDim + c8 * 8;
        float x[2][8];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int h = 2 * hp + t;
#pragma unroll
            for (int e = 0; e < 8; ++e) x[t][e] = 0.0f;
            if (h >= G) continue;  // the zero head of an odd group / an unused bucket head
            if (D.pool >= 4) {  // MeanQ / MaxQ (f3, reading R-12): every head scores the pooled query
                uint4 w = *reinterpret_cast<const uint4*>(qg);
#pragma unroll
                for (int e = 0; e < 8; ++e) x[t][e] = (e & 1) ? bf16_hi(ly_u4w(w, e >> 1)) : bf16_lo(ly_u4w(w, e >> 1));
                for (int g = 1; g < G; ++g) {
                    w = *reinterpret_cast<const uint4*>(qg + (size_t)g * kHeadDim);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float y = (e & 1) ? bf16_hi(ly_u4w(w, e >> 1)) : bf16_lo(ly_u4w(w, e >> 1));
                        x[t][e] = D.pool == 4 ? __fadd_rn(x[t][e], y) : (y > x[t][e] ? y : x[t][e]);
                    }
                }
                if (D.pool == 4)
#pragma unroll
                    for (int e = 0; e < 8; ++e) x[t][e] = __fdiv_rn(x[t][e], (float)G);
            } else {
                const uint4 w = *reinterpret_cast<const uint4*>(qg + (size_t)h * kHeadDim);
#pragma unroll
                for (int e = 0; e < 8; ++e) x[t][e] = (e & 1) ? bf16_hi(ly_u4w(w, e >> 1)) : bf16_lo(ly_u4w(w, e >> 1));
            }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float a = x[0][e], c = x[1][e];
            s_q[(c8 * 8 + e) * GP + hp] = make_float4(a >= 0.0f ? a : 0.0f, c >= 0.0f ? c : 0.0f,
                                                      a >= 0.0f ? 0.0f : a, c >= 0.0f ? 0.0f : c);
        }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < GM; ++g)
#pragma unroll
        for (int l = 0; l < LPT; ++l) sv[g][l] = -INFINITY;
    if (!active) return;
    unsigned long long acc[LPT][GP];
#pragma unroll
    for (int l = 0; l < LPT; ++l)
#pragma unroll
        for (int hp = 0; hp < GP; ++hp) acc[l][hp] = 0ull;
#pragma unroll 1
    for (int c8 = 0; c8 < kHeadDim / 8; ++c8) {
        const int slot = c8 % NS;
        mbar_wait(&sbar[slot], (uint32_t)(c8 / NS) & 1u);
        const uint4* st = reinterpret_cast<const uint4*>(ring + slot * SB);
        uint4 mn[LPT], mx[LPT];
#pragma unroll
        for (int l = 0; l < LPT; ++l) {  // page jb + l: entry lane * LPT + l of the stage
            mn[l] = st[lane * LPT + l];
            mx[l] = st[32 * LPT + lane * LPT + l];
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int c = c8 * 8 + e;
            unsigned long long mx2[LPT], mn2[LPT];
#pragma unroll
            for (int l = 0; l < LPT; ++l) {
                const float fx = (e & 1) ? bf16_hi(ly_u4w(mx[l], e >> 1)) : bf16_lo(ly_u4w(mx[l], e >> 1));
                const float fn = (e & 1) ? bf16_hi(ly_u4w(mn[l], e >> 1)) : bf16_lo(ly_u4w(mn[l], e >> 1));
                mx2[l] = ly_pk2(fx, fx);
                mn2[l] = ly_pk2(fn, fn);
            }
#pragma unroll
            for (int hp = 0; hp < GP; ++hp) {
                const float4 qq = s_q[c * GP + hp];
                const unsigned long long qp = ly_pk2(qq.x, qq.y), qm = ly_pk2(qq.z, qq.w);
#pragma unroll
                for (int l = 0; l < LPT; ++l) {
                    ly_ffma2(acc[l][hp], qp, mx2[l]);
                    ly_ffma2(acc[l][hp], qm, mn2[l]);
                }
            }
        }
        __syncwarp();  // every lane is done with this stage
        if (lane == 0 && c8 + NS < kHeadDim / 8) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(slot, c8 + NS);
        }
    }
#pragma unroll
    for (int l = 0; l < LPT; ++l) {
        const int j = jb + l;
        if (j >= D.n_sink && j < n_off) {
#pragma unroll
            for (int g = 0; g < GM; ++g) {
                if (g < G) {
                    const unsigned long long a = acc[l][GM >= 2 ? g >> 1 : 0];
                    const float uu = (g & 1) ? __uint_as_float((uint32_t)(a >> 32)) : __uint_as_float((uint32_t)a);
                    sv[g][l] = __fmul_rn(uu, D.score_r);  // CFR-3
                }
            }
        }
    }
}

template <int C, int GM, int LPT>
__global__ void __launch_bounds__(kLyThreads, 2)
    fkv_layer_kernel(FkvDims D, FkvLayer L, FkvScratch X, const uint16_t* __restrict__ q,
                     const uint16_t* __restrict__ k_new, const uint16_t* __restrict__ v_new, float* __restrict__ out,
                     const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_h) {
    constexpr int W = kLyWarps, NW = W * C, NT = kLyThreads;
    extern __shared__ __align__(1024) uint8_t s_stage[];
    __shared__ __align__(8) uint64_t abar[W][kLyNst];  // attention slab ring
    __shared__ __align__(8) uint64_t sbar[W][8];       // scoring ring
    __shared__ int s_flag;
    __shared__ float s_cos[kMaxG];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int u = blockIdx.x / C;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int G = D.G, b = u / D.n_kv, m = u % D.n_kv, K = D.K;
    const bool leader = rank == 0;
    auto* S = reinterpret_cast<SelSmem<W, GM, C>*>(s_stage);                       // select phase
    auto* U = reinterpret_cast<UnitSmem*>(s_stage + kLyWarpBytes);                // select phase (leader)
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kLyNst; ++i) mbar_init(&abar[warp][i], 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) mbar_init(&sbar[warp][i], 1);
        fence_mbar_init();
    }
    cl.sync();  // every CTA of the cluster has started (DSMEM) and initialised its barriers
    // ---- state of the previous step (before the PDL wait): context, frontier, R
    const int ctx0 = L.ctx[u];
    const int Lc = ctx0 + 1;  // this step's token is appended below
    const int n_off = max(L.n_off[u], frontier_for(D, Lc));
    const int res_valid = D.full_refresh ? 0 : L.res_valid[u];
    const int res_front = L.res_front[u];
    int r_page[2] = {-1, -1}, r_slot[2] = {-1, -1};  // R (the leader stages it for the delta)
    if (leader && res_valid)
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (tid + i * NT < K) {
                r_page[i] = L.res_pages[(size_t)u * K + tid + i * NT];
                r_slot[i] = L.res_slot[(size_t)u * K + tid + i * NT];
            }
    const int n_res = res_valid ? L.res_cnt[u] : 0;
    if (tid == 0) trace_stamp(X.trace, 4, blockIdx.x, 0);
    pdl_wait();  // q_i and this step's token are the layer's inputs
    pdl_trigger();
    // ---- a1 + a9 (leader): correction flag, append; the flag reaches every CTA over DSMEM
    if (leader) {
        if (tid < G) {
            const size_t row = ((size_t)b * D.n_qo + m * G + tid) * kHeadDim;
            s_cos[tid] = cos_cfr10(q + row, L.q_prev + row);
        }
        __syncthreads();
        if (tid == 0) {
            const float pooled = pool_cos(s_cos, G, D.corr_pool);
            const int flag = correction_flag(D, pooled, res_valid);
            L.flags[u] = (uint8_t)flag;
            L.cbar[u] = pooled;
            for (int r = 0; r < C; ++r) *cl.map_shared_rank(&s_flag, r) = flag;
        }
        append_unit(D, L, u, ctx0, k_new, v_new, 1, reinterpret_cast<uint4*>(s_stage));
        asm volatile("fence.proxy.async.global;" ::: "memory");  // the ring page is read by TMA below
    }
    cl.sync();
    if (tid == 0) trace_stamp(X.trace, 4, blockIdx.x, 1);
    const int flag = s_flag;
    const int n_cand = n_off - D.n_sink;
    const bool rank_all = n_cand <= K;  // A-11 (cluster-uniform)
    // ---- a2-a4: scores in registers, then the cluster's ranking and the leader's delta
    // the leader's resident set and free slots for the delta (from the registers loaded at the start)
    auto stage_r = [&]() {
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (tid + i * NT < K) {
                U->res[tid + i * NT] = r_page[i];
                U->res_slot[tid + i * NT] = r_slot[i];
            }
        for (int i = tid; i < 2 * K; i += NT) U->used[i] = 0;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 2; ++i)
            if (r_page[i] >= 0) U->used[r_slot[i]] = 1;
        __syncthreads();
        if (warp == 0) {  // free slots (not in R), ascending -- slot double-buffering
            int nfree = 0;
            for (int base = 0; base < 2 * K; base += 32) {
                const int sl = base + lane;
                const bool fr = sl < 2 * K && !U->used[sl];
                const unsigned bal = __ballot_sync(0xffffffffu, fr);
                if (fr) U->free_[nfree + __popc(bal & ((1u << lane) - 1u))] = sl;
                nfree += __popc(bal);
            }
        }
        __syncthreads();
    };
    auto select_phase = [&](int list_flag) {
        if (rank_all) {
            __syncthreads();
            if (leader) {
                stage_r();
                for (int i = tid; i < K; i += NT) S->sel[i] = i < n_cand ? D.n_sink + i : -1;
                __syncthreads();
                finish_unit<NT>(D, L, X, u, Lc, n_off, S->sel, n_cand > 0 ? n_cand : 0, *U, n_res, res_front,
                                list_flag, 0, nullptr);
            }
            return;
        }
        float sv[GM][LPT];
        const int jb = (rank * NT + tid) * LPT;
        score_leaves<GM, LPT>(D, L, u, jb, n_off, q, s_stage, sbar[warp], sv);
        if (tid == 0) trace_stamp(X.trace, 4, blockIdx.x, 2);
        __syncthreads();  // the rings / q pairs are dead: the select state takes the region
        rank_clear<NT>(*S);
        csync<C>();  // every CTA cleared its state before any DSMEM store
        // a3 over the cluster (per-head max and Z exchanged), then every key to the leader, which
        // ranks alone (no further cluster rounds)
        uint32_t key[LPT];
        softmax_keys<LPT, GM, C, NT>(D, rank, n_off, sv, *S, key, X.trace, blockIdx.x);
        uint32_t* kbuf = reinterpret_cast<uint32_t*>(s_stage + kLyKeyOff);
        uint32_t* kb0 = cl.map_shared_rank(kbuf, 0);
#pragma unroll
        for (int l = 0; l < LPT; ++l) kb0[jb + l] = key[l];
        csync<C>();  // the leader holds every key
        if (tid == 0) trace_stamp(X.trace, 4, blockIdx.x, 3);
        if (leader) {
            constexpr int LK = LPT * C;
            uint32_t k2[LK];
#pragma unroll
            for (int l = 0; l < LK; ++l) k2[l] = kbuf[tid * LK + l];
            topk_keys<LK, 1, NT>(D, 0, n_off, k2, *S, X.trace, blockIdx.x);
            stage_r();
            finish_unit<NT>(D, L, X, u, Lc, n_off, S->sel, K, *U, n_res, res_front, list_flag, 0, nullptr);
        }
        if (tid == 0) trace_stamp(X.trace, 4, blockIdx.x, 4);
    };
    // ---- a7: this warp's share of the unit's page list, in 16-token slabs
    auto attend = [&](auto src, int n_pages) {
        const int k = rank * W + warp;
        const int spp = D.p >> 4, TS = D.P_max * spp;
        const int sa = (int)((long long)k * TS / NW), sb = (int)((long long)(k + 1) * TS / NW);
        const int pa = sa / spp, pbc = (sb + spp - 1) / spp;
        const int skip = sa - pa * spp, trim = pbc * spp - sb;
        float oacc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) oacc[i][j] = 0.0f;
        float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.0f, 0.0f};
        uint4 qa[2][2];
        load_q_frags(D, q, u, qa);
        uint32_t phase_bits = 0u;
        uint8_t* ring = s_stage + warp * kLyWarpBytes;
        __syncthreads();  // the region's previous contents are dead in every warp
        if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        const int pe = min(pbc, n_pages);
        attend_pages<kLyNst>(D, X, qa, &tmap, &tmap_h, src, pa, pe, ring, abar[warp], phase_bits, m_run, l_run, oacc, 5,
                             blockIdx.x * W + warp, 0, skip, pe == pbc ? trim : 0);
        __syncwarp();
        write_record(reinterpret_cast<float*>(ring), G, oacc, m_run, l_run);
        cl.sync();  // every record of the unit is in its CTA's shared memory
        if (leader) {
            for (int e = tid; e < G * (kHeadDim / 4); e += NT) {
                const float4 o4 = merge_records<NW>(G, e, [&](int r) {
                    return cl.map_shared_rank(reinterpret_cast<const float*>(s_stage + (r % W) * kLyWarpBytes),
                                              r / W);
                });
                const size_t row = (size_t)b * D.n_qo + m * G + e / (kHeadDim / 4);
                reinterpret_cast<float4*>(out + row * kHeadDim)[e % (kHeadDim / 4)] = o4;
            }
        }
        cl.sync();  // the leader has read every record
        if (tid == 0) trace_stamp(X.trace, 4, blockIdx.x, 5);
    };
    if (!flag) {
        // not corrected: attend R = S_{i-1} and select S_i for step i+1 -- independent, so
        // units alternate the order: the two CTAs an SM holds then mostly run different phases (the
        // HBM-bound attention beside the latency-bound scoring / ranking) instead of the same one
        const ResSrc rsrc = res_src(D, L, u, Lc);
        if ((u & 1) && !(D.dbg_order & 1)) {
            select_phase(0);
            attend(rsrc, rsrc.count());
        } else {
            attend(rsrc, rsrc.count());
            select_phase(0);
        }
    } else {
        // corrected: select S_i first, then attend it; the leader's page list (global) is
        // visible to the cluster after the barrier
        select_phase(1);
        cl.sync();
        const TableSrc tsrc{X.page_rows + (size_t)u * D.P_max, X.page_valid + (size_t)u * D.P_max,
                            X.page_dst + (size_t)u * D.P_max};
        attend(tsrc, __ldcg(X.page_cnt + u));
    }
    // ---- a8 (leader): q_prev := q_i, R := S_i, the new context length
    if (leader) {
        __syncthreads();
        const size_t row0 = ((size_t)b * D.n_qo + m * G) * kHeadDim;
        for (int i = tid; i < G * (kHeadDim / 8); i += NT)
            reinterpret_cast<uint4*>(L.q_prev + row0)[i] = reinterpret_cast<const uint4*>(q + row0)[i];
        for (int i = tid; i < K; i += NT) {
            L.res_pages[(size_t)u * K + i] = L.pend_pages[(size_t)u * K + i];
            L.res_slot[(size_t)u * K + i] = L.pend_slot[(size_t)u * K + i];
        }
        if (tid == 0) {
            L.res_front[u] = L.pend_front[u];
            L.res_cnt[u] = L.pend_cnt[u];
            L.res_valid[u] = 1;
            L.pend_valid[u] = 0;
            L.ctx[u] = Lc;
            L.n_off[u] = n_off;
        }
    }
    if (tid == 0) trace_stamp(X.trace, 4, blockIdx.x, 6);
}

template <int C, int GM, int LPT>
static cudaError_t launch_layer_t(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                  const uint16_t* k_new, const uint16_t* v_new, float* out, const CUtensorMap& tmap,
                                  const CUtensorMap& tmap_h, bool pdl, cudaStream_t s) {
    auto kern = fkv_layer_kernel<C, GM, LPT>;
    cudaError_t e = func_smem((const void*)kern, kLySmem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.U * C);
    cfg.blockDim = dim3(kLyThreads);
    cfg.dynamicSmemBytes = kLySmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = C;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, D, L, X, q, k_new, v_new, out, tmap, tmap_h);
}

// c = CTAs per unit (2, 4, 8), lpt = leaves (pages) per thread with c * 128 * lpt >= the tree size
bool layer_supported(const FkvDims& D, int c, int lpt) {
    return (c == 2 || c == 4 || c == 8) && (lpt == 1 || lpt == 2 || lpt == 4 || lpt == 8) && D.G <= 8 &&
           D.n_win >= 1 && D.direct;
}

cudaError_t launch_layer(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                         const uint16_t* k_new, const uint16_t* v_new, float* out, const CUtensorMap& tmap,
                         const CUtensorMap& tmap_h, int c, int lpt, bool pdl, cudaStream_t s) {
#define FKV_LY(CC, GMV, LP) return launch_layer_t<CC, GMV, LP>(D, L, X, q, k_new, v_new, out, tmap, tmap_h, pdl, s)
#define FKV_LY_L(CC, GMV)           \
    do {                            \
        if (lpt == 1) FKV_LY(CC, GMV, 1); \
        if (lpt == 2) FKV_LY(CC, GMV, 2); \
        if (lpt == 4) FKV_LY(CC, GMV, 4); \
        FKV_LY(CC, GMV, 8);         \
    } while (0)
#define FKV_LY_G(CC)                       \
    do {                                   \
        if (D.G <= 4) FKV_LY_L(CC, 4);     \
        FKV_LY_L(CC, 8);                   \
    } while (0)
    if (c == 2) FKV_LY_G(2);
    if (c == 4) FKV_LY_G(4);
    FKV_LY_G(8);
#undef FKV_LY_G
#undef FKV_LY_L
#undef FKV_LY
}

}  // namespace fkv
