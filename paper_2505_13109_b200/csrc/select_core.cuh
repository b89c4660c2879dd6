// select_core.cuh -- rows a3 / a4 as device functions of the select kernel (select.cu):
//
//   rank_unit    a3 + a4: per-head softmax over the candidate pages (CFR-4..7), group pooling
//                (MeanS / MaxS, CFR-8; the QK variants pooled before), top-K with lowest-id ties
//                (CFR-9) -- PAPER.md P:232-234
//   finish_unit  a4: delta vs the resident set (A-18), slot assignment (slot double-buffering),
//                fetch list, pending selection, the attention page list of a corrected unit
//                 -- P:296
//
// One cluster of NC CTAs of NT threads per unit.  CTA r owns the leaves (page ids)
// [r P2/NC, (r+1) P2/NC) of the pairwise tree of CFR-6 (P2 = NC * NT * LPT, zero-padded), thread t
// of it LPT contiguous leaves -- a power-of-two-aligned partition, so thread-local trees, xor
// butterflies over the lanes, over the warps and finally over the NC CTA partials reproduce the
// balanced tree over page ids exactly.  The cluster exchanges over DSMEM the per-head maxima, the
// CTA subtree sums, the radix histograms (every CTA's warp 0 sums them redundantly, so all CTAs
// reach the same boundary without another round), the <= 32 boundary-bin keys and the (#gt, #eq)
// totals; each CTA then scatters its selected page ids into the leader's list in ascending order.
//
// Every floating-point step that decides an index follows the canonical fp32 recipe (DESIGN.md
// §3) with explicit round-to-nearest intrinsics, so page indices are bit-identical to the CPU
// oracle.
#pragma once
#include <cooperative_groups.h>

#include "fkv_internal.cuh"

namespace fkv {

namespace cg = cooperative_groups;

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

constexpr int kMaxK = 256;
constexpr int kHistBins = 4096;  // 12-bit radix digits; two 16-bit counters per 32-bit word

// cluster-wide barrier with release/acquire of shared memory (a CTA barrier when NC = 1): the CTA
// barrier orders every thread's writes before thread 0's cluster-scope fence, so the other
// threads arrive relaxed (one fence per CTA instead of one per thread)
template <int NC>
__device__ __forceinline__ void csync() {
    if constexpr (NC > 1) {
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("fence.acq_rel.cluster;" ::: "memory");
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
}
__device__ __forceinline__ int hist_get(const uint32_t* h2, int bin) {
    return (int)((h2[bin >> 1] >> ((bin & 1) * 16)) & 0xffffu);
}
// shared-memory pointer of CTA r of the cluster (DSMEM)
template <int NC, class T>
__device__ __forceinline__ T* rmt(T* p, int r) {
    if constexpr (NC == 1)
        return p;
    else
        return cg::this_cluster().map_shared_rank(p, r);
}

// Shared memory of rank_unit (every CTA of the cluster)
template <int W, int GM, int NC>
struct SelSmem {
    float redm[W][GM], redz[W][GM];
    float cm[NC][GM], cz[NC][GM];
    __align__(16) uint32_t h[kHistBins / 2];  // packed 16-bit bin counters
    __align__(16) int sup[kHistBins / 32];
    uint32_t bk[32];
    int bid[32], bn;
    int dig[4];
    unsigned wsum[W];
    unsigned ctot[NC];
    int sel[kMaxK];  // the leader's S_i (ascending, -1 padded)
};

// Shared memory of finish_unit (the leader CTA): the resident set and the free slots
struct UnitSmem {
    int res[kMaxK], res_slot[kMaxK], isfetch[kMaxK], pslot[kMaxK];
    int free_[2 * kMaxK];
    unsigned char used[2 * kMaxK];
    float cos[kMaxG];
    int flag;
};

// Stage R (state of the previous step) and the free-slot list of unit u; leader CTA, every thread.
// Ends with a CTA barrier.  Returns res_cnt (0 when R is not valid: bootstrap, A-12).
template <int NT>
__device__ __forceinline__ int stage_resident(const FkvDims& D, const FkvLayer& L, int u, int res_valid, UnitSmem& U) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, K = D.K;
    for (int i = tid; i < K; i += NT) {
        U.res[i] = res_valid ? L.res_pages[(size_t)u * K + i] : -1;
        U.res_slot[i] = res_valid ? L.res_slot[(size_t)u * K + i] : -1;
    }
    for (int i = tid; i < 2 * K; i += NT) U.used[i] = 0;
    __syncthreads();
    for (int i = tid; i < K; i += NT)
        if (U.res[i] >= 0) U.used[U.res_slot[i]] = 1;
    __syncthreads();
    if (warp == 0) {  // free slots (not in R), ascending -- slot double-buffering
        int nfree = 0;
        for (int base = 0; base < 2 * K; base += 32) {
            const int sl = base + lane;
            const bool fr = sl < 2 * K && !U.used[sl];
            const unsigned bal = __ballot_sync(0xffffffffu, fr);
            if (fr) U.free_[nfree + __popc(bal & ((1u << lane) - 1u))] = sl;
            nfree += __popc(bal);
        }
    }
    __syncthreads();
    return res_valid ? L.res_cnt[u] : 0;
}

// Clear the histogram state before rank_unit (every CTA; a CTA barrier must follow before use).
template <int NT, int W, int GM, int NC>
__device__ __forceinline__ void rank_clear(SelSmem<W, GM, NC>& S) {
    for (int i = threadIdx.x; i < kHistBins / 2; i += NT) S.h[i] = 0u;
    for (int i = threadIdx.x; i < kHistBins / 32; i += NT) S.sup[i] = 0;
    if (threadIdx.x == 0) S.bn = 0;
}

// a3 for one unit: CFR-9 keys (bits of the pooled softmax weight) of this thread's leaves.
// sv[g][l]: the score (CFR-3 base-2 logit) of head g at leaf jb + l (jb = (rank * NT + tid) * LPT),
// -inf for non-candidates (not in [n_sink, n_off)).  Every CTA of the cluster calls it (cluster
// already started).  Non-candidates get key 0.
template <int LPT, int GM, int NC, int NT>
__device__ __forceinline__ void softmax_keys(const FkvDims& D, int rank, int n_off, float (&sv)[GM][LPT],
                                             SelSmem<NT / 32, GM, NC>& S, uint32_t (&key)[LPT],
                                             unsigned long long* tr = nullptr, int ent = 0) {
    constexpr int W = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto stamp = [&](int i) {  // diagnostics: phase stamps (trace class 9)
        if (tr && tid == 0) trace_stamp(tr, 9, ent, i);
    };
    stamp(0);
    const int G = D.G, K = D.K;
    const int jb = (rank * NT + tid) * LPT;
    bool cand[LPT];
#pragma unroll
    for (int l = 0; l < LPT; ++l) cand[l] = jb + l >= D.n_sink && jb + l < n_off;
    // group-consistency variants (f3, reading R-12): QK pools the heads' scores into head
    // 0; Q pooled the queries before scoring (every head holds the same scores); both then run one
    // softmax
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
    // ---- CFR-4: max per head (exact, order-free): redux per warp, over the warps, over the CTAs
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
        for (int g = 0; g < GM; ++g) S.redm[warp][g] = M[g];
    __syncthreads();
#pragma unroll
    for (int g = 0; g < GM; ++g) M[g] = warp_max_f32(lane < W ? S.redm[lane][g] : -INFINITY);
    if constexpr (NC > 1) {
        if (warp == 0)
            for (int i = lane; i < NC * GM; i += 32) {
                float v = M[0];
#pragma unroll
                for (int g = 1; g < GM; ++g) v = (i % GM == g) ? M[g] : v;
                *rmt<NC>(&S.cm[rank][i % GM], i / GM) = v;
            }
        csync<NC>();
#pragma unroll
        for (int g = 0; g < GM; ++g) {
            float v = S.cm[0][g];
#pragma unroll
            for (int r = 1; r < NC; ++r) v = fmaxf(v, S.cm[r][g]);
            M[g] = v;
        }
    }
    stamp(1);
    // ---- CFR-5/6: e = cexp2(s - m); Z = pairwise tree in page-id order: thread-local tree over its
    // LPT contiguous leaves, xor butterfly over the 32 lanes, over the W warp partials (lanes >= W
    // hold +0 leaves), then over the NC CTA subtrees
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
        for (int g = 0; g < GM; ++g) S.redz[warp][g] = Z[g];
    __syncthreads();
#pragma unroll
    for (int g = 0; g < GM; ++g) Z[g] = lane < W ? S.redz[lane][g] : 0.0f;
#pragma unroll
    for (int o = 1; o < W; o <<= 1)
#pragma unroll
        for (int g = 0; g < GM; ++g) Z[g] = __fadd_rn(Z[g], __shfl_xor_sync(0xffffffffu, Z[g], o));
#pragma unroll
    for (int g = 0; g < GM; ++g) Z[g] = __shfl_sync(0xffffffffu, Z[g], 0);
    if constexpr (NC > 1) {
        if (warp == 0)
            for (int i = lane; i < NC * GM; i += 32) {
                float v = Z[0];
#pragma unroll
                for (int g = 1; g < GM; ++g) v = (i % GM == g) ? Z[g] : v;
                *rmt<NC>(&S.cz[rank][i % GM], i / GM) = v;
            }
        csync<NC>();
#pragma unroll
        for (int g = 0; g < GM; ++g) {
            float t[NC];
#pragma unroll
            for (int r = 0; r < NC; ++r) t[r] = S.cz[r][g];
#pragma unroll
            for (int w = 1; w < NC; w <<= 1)
#pragma unroll
                for (int r = 0; r < NC; r += 2 * w) t[r] = __fadd_rn(t[r], t[r + w]);
            Z[g] = t[0];
        }
    }
    stamp(2);
    // ---- CFR-7/8: p = e / Z; pooled over the group (MeanS: sequential sum; MaxS: max); CFR-9 keys
#pragma unroll
    for (int l = 0; l < LPT; ++l) {
        float pi = 0.0f;
        if (cand[l]) {
#pragma unroll
            for (int g = 0; g < GM; ++g) {
                if (g < Gs) {
                    const float pg = __fdiv_rn(sv[g][l], Z[g]);
                    pi = g == 0 ? pg : (D.pool == 1 ? (pg > pi ? pg : pi) : __fadd_rn(pi, pg));
                }
            }
        }
        const uint32_t kk = __float_as_uint(pi);
        key[l] = kk == 0x80000000u ? 0u : kk;
    }
}

// a4 for one unit: the K largest keys (ties -> lower page id, CFR-9) of the leaves
// [n_sink, n_off), this thread's leaves jb .. jb + LPT - 1 (jb = (rank * NT + tid) * LPT).  Every
// CTA of the cluster calls it (histogram cleared and a barrier passed).  On return the leader's
// S.sel holds the K selected page ids in ascending order (the cluster has synchronised).
template <int LPT, int NC, int NT, class SS>
__device__ __forceinline__ void topk_keys(const FkvDims& D, int rank, int n_off, const uint32_t (&key)[LPT], SS& S,
                                          unsigned long long* tr = nullptr, int ent = 0) {
    constexpr int W = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = D.K;
    const int jb = (rank * NT + tid) * LPT;
    auto stamp = [&](int i) {  // diagnostics: phase stamps (trace class 9)
        if (tr && tid == 0) trace_stamp(tr, 9, ent, i);
    };
    bool cand[LPT];
#pragma unroll
    for (int l = 0; l < LPT; ++l) cand[l] = jb + l >= D.n_sink && jb + l < n_off;
    // ---- exact K-th largest key: radix passes of 12, 12 and 7 bits over the cluster-summed
    // histogram; as soon as the boundary bin holds <= 32 keys, they are ranked directly
    uint32_t prefix = 0u, mask = 0u, T = 0u;
    int k_rem = K;
    bool resolved = false;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
        // keys are bits of non-negative floats (bit 31 always 0): the digits cover bits 30..19,
        // 18..7 and 6..0, so the first one is exponent + 4 mantissa bits (1/16-octave bins) and
        // the boundary bin usually holds <= 32 keys after it
        const int shift = pass == 0 ? 19 : (pass == 1 ? 7 : 0);
        const int nbits = pass == 2 ? 7 : 12;
        const uint32_t dmask = (1u << nbits) - 1u;
        if (pass > 0) {  // fallback passes (rare): every CTA is done reading the histograms
            csync<NC>();
            for (int i = tid; i < kHistBins / 2; i += NT) S.h[i] = 0u;
            for (int i = tid; i < kHistBins / 32; i += NT) S.sup[i] = 0;
            __syncthreads();
        }
#pragma unroll
        for (int l = 0; l < LPT; ++l) {
            if (cand[l] && (key[l] & mask) == prefix) {
                const int dg = (int)((key[l] >> shift) & dmask);
                atomicAdd(&S.h[dg >> 1], 1u << ((dg & 1) * 16));
                atomicAdd(&S.sup[dg >> 5], 1);
            }
        }
        stamp(3);
        csync<NC>();
        stamp(4);
        if (warp == 0) {
            // level 1: 32-bin groups (lane owns 4 contiguous groups, one 16-byte load per CTA);
            // level 2: the 32 bins of the boundary group, one per lane
            const int nsup = (int)(dmask + 1u) >> 5;  // 128 or 8
            int4 c4 = make_int4(0, 0, 0, 0);
#pragma unroll
            for (int r = 0; r < NC; ++r) {
                const int* sup = rmt<NC>(S.sup, r);
                if (nsup == 128) {
                    const int4 v = *reinterpret_cast<const int4*>(&sup[lane * 4]);
                    c4.x += v.x;
                    c4.y += v.y;
                    c4.z += v.z;
                    c4.w += v.w;
                } else if (lane < nsup) {
                    c4.x += sup[lane];
                }
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
            int cb = 0;
#pragma unroll
            for (int r = 0; r < NC; ++r) cb += hist_get(rmt<NC>(S.h, r), grp * 32 + lane);
            int suf2 = cb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_down_sync(0xffffffffu, suf2, o);
                if (lane + o < 32) suf2 += y;
            }
            const int ab = above_g + suf2 - cb;  // keys in higher bins
            if (ab < k_rem && ab + cb >= k_rem) {
                S.dig[0] = grp * 32 + lane;
                S.dig[1] = ab;
                S.dig[2] = cb;
            }
        }
        __syncthreads();
        k_rem -= S.dig[1];
        prefix |= (uint32_t)S.dig[0] << shift;
        mask |= dmask << shift;
        if (pass == 2) {  // every bit fixed: T = prefix, take k_rem of the keys equal to it
            T = prefix;
            resolved = true;
            break;
        }
        if (S.dig[2] <= 32) break;
    }
    stamp(5);
    if (!resolved) {
        // the boundary bin's (key, id) pairs (<= 32 over the cluster) -> every CTA's warp 0 ranks
        // them (ties -> lower id): the (k_rem)-th largest is the threshold T
#pragma unroll
        for (int l = 0; l < LPT; ++l) {
            if (cand[l] && (key[l] & mask) == prefix) {
                const int at = atomicAdd(&S.bn, 1);
                S.bk[at] = key[l];
                S.bid[at] = jb + l;
            }
        }
        csync<NC>();
        if (warp == 0) {
            // lane i takes entry i of the concatenation of the CTAs' lists (rank order)
            const int cnt_r = lane < NC ? *rmt<NC>(&S.bn, lane) : 0;
            int incl = cnt_r;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int n = __shfl_sync(0xffffffffu, incl, 31);
            int r = 0, before = 0;  // the CTA whose list holds entry `lane`
#pragma unroll
            for (int rr = 0; rr < NC; ++rr) {
                const int inc = __shfl_sync(0xffffffffu, incl, rr);
                if (lane >= inc) {
                    r = rr + 1;
                    before = inc;
                }
            }
            uint32_t mk = 0u;
            int mi = 0x7fffffff;
            if (lane < n) {
                mk = rmt<NC>(S.bk, r)[lane - before];
                mi = rmt<NC>(S.bid, r)[lane - before];
            }
            int rnk = 0, gt = 0;
            for (int i = 0; i < n; ++i) {
                const uint32_t ok = __shfl_sync(0xffffffffu, mk, i);
                const int oi = __shfl_sync(0xffffffffu, mi, i);
                rnk += (ok > mk || (ok == mk && oi < mi)) ? 1 : 0;
                gt += ok > mk ? 1 : 0;
            }
            if (lane < n && rnk == k_rem - 1) {
                S.dig[2] = (int)mk;
                S.dig[3] = k_rem - gt;
            }
        }
        __syncthreads();
        T = (uint32_t)S.dig[2];
        k_rem = S.dig[3];
    }
    stamp(6);
    // ---- ascending output: one packed (#gt, #eq) scan in page-id order over the cluster
    unsigned n_gt = 0, n_eq = 0;
#pragma unroll
    for (int l = 0; l < LPT; ++l) {
        n_gt += cand[l] && key[l] > T;
        n_eq += cand[l] && key[l] == T;
    }
    const unsigned own = (n_gt << 16) | n_eq;
    unsigned x = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) S.wsum[warp] = x;
    __syncthreads();
    unsigned woff = lane < warp ? S.wsum[lane] : 0u;
    unsigned ctot = lane < W ? S.wsum[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        woff += __shfl_xor_sync(0xffffffffu, woff, o);
        ctot += __shfl_xor_sync(0xffffffffu, ctot, o);
    }
    unsigned coff = 0u;
    if constexpr (NC > 1) {
        if (warp == 0 && lane < NC) *rmt<NC>(&S.ctot[rank], lane) = ctot;
        csync<NC>();
        for (int r = 0; r < rank; ++r) coff += S.ctot[r];
    }
    const unsigned ex = coff + woff + x - own;
    int gt_before = (int)(ex >> 16), eq_before = (int)(ex & 0xffffu);
    int* sel_l = rmt<NC>(S.sel, 0);
#pragma unroll
    for (int l = 0; l < LPT; ++l) {
        if (!cand[l]) continue;
        const bool gt = key[l] > T, eq = key[l] == T;
        if (gt || (eq && eq_before < k_rem)) sel_l[gt_before + min(eq_before, k_rem)] = jb + l;
        gt_before += gt;
        eq_before += eq;
    }
    if (rank == 0)
        for (int i = tid + K; i < kMaxK; i += NT) S.sel[i] = -1;
    csync<NC>();  // the leader holds S_i
    stamp(7);
}

// a3 + a4 for one unit with n_cand > K candidates (softmax_keys, then topk_keys over the cluster).
// On return the leader's S.sel holds the K selected page ids in ascending order.
template <int LPT, int GM, int NC, int NT>
__device__ __forceinline__ void rank_unit(const FkvDims& D, int rank, int n_off, float (&sv)[GM][LPT],
                                          SelSmem<NT / 32, GM, NC>& S, unsigned long long* tr = nullptr,
                                          int ent = 0) {
    uint32_t key[LPT];
    softmax_keys<LPT, GM, NC, NT>(D, rank, n_off, sv, S, key, tr, ent);
    topk_keys<LPT, NC, NT>(D, rank, n_off, key, S, tr, ent);
}

// a4, leader CTA (every thread): delta of S_i (sel[0, cnt), ascending) vs R (U, staged by
// stage_resident; n_res valid ascending entries), slot assignment (the r-th fetched page takes the
// r-th free slot), fetch list, pending selection (pend_*, pend_valid), pages_out, and -- when
// list_all or the unit is corrected -- this step's attention page list (row a7): arena row of each
// page's K block and its valid tokens (sink pages, the pages in use: S_i if corrected, R otherwise,
// P:223/P:255, local pages [f p, Lc), reading A-9; in direct mode a fetched page of a corrected unit
// is a host-pool row to be written back to its slot).  Ends with a CTA barrier.
template <int NT>
__device__ __forceinline__ void finish_unit(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, int u, int Lc,
                                            int n_off, const int* sel, int cnt, UnitSmem& U, int n_res, int res_front,
                                            int flag, int list_all, int32_t* __restrict__ pages_out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, K = D.K;
    const int b = u / D.n_kv, m = u % D.n_kv;
    if (warp == 0) {
        int nf = 0;
        for (int base = 0; base < K; base += 32) {
            const int a = base + lane;
            int fe = 0, slot = -1;
            const int Sa = (a < K && a < cnt) ? sel[a] : -1;
            if (Sa >= 0) {  // membership in R: binary search over R's ascending page list
                fe = 1;
                int lo = 0, hi = n_res;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (U.res[mid] < Sa) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < n_res && U.res[lo] == Sa) {
                    fe = 0;
                    slot = U.res_slot[lo];
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, fe);
            if (fe) {  // the r-th fetched page takes the r-th free slot (ascending)
                const int r = nf + __popc(bal & ((1u << lane) - 1u));
                slot = U.free_[r];
                L.fetch_page[(size_t)u * K + r] = Sa;
                L.fetch_slot[(size_t)u * K + r] = slot;
            }
            nf += __popc(bal);
            if (a < K) {
                U.isfetch[a] = fe;
                U.pslot[a] = slot;
                L.pend_pages[(size_t)u * K + a] = Sa;
                L.pend_slot[(size_t)u * K + a] = slot;
                if (pages_out) pages_out[(size_t)u * K + a] = Sa;
            }
        }
        if (lane == 0) {
            L.n_fetch[u] = nf;
            L.pend_front[u] = n_off;
            L.pend_cnt[u] = cnt;
            L.pend_valid[u] = 1;
        }
    }
    __syncthreads();
    if (list_all || flag) {
        const int p = D.p;
        const int sink_tok = min(D.S_tok, Lc);
        const int n_sp = (sink_tok + p - 1) / p;
        const int n_sel = flag ? cnt : n_res;
        const int f = flag ? n_off : res_front;
        const int n_last = (Lc - 1) / p;
        const int n_loc = (Lc > f * p) ? (n_last - f + 1) : 0;
        const size_t pe = page_elems(D);
        const int total = n_sp + n_sel + n_loc;
        for (int i = tid; i < total; i += NT) {
            const uint16_t* base;
            int valid;
            if (i < n_sp) {
                base = L.sink + ((size_t)u * D.n_sink + i) * pe;
                valid = min(p, sink_tok - i * p);
            } else if (i < n_sp + n_sel) {
                const int a = i - n_sp;
                const int slot = flag ? U.pslot[a] : U.res_slot[a];
                base = L.slots + ((size_t)u * 2 * K + slot) * pe;
                valid = p;
                if (flag && D.direct && U.isfetch[a]) {
                    const int j = sel[a];
                    X.page_rows[(size_t)u * D.P_max + i] =
                        L.host_row0 + (int)((((size_t)b * D.n_page_host + j) * D.n_kv + m) * 2 * p);
                    X.page_valid[(size_t)u * D.P_max + i] = (uint8_t)(p | 0x80);
                    X.page_dst[(size_t)u * D.P_max + i] = (int)((base - L.arena) / kHeadDim);
                    continue;
                }
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
    __syncthreads();
}

}  // namespace fkv
