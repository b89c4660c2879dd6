// attn.cu -- rows a7/a8: sparse decode attention over the gathered pages and
// the speculative advance.
//
// PAPER.md P:95-97 (§2.1): o_h = softmax(q_h K^T / sqrt(d)) V over the token
// set T = sink tokens U selected pages U local region (reading A-9),
// with the pages of S_i for corrected units and the resident set otherwise
// (P:223).  After attention the step commits R := S_i, q_prev := q_i
// (fig:algo1).
//
// Balanced split-KV flash decode.  The U units' page lists are laid end to end
// in a virtual list of U * P_max pages; a grid of exactly T resident warps
// (one wave) gives warp w the contiguous range [w*V/T, (w+1)*V/T), so every
// warp streams the same number of pages (~3.6 at c2) and a range spans at most
// two units.  Each warp keeps an online softmax per unit segment and writes one
// partial record per segment; the combine kernel merges a unit's records.
//
// The G <= 8 heads of a GQA group ride as one MMA tile, so every KV byte is
// loaded once, straight from HBM into registers in MMA fragment order:
//   S   = Q K^T   : mma.m16n8k16  A = Q (16 rows, heads 0..7 real), B = K^T
//   O^T = V^T P^T : mma.m16n8k16  A = V^T (d rows), B = P^T (heads as N = 8)
// The contraction order over d and over tokens is free, so channels and
// tokens are permuted such that every lane issues contiguous 16-byte loads;
// V^T fragments are built with byte permutes.  The next 16-token slab is
// loaded while the current one is computed (register double buffering), so
// each warp always has 8 KiB in flight.  P is split into bf16 hi + lo parts
// (two PV MMAs) so its rounding stays ~2^-17, far inside the 2e-3 output
// tolerance (readings A-19/A-21).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "attn_core.cuh"
#include "append_unit.cuh"

namespace cg = cooperative_groups;

namespace fkv {

__device__ __forceinline__ long long range_start(long long w, long long V, long long T) { return w * V / T; }

// Units attended in `phase`: all (0), unflagged (1), corrected (2).  Phases 1/2 lay only
// their own units end to end, so each phase's warps share exactly that phase's pages.
__device__ __forceinline__ bool in_phase(const FkvLayer& L, int u, int phase) {
    return phase == 0 || ((L.flags[u] != 0) == (phase == 2));
}

// Warp-cooperative: number of phase units, and the units of ranks r0 and r0 + 1.
__device__ __forceinline__ int phase_units(const FkvDims& D, const FkvLayer& L, int phase, int r0, int lane,
                                           int& u0, int& u1) {
    u0 = u1 = -1;
    if (phase == 0) {
        u0 = r0;
        u1 = r0 + 1;
        return D.U;
    }
    int cnt = 0;
    for (int base = 0; base < D.U; base += 32) {
        const int u = base + lane;
        const bool f = u < D.U && in_phase(L, u, phase);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        const int before = __popc(bal & ((1u << lane) - 1u));
        if (f && cnt + before == r0) u0 = u;
        if (f && cnt + before == r0 + 1) u1 = u;
        cnt += __popc(bal);
    }
    // broadcast the (single) owners
    const unsigned h0 = __ballot_sync(0xffffffffu, u0 >= 0), h1 = __ballot_sync(0xffffffffu, u1 >= 0);
    u0 = h0 ? __shfl_sync(0xffffffffu, u0, __ffs(h0) - 1) : -1;
    u1 = h1 ? __shfl_sync(0xffffffffu, u1, __ffs(h1) - 1) : -1;
    return cnt;
}

// phase: 0 = every unit; 1 = unflagged units only (their pages are resident, so this
// half runs while the synchronous recall of the corrected units is in flight);
// 2 = corrected units only (after that recall).  Each unit is attended in exactly
// one phase, so every partial record is written once per step.
template <int NST, int WPC>
__global__ void __launch_bounds__(WPC * 32, WPC == 8 ? 1 : (NST == 2 ? 3 : 2)) fkv_attn_split_kernel(FkvDims D, FkvLayer L, FkvScratch X,
                                                                               const uint16_t* __restrict__ q,
                                                                               int phase,
                                                                               const __grid_constant__ CUtensorMap tmap,
                                                                               const __grid_constant__ CUtensorMap tmap_h,
                                                                               const uint16_t* arena) {
    constexpr int kStages = NST;
    extern __shared__ __align__(1024) uint8_t s_stage[];  // [warps][kStages][8 KiB]
    __shared__ __align__(8) uint64_t bar[WPC][kStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int w = blockIdx.x * WPC + warp;
    const int T = phase == 1 ? D.attn_warps_p1 : D.attn_warps;  // this launch's warps
    pdl_trigger();  // the next kernel (attention phase 2 / combine) may start its prologue
    if (w >= T) return;
    const int tcls = 4 + phase;  // trace class 4/5/6 = attention phase 0/1/2
    if (lane == 0) trace_stamp(X.trace, tcls, w, 0);
    uint8_t* ring = s_stage + warp * (kStages * kSlabBytes);
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kStages; ++i) mbar_init(&bar[warp][i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase_bits = 0u;  // parity of each stage's next completion
    pdl_wait();  // the select kernel's page lists and flags are complete
    const int G = D.G;
    // this phase's virtual page list: its units end to end, P_max pages each
    int nu = D.U;
    if (phase != 0) {
        int d0, d1;
        nu = phase_units(D, L, phase, 0, lane, d0, d1);
    }
    const long long V = (long long)nu * D.P_max;
    const int Tp = (int)min((long long)T, V);  // warps of this phase: every one owns >= 1 page
    if (w >= Tp) return;
    const long long s0 = range_start(w, V, Tp), s1 = range_start(w + 1, V, Tp);
    int ua = -1, ub = -1;  // units of ranks s0 / P_max and s0 / P_max + 1
    if (s0 < s1) phase_units(D, L, phase, (int)(s0 / D.P_max), lane, ua, ub);
    const int rec_base = phase == 2 ? D.attn_warps_p1 : 0;  // records of phase 2 live after phase 1's
    int k_rec = 0;
    for (long long seg = s0; seg < s1; ++k_rec) {
        const int r = (int)(seg / D.P_max);
        const int u = k_rec == 0 ? ua : ub;
        const long long seg_end = min(s1, (long long)(r + 1) * D.P_max);
        const int pa = (int)(seg - (long long)r * D.P_max);
        seg = seg_end;
        const int pb_cap = (int)(seg_end - (long long)r * D.P_max);
        float oacc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) oacc[i][k] = 0.0f;
        float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.0f, 0.0f};  // heads 2t, 2t+1
        uint4 qa[2][2];
        load_q_frags(D, q, u, qa);
        const TableSrc tsrc{X.page_rows + (size_t)u * D.P_max, X.page_valid + (size_t)u * D.P_max,
                            X.page_dst + (size_t)u * D.P_max};
        attend_pages<NST>(D, X, qa, &tmap, &tmap_h, tsrc, pa, min(pb_cap, X.page_cnt[u]), ring, bar[warp], phase_bits,
                          m_run, l_run, oacc, tcls, w);
        if (lane == 0) trace_stamp(X.trace, tcls, w, 3);
        // ---- partial record (w, k_rec) of unit u: unnormalised, relative to m_run.  Lane (g, t)
        // holds heads 2t, 2t+1; l is summed over the 8 lanes g of the same t
        float l0 = l_run[0], l1 = l_run[1];
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        const size_t rec = (size_t)(rec_base + w) * 2 + k_rec;
        if (g == 0) {
            if (2 * t < G) {
                X.part_ml[(rec * G + 2 * t) * 2 + 0] = m_run[0];
                X.part_ml[(rec * G + 2 * t) * 2 + 1] = l0;
            }
            if (2 * t + 1 < G) {
                X.part_ml[(rec * G + 2 * t + 1) * 2 + 0] = m_run[1];
                X.part_ml[(rec * G + 2 * t + 1) * 2 + 1] = l1;
            }
        }
        // logical channel (mt, g) lives at physical 64(g/4) + 8(g%4) + 32(mt/4) + 2(mt%4); (mt, g+8) at +1
        const int base0 = 64 * (g >> 2) + 8 * (g & 3);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int h = 2 * t + hh;
            if (h < G) {
                float* dst = X.part_o + (rec * G + h) * kHeadDim + base0;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    float4* d4 = reinterpret_cast<float4*>(dst + 32 * half);
                    const int mb = 4 * half;
                    d4[0] = make_float4(oacc[mb][hh], oacc[mb][2 + hh], oacc[mb + 1][hh], oacc[mb + 1][2 + hh]);
                    d4[1] = make_float4(oacc[mb + 2][hh], oacc[mb + 2][2 + hh], oacc[mb + 3][hh], oacc[mb + 3][2 + hh]);
                }
            }
        }
    }
    if (lane == 0) trace_stamp(X.trace, tcls, w, 4);
}

static int attn_stages();

// ---- clustered attention: one cluster of C CTAs (4 warps each) per unit; warp k of the 4C
// warps attends its even share of the unit's page list in 16-token slabs, leaves its partial
// record (unnormalised o, running max m, sum l per head) in its own shared memory, and after one
// cluster barrier the leader CTA merges the 4C records over DSMEM, writes the output and commits
// the speculative advance (row a8) -- no global records, no second kernel.
//
// mode 0 (primitive API, serial step): the select kernel wrote every unit's page list; wait for it
//   (PDL); commit R := S_i for every unit.
// mode 1 (speculative decode step): launched right after the pre kernel (append,
//   correction flags, deferred commit) while this step's scoring and selection run on a side stream.
//   A unit that is not corrected attends its resident set R = S_{i-1} at once (list built here,
//   ResSrc); its S_i is committed by the next step's pre kernel.  A corrected unit waits for
//   X.ready[u] (its S_i page list from the side chain's select) and commits S_i itself.
// mode 2 (serial decode step): see below; the select of this step runs before it.
// mode 3 (first_layer_dense): every page [0, Lc) of the unit from the dense pool; no commit.
template <int NST, int C>
__global__ void __launch_bounds__(kAttnWarpsPerCta * 32, 3)
    fkv_attn_cluster_kernel(FkvDims D, FkvLayer L, FkvScratch X, const uint16_t* __restrict__ q,
                            float* __restrict__ out, const __grid_constant__ CUtensorMap tmap,
                            const __grid_constant__ CUtensorMap tmap_h, int mode, int pending) {
    constexpr int kStages = NST, W = kAttnWarpsPerCta, NW = W * C;
    extern __shared__ __align__(1024) uint8_t s_stage[];  // [W][kStages][8 KiB]; then the records
    __shared__ __align__(8) uint64_t bar[W][kStages];
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const int u = blockIdx.x / C;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int g = lane >> 2, t = lane & 3;
    const int G = D.G;
    pdl_trigger();
    const int w = u * NW + crank * W + warp;  // trace entity
    if (lane == 0) {
        trace_stamp(X.trace, 4, w, 0);
        if (X.trace && w < kTraceEnt) {  // diagnostics: the SM of this warp
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            X.trace[((size_t)4 * kTraceEnt + w) * kTraceStamps + 7] = smid;
        }
    }
    uint8_t* ring = s_stage + warp * (kStages * kSlabBytes);
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kStages; ++i) mbar_init(&bar[warp][i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase_bits = 0u;
    const int k = crank * W + warp;
    // this warp's share of the unit's page list, in 16-token slabs (an even split of P_max * spp
    // slabs; whole entries [pa, pbc) minus `skip` slabs at the front and `trim` at the back)
    // mode 3 (dense layer): launched without PDL after the append, so the context is final here
    const int spp = D.p >> 4, TS = (mode == 3 ? (L.ctx[u] + D.p - 1) / D.p : D.P_max) * spp;
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
    // mode 2 (serial decode step): the pre kernel has completed when this grid launches (the select
    // before it triggers after its own wait, the score before that after its own), so the flags,
    // the context length and R are final.  A unit that is not corrected attends the same list the
    // select would write for it -- sink pages, R, local pages -- built from R here, and its first
    // slabs are in flight before the wait for the select
    int flag = 0, Lc = 0, pre = 0;
    if (mode == 2) {
        Lc = L.ctx[u] + pending;
        flag = __ldcg(L.flags + u);
        if (!flag) {
            const ResSrc rsrc = res_src(D, L, u, Lc);
            const int n_pages = rsrc.count();
#pragma unroll
            for (int i = 0; i < kStages; ++i) {
                const int x = sa + i;
                if (x >= sb) break;
                const int pi = x / spp, sl = x - pi * spp;
                if (pi >= n_pages) break;
                int row, valid, dst;
                rsrc.load(pi, row, valid, dst);
                if (valid - sl * 16 <= 0) break;
                if (lane == 0) issue_slab(&tmap, ring + i * kSlabBytes, &bar[warp][i], row + sl * 16, D.p, X.arena);
                pre = i + 1;
            }
        }
    }
    // a unit that is not corrected needs nothing from the select until its commit (R := S_i): with
    // D.attn_early it attends its whole resident set while the select still runs and waits only
    // before the commit (the selection leaves the attention's critical path)
    const bool early = mode == 2 && !flag && D.attn_early;
    if (!early) pdl_wait();  // mode 0/2: the select kernel's page lists are complete; mode 1: the pre kernel is done
    if (mode != 2) {
        flag = mode == 3 ? 0 : L.flags[u];
        Lc = L.ctx[u];
    }
    load_q_frags(D, q, u, qa);
    if (mode == 1 && flag) {  // corrected unit: its S_i page list comes from the select kernel
        if (lane == 0)
            spin_until_ge(X.ready + u, 1);
        __syncwarp();
    }
    if (mode == 3) {  // first_layer_dense: T = [0, Lc) (O-7), every page from the dense pool
        const DenseSrc dsrc{(int)((L.dense - L.arena) / kHeadDim) + u * D.n_page_max * 2 * D.p, D.p, Lc, 2 * D.p};
        const int pe = min(pbc, dsrc.count());
        attend_pages<NST>(D, X, qa, &tmap, &tmap_h, dsrc, pa, pe, ring, bar[warp], phase_bits, m_run, l_run, oacc, 4,
                          w, 0, skip, pe == pbc ? trim : 0);
    } else if (mode == 0 || flag) {
        const TableSrc tsrc{X.page_rows + (size_t)u * D.P_max, X.page_valid + (size_t)u * D.P_max,
                            X.page_dst + (size_t)u * D.P_max};
        const int pe = min(pbc, __ldcg(X.page_cnt + u));
        attend_pages<NST>(D, X, qa, &tmap, &tmap_h, tsrc, pa, pe, ring, bar[warp], phase_bits, m_run, l_run, oacc, 4,
                          w, 0, skip, pe == pbc ? trim : 0);
    } else {
        const ResSrc rsrc = res_src(D, L, u, Lc);
        const int pe = min(pbc, rsrc.count());
        attend_pages<NST>(D, X, qa, &tmap, &tmap_h, rsrc, pa, pe, ring, bar[warp], phase_bits, m_run, l_run, oacc, 4,
                          w, pre, skip, pe == pbc ? trim : 0);
    }
    if (lane == 0) trace_stamp(X.trace, 4, w, 3);
    // ---- this warp's record, in its own (now idle) ring: o [G][128], then m [G], l [G]
    __syncwarp();
    write_record(reinterpret_cast<float*>(ring), G, oacc, m_run, l_run);
    // the leader's q_prev inputs, loaded before the barrier (independent of the records)
    constexpr int kQv = (kMaxG * (kHeadDim / 4) + kAttnWarpsPerCta * 32 - 1) / (kAttnWarpsPerCta * 32);
    uint2 qv[kQv];
    const int b = u / D.n_kv, m = u % D.n_kv;
    // ... and the leader's commit inputs (the select's pending selection): an early unit waits
    // for the select here, so these loads overlap the merges below instead of following them
    const bool commit = mode != 3 && (mode != 1 || flag);
    constexpr int kPend = (256 + kAttnWarpsPerCta * 32 - 1) / (kAttnWarpsPerCta * 32);  // K <= 256
    int pend_pg[kPend], pend_sl[kPend], pend_fr = 0, pend_ct = 0;
    if (crank == 0) {
#pragma unroll
        for (int i = 0; i < kQv; ++i) {
            const int e = tid + i * (int)blockDim.x;
            if (e < G * (kHeadDim / 4)) {
                const size_t row = (size_t)b * D.n_qo + m * G + e / (kHeadDim / 4);
                qv[i] = reinterpret_cast<const uint2*>(q + row * kHeadDim)[e % (kHeadDim / 4)];
            }
        }
        if (early) pdl_wait();  // q_prev is read by this step's score grid; R by the select
        if (commit) {
#pragma unroll
            for (int i = 0; i < kPend; ++i) {
                const int a = tid + i * (int)blockDim.x;
                if (a < D.K) {
                    pend_pg[i] = __ldcg(L.pend_pages + (size_t)u * D.K + a);
                    pend_sl[i] = __ldcg(L.pend_slot + (size_t)u * D.K + a);
                }
            }
            if (tid == 0) {
                pend_fr = __ldcg(L.pend_front + u);
                pend_ct = __ldcg(L.pend_cnt + u);
            }
        }
    }
    // CTA-level merge of the W warp records into one CTA record (warp 0's second stage), then the
    // leader merges the C CTA records over DSMEM: C remote records per output instead of W * C
    __syncthreads();
    float* crec = reinterpret_cast<float*>(s_stage + kSlabBytes);
    for (int e = tid; e < G * (kHeadDim / 4); e += blockDim.x) {
        const int h = e / (kHeadDim / 4), c4 = e % (kHeadDim / 4);
        float M = -INFINITY;
#pragma unroll
        for (int r = 0; r < W; ++r)
            M = fmaxf(M, reinterpret_cast<const float*>(s_stage + r * (kStages * kSlabBytes))[G * kHeadDim + h]);
        float Ls = 0.0f;
        float4 O = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int r = 0; r < W; ++r) {
            const float* rr = reinterpret_cast<const float*>(s_stage + r * (kStages * kSlabBytes));
            const float mr = rr[G * kHeadDim + h];
            const float wgt = mr == -INFINITY ? 0.0f : exp2f(mr - M);
            const float4 o = reinterpret_cast<const float4*>(rr + h * kHeadDim)[c4];
            Ls += wgt * rr[G * kHeadDim + G + h];
            O.x += wgt * o.x;
            O.y += wgt * o.y;
            O.z += wgt * o.z;
            O.w += wgt * o.w;
        }
        reinterpret_cast<float4*>(crec + h * kHeadDim)[c4] = O;
        if (c4 == 0) {
            crec[G * kHeadDim + h] = M;
            crec[G * kHeadDim + G + h] = Ls;
        }
    }
    cl.sync();  // every CTA record of the unit is in its CTA's shared memory
    if (crank == 0) {
        if (tid == 0) trace_stamp(X.trace, 7, u, 0);
        // thread -> (head h, 4 channels); CTA records read over DSMEM, merged with an online max
#pragma unroll
        for (int qi = 0; qi < kQv; ++qi) {
            const int e = tid + qi * (int)blockDim.x;
            if (e >= G * (kHeadDim / 4)) break;
            const float4 o4 = merge_records<C>(G, e, [&](int r) {
                return cl.map_shared_rank(reinterpret_cast<const float*>(s_stage + kSlabBytes), r);
            });
            const size_t row = (size_t)b * D.n_qo + m * G + e / (kHeadDim / 4);
            reinterpret_cast<float4*>(out + row * kHeadDim)[e % (kHeadDim / 4)] = o4;
        }
        // q_prev := q_i -- after the select (and so the score grid, whose correction check reads
        // q_prev) is complete when this unit attended early (waited above)
#pragma unroll
        for (int qi = 0; qi < kQv; ++qi) {
            const int e = tid + qi * (int)blockDim.x;
            if (e >= G * (kHeadDim / 4)) break;
            const size_t row = (size_t)b * D.n_qo + m * G + e / (kHeadDim / 4);
            reinterpret_cast<uint2*>(L.q_prev + row * kHeadDim)[e % (kHeadDim / 4)] = qv[qi];
        }
        // commit R := S_i: every unit in modes 0 and 2; in mode 1 the corrected units (the
        // others' S_i is committed by the next step's pre kernel, after their background recall)
        if (commit) {
#pragma unroll
            for (int i = 0; i < kPend; ++i) {
                const int a = tid + i * (int)blockDim.x;
                if (a < D.K) {
                    L.res_pages[(size_t)u * D.K + a] = pend_pg[i];
                    L.res_slot[(size_t)u * D.K + a] = pend_sl[i];
                }
            }
            if (tid == 0) {
                L.res_front[u] = pend_fr;
                L.res_cnt[u] = pend_ct;
                L.res_valid[u] = 1;
                L.pend_valid[u] = 0;
                X.ready[u] = 0;
                if (pending) {  // the token the score grid appended is now part of the context
                    L.ctx[u] = Lc;
                    L.n_off[u] = max(L.n_off[u], frontier_for(D, Lc));
                }
            }
        }
        if (tid == 0) trace_stamp(X.trace, 7, u, 1);
    }
    cl.sync();  // the leader has read every record: the other CTAs may exit
}

template <int NST, int C>
static cudaError_t launch_cluster_c(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                    float* out, const CUtensorMap& tmap, const CUtensorMap& tmap_h, int mode, bool pdl,
                                    int prio, cudaStream_t s, int pending) {
    auto kern = fkv_attn_cluster_kernel<NST, C>;
    const int smem = kAttnWarpsPerCta * NST * kSlabBytes;
    cudaError_t e = func_smem((const void*)kern, smem);
    if (e != cudaSuccess) return e;
    if (C > 8) {  // 16-CTA clusters are a non-portable size (opt-in)
        e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.U * C);
    cfg.blockDim = dim3(kAttnWarpsPerCta * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[3];
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
    if (prio) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na].val.priority = prio;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, D, L, X, q, out, tmap, tmap_h, mode, pending);
}

// Clustered attention + merge + commit; c = CTAs per unit (1, 2, 4, 8)
cudaError_t launch_attn_cluster(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                float* out, const CUtensorMap& tmap, const CUtensorMap& tmap_h, int mode, int c,
                                bool pdl, int prio, cudaStream_t s, int pending) {
    const int nst = D.attn_nst ? D.attn_nst : attn_stages();
#define FKV_CL(NS)                                                                                         \
    do {                                                                                                   \
        if (c == 1) return launch_cluster_c<NS, 1>(D, L, X, q, out, tmap, tmap_h, mode, pdl, prio, s, pending); \
        if (c == 2) return launch_cluster_c<NS, 2>(D, L, X, q, out, tmap, tmap_h, mode, pdl, prio, s, pending); \
        if (c == 4) return launch_cluster_c<NS, 4>(D, L, X, q, out, tmap, tmap_h, mode, pdl, prio, s, pending); \
        if (c == 16) return launch_cluster_c<NS, 16>(D, L, X, q, out, tmap, tmap_h, mode, pdl, prio, s, pending); \
        return launch_cluster_c<NS, 8>(D, L, X, q, out, tmap, tmap_h, mode, pdl, prio, s, pending);             \
    } while (0)
    if (nst == 2) FKV_CL(2);
    FKV_CL(3);
#undef FKV_CL
}

// Merge a unit's partial records and commit the speculative advance (row a8).
// The records of unit u are the contiguous warps w_first..w_last whose page
// ranges intersect [u*P_max, (u+1)*P_max) (every warp owns >= 1 page, T <= V;
// 32-bit range math, T * V < 2^31 is guaranteed on the host).  A record is
// G x 128 floats; thread (rg, e) owns float4 e of it and merges the records
// r = rg (mod RG) with an online max, all of its loads in flight at once (one
// round trip for up to kCombBatch records per group); the RG partial states
// are then merged through shared memory.
constexpr int kCombThreads = 512;
constexpr int kCombBatch = 8;
constexpr int kMaxRecs = 256;  // records per unit (host guarantees P_max * T / V + 2 <= 256)

__global__ void __launch_bounds__(kCombThreads, 2) fkv_attn_combine_kernel(FkvDims D, FkvLayer L, FkvScratch X,
                                                                        const uint16_t* __restrict__ q,
                                                                        float* __restrict__ out, int split,
                                                                        int commit) {
    if (threadIdx.x == 0) trace_stamp(X.trace, 7, blockIdx.x, 0);
    // everything below reads state of this step: with PDL the kernel may start while the
    // select kernel (two launches back) is still running, so nothing is read before this
    pdl_wait();  // the attention's partial records (and the select kernel's lists) are complete
    const int u = blockIdx.x, b = u / D.n_kv, m = u % D.n_kv, G = D.G;
    const int E = G * (kHeadDim / 4);  // float4 per record
    const int RG = kCombThreads / E;   // record groups
    const int e = threadIdx.x % E, rg = threadIdx.x / E, h = e / (kHeadDim / 4);
    // independent loads first (one round trip): this thread's q (for q_prev), commit lists
    const size_t row = (size_t)b * D.n_qo + m * G + h;
    const int c4 = e % (kHeadDim / 4);
    uint2 qv = make_uint2(0u, 0u);
    if (rg == 0) qv = reinterpret_cast<const uint2*>(q + row * kHeadDim)[c4];
    int rp = 0, rs = 0;
    if (threadIdx.x < D.K) {
        rp = L.pend_pages[(size_t)u * D.K + threadIdx.x];
        rs = L.pend_slot[(size_t)u * D.K + threadIdx.x];
    }
    int pf = 0, pc = 0;
    if (threadIdx.x == 0) {
        pf = L.pend_front[u];
        pc = L.pend_cnt[u];
    }
    // rank of u among the units of its attention phase (split: by correction flag); the
    // flags are loaded in one batch (<= 8 per lane), not one dependent load per 32 units
    __shared__ int s_rank, s_n;
    const int my_flag = L.flags[u];
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int my_phase = split ? (my_flag ? 2 : 1) : 0;
        int cnt = 0, rank = 0;
        for (int base0 = 0; base0 < D.U; base0 += 256) {
            uint8_t fv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int v = base0 + 32 * i + lane;
                fv[i] = (split && v < D.U) ? L.flags[v] : 0;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int base = base0 + 32 * i, v = base + lane;
                const bool f = v < D.U && (my_phase == 0 || ((fv[i] != 0) == (my_phase == 2)));
                const unsigned bal = __ballot_sync(0xffffffffu, f);
                if (base <= u && u < base + 32) rank = cnt + __popc(bal & ((1u << (u - base)) - 1u));
                cnt += __popc(bal);
            }
        }
        if (lane == 0) {
            s_rank = rank;
            s_n = cnt;
        }
    }
    __syncthreads();
    const int rec_base = (split && my_flag) ? D.attn_warps_p1 : 0;
    const unsigned V = (unsigned)(s_n * D.P_max);
    const unsigned Tl = (split && !my_flag) ? (unsigned)D.attn_warps_p1 : (unsigned)D.attn_warps;  // the launch's warps
    const unsigned T = min(Tl, V);  // the phase's warp count (see the split kernel)
    const unsigned x0 = (unsigned)s_rank * D.P_max, x1 = x0 + D.P_max;
    const int w_first = (int)(((x0 + 1) * T + V - 1) / V) - 1;
    const int w_last = (int)((x1 * T + V - 1) / V) - 1;
    const int nr = w_last - w_first + 1;
    // record indices, computed once (integer division is ~30 instructions)
    __shared__ int s_rec[kMaxRecs];
    for (int r = threadIdx.x; r < nr && r < kMaxRecs; r += blockDim.x) {
        const unsigned w = (unsigned)(w_first + r);
        const unsigned a = w * V / T;
        s_rec[r] = (int)((rec_base + w) * 2 + ((a / D.P_max == (unsigned)s_rank) ? 0 : 1));
    }
    __syncthreads();
    float M = -INFINITY, Ls = 0.0f;
    float4 O = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    const float4* po = reinterpret_cast<const float4*>(X.part_o);
    if (rg < RG) {
        for (int r0 = rg; r0 < nr; r0 += kCombBatch * RG) {
            float vm[kCombBatch], vl[kCombBatch];
            float4 vo[kCombBatch];
#pragma unroll
            for (int i = 0; i < kCombBatch; ++i) {
                const int r = r0 + i * RG;
                vm[i] = -INFINITY;
                vl[i] = 0.0f;
                vo[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                if (r < nr) {
                    const size_t rec = (size_t)s_rec[r];
                    vm[i] = X.part_ml[(rec * G + h) * 2 + 0];
                    vl[i] = X.part_ml[(rec * G + h) * 2 + 1];
                    vo[i] = po[rec * E + e];
                }
            }
            float Mb = M;
#pragma unroll
            for (int i = 0; i < kCombBatch; ++i) Mb = fmaxf(Mb, vm[i]);
            if (Mb != -INFINITY) {
                const float sc = exp2f(M - Mb);  // M = -inf -> 0
                Ls *= sc;
                O.x *= sc;
                O.y *= sc;
                O.z *= sc;
                O.w *= sc;
#pragma unroll
                for (int i = 0; i < kCombBatch; ++i) {
                    const float wgt = vm[i] == -INFINITY ? 0.0f : exp2f(vm[i] - Mb);
                    Ls += wgt * vl[i];
                    O.x += wgt * vo[i].x;
                    O.y += wgt * vo[i].y;
                    O.z += wgt * vo[i].z;
                    O.w += wgt * vo[i].w;
                }
                M = Mb;
            }
        }
    }
    // merge the RG group states: group g > 0 publishes, group 0 folds them in
    __shared__ float4 s_o[kCombThreads];
    __shared__ float s_m[kCombThreads], s_l[kCombThreads];
    if (rg > 0 && rg < RG) {
        s_o[threadIdx.x] = O;
        s_m[threadIdx.x] = M;
        s_l[threadIdx.x] = Ls;
    }
    __syncthreads();
    const bool do_commit = commit == 0 || my_flag != 0;
    if (rg == 0) {
        float Mb = M;
        for (int g2 = 1; g2 < RG; ++g2) Mb = fmaxf(Mb, s_m[g2 * E + e]);
        float wgt = M == -INFINITY ? 0.0f : exp2f(M - Mb);
        float Lt = wgt * Ls;
        float4 Ot = make_float4(wgt * O.x, wgt * O.y, wgt * O.z, wgt * O.w);
        for (int g2 = 1; g2 < RG; ++g2) {
            const float mg = s_m[g2 * E + e];
            const float wg = mg == -INFINITY ? 0.0f : exp2f(mg - Mb);
            const float4 og = s_o[g2 * E + e];
            Lt += wg * s_l[g2 * E + e];
            Ot.x += wg * og.x;
            Ot.y += wg * og.y;
            Ot.z += wg * og.z;
            Ot.w += wg * og.w;
        }
        reinterpret_cast<float4*>(out + row * kHeadDim)[c4] = make_float4(Ot.x / Lt, Ot.y / Lt, Ot.z / Lt, Ot.w / Lt);
        // q_prev := q_i (4 bf16 = 8 bytes per thread)
        if (do_commit) reinterpret_cast<uint2*>(L.q_prev + row * kHeadDim)[c4] = qv;
    }
    if (!do_commit) return;
    if (threadIdx.x < D.K) {
        L.res_pages[(size_t)u * D.K + threadIdx.x] = rp;
        L.res_slot[(size_t)u * D.K + threadIdx.x] = rs;
    }
    for (int i = threadIdx.x + blockDim.x; i < D.K; i += blockDim.x) {  // K > block size
        L.res_pages[(size_t)u * D.K + i] = L.pend_pages[(size_t)u * D.K + i];
        L.res_slot[(size_t)u * D.K + i] = L.pend_slot[(size_t)u * D.K + i];
    }
    if (threadIdx.x == 0) {
        L.res_front[u] = pf;
        L.res_cnt[u] = pc;
        L.res_valid[u] = 1;
        L.pend_valid[u] = 0;
        X.ready[u] = 0;
        trace_stamp(X.trace, 7, blockIdx.x, 1);
    }
}

// Resident warps of the split kernel, minus headroom of ~1/8 of the CTA slots so
// the recall kernels (other streams) can be scheduled while attention runs.
static int attn_stages() {
    static int st = 0;
    if (!st) {
        const char* e = getenv("FREEKV_ATTN_STAGES");
        st = (e && (e[0] == '2' || e[0] == '4')) ? e[0] - '0' : 3;
    }
    return st;
}

template <int NST>
static cudaError_t attn_setup(int cps_want, int* warps) {
    const int smem = kAttnWarpsPerCta * NST * kSlabBytes;
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = func_smem((const void*)fkv_attn_split_kernel<NST, 4>, smem);
    if (e == cudaSuccess) e = func_smem((const void*)fkv_attn_combine_kernel, 0);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fkv_attn_split_kernel<NST, 4>,
                                                          kAttnWarpsPerCta * 32, smem);
    const int cps = std::max(1, std::min(per_sm, cps_want));
    *warps = sms * cps * kAttnWarpsPerCta;
    return e;
}

// Resident warps of the split kernel (stage count from FREEKV_ATTN_STAGES: 2, 3 or 4).
cudaError_t attn_resident_warps(int cps, int* warps) {
    switch (attn_stages()) {
        case 2: return attn_setup<2>(cps, warps);
        case 4: return attn_setup<4>(cps, warps);
        default: return attn_setup<3>(cps, warps);
    }
}

// Split-KV attention over the page lists of the select kernel (paper-order recall mode,
// FREEKV_CORR=recall): phase 1 = units with resident pages, phase 2 = corrected units after
// their synchronous recall; the combine kernel merges the records and commits.
cudaError_t launch_attn_split(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              int phase, const CUtensorMap& tmap, const CUtensorMap& tmap_h, const uint16_t* arena,
                              bool pdl, cudaStream_t s) {
    const int T = phase == 1 ? D.attn_warps_p1 : D.attn_warps;
    const int nst = attn_stages();
#define FKV_ATTN(NS)                                                                                            \
    return launch_ex(fkv_attn_split_kernel<NS, 4>, dim3((T + 3) / 4), dim3(4 * 32), 4 * NS * kSlabBytes, s, pdl, 0, \
                     D, L, X, q, phase, tmap, tmap_h, arena)
    if (nst == 2) FKV_ATTN(2);
    if (nst == 4) FKV_ATTN(4);
    FKV_ATTN(3);
#undef FKV_ATTN
}

cudaError_t launch_attn_combine(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                float* out, int split, int commit, bool pdl, cudaStream_t s) {
    return launch_ex(fkv_attn_combine_kernel, dim3(D.U), dim3(kCombThreads), 0, s, pdl, 0, D, L, X, q, out, split,
                     commit);
}

}  // namespace fkv
