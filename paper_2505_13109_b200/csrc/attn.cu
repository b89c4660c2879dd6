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

#include "fkv_internal.cuh"

namespace cg = cooperative_groups;

namespace fkv {

constexpr int kAttnWarpsPerCta = 4;

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ldg_stream(const uint16_t* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint32_t u4get(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

struct UnitMeta {
    const int32_t* sel_slot;
    int n_sp, n_sel, n_loc, n_pages, f, Lc, sink_tok;
};

__device__ __forceinline__ UnitMeta load_meta(const FkvDims& D, const FkvLayer& L, int u) {
    UnitMeta M;
    const int flag = L.flags[u];
    M.sel_slot = (flag ? L.pend_slot : L.res_slot) + (size_t)u * D.K;
    M.n_sel = flag ? L.pend_cnt[u] : L.res_cnt[u];
    M.f = flag ? L.pend_front[u] : L.res_front[u];
    M.Lc = L.ctx[u];
    M.sink_tok = min(D.S_tok, M.Lc);
    M.n_sp = (M.sink_tok + D.p - 1) / D.p;
    const int n_last = (M.Lc - 1) / D.p;
    M.n_loc = (M.Lc > M.f * D.p) ? (n_last - M.f + 1) : 0;
    M.n_pages = M.n_sp + M.n_sel + M.n_loc;
    return M;
}

// Entry i of unit u's page list: sink pages, selected slots, local ring pages.
__device__ __forceinline__ const uint16_t* page_ptr(const FkvDims& D, const FkvLayer& L, int u, const UnitMeta& M,
                                                    int i, int& valid) {
    const size_t pe = page_elems(D);
    if (i < M.n_sp) {
        valid = min(D.p, M.sink_tok - i * D.p);
        return L.sink + ((size_t)u * D.n_sink + i) * pe;
    }
    i -= M.n_sp;
    if (i < M.n_sel) {
        valid = D.p;
        return L.slots + ((size_t)u * 2 * D.K + M.sel_slot[i]) * pe;
    }
    i -= M.n_sel;
    const int j = M.f + i;
    valid = min(D.p, M.Lc - j * D.p);
    return L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe;
}

// ---- TMA staging.  The whole device arena is one 2D tensor of 256-byte rows
// (128 bf16 channels); a 16-token slab of a page is K rows [row, row+16) and V
// rows [row+p, row+p+16), fetched as four {64 ch x 16 rows} boxes with the
// 128-byte swizzle (16-byte chunk c of row r lives at chunk c ^ (r % 8)).  The
// fragment mapping below is chosen so every quarter-warp LDS.128 hits 8
// distinct chunks (conflict-free) under that swizzle.
// slab stages per warp: template parameter NST (2, 3 or 4), FREEKV_ATTN_STAGES
constexpr int kBoxBytes = 16 * 128; // 16 rows x 64 channels bf16
constexpr int kSlabBytes = 4 * kBoxBytes;

__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(smem)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }

// valid tokens of slab x of unit u (<= 0: empty), and its first K row in the arena tensor
__device__ __forceinline__ int slab_info(const FkvDims& D, const FkvLayer& L, int u, const UnitMeta& M, int x,
                                         const uint16_t* arena, int& row) {
    const int spp = D.p >> 4;
    const int pi = x / spp, slab = x - pi * spp;
    int pv;
    const uint16_t* base = page_ptr(D, L, u, M, pi, pv);
    row = (int)((base - arena) / kHeadDim) + slab * 16;
    return pv - slab * 16;
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* smem) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(x),
                 "r"(y), "r"(smem_u32(smem))
                 : "memory");
}

// direct mode: write a slab that was read from the host pool back into its slot
// (arena rows [row, row+16) and [row+p, row+p+16)); one bulk group per slab
__device__ __forceinline__ void store_slab(const CUtensorMap* map, const uint8_t* st, int row, int p) {
    tma_store_2d(map, 0, row, st + 0 * kBoxBytes);
    tma_store_2d(map, 64, row, st + 1 * kBoxBytes);
    tma_store_2d(map, 0, row + p, st + 2 * kBoxBytes);
    tma_store_2d(map, 64, row + p, st + 3 * kBoxBytes);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void issue_slab(const CUtensorMap* map, uint8_t* st, uint64_t* bar, int row, int p) {
    mbar_expect_tx(bar, kSlabBytes);
    tma_load_2d(st + 0 * kBoxBytes, map, 0, row, bar);
    tma_load_2d(st + 1 * kBoxBytes, map, 64, row, bar);
    tma_load_2d(st + 2 * kBoxBytes, map, 0, row + p, bar);
    tma_load_2d(st + 3 * kBoxBytes, map, 64, row + p, bar);
}

__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}

// One 16-token slab.  S^T = K Q^T on mma.m16n8k16 with M = 16 tokens, N = 8 heads
// (no padded rows), so lane (g, t) holds S for tokens g and g+8 of heads 2t and
// 2t+1: the per-head softmax state (max, rescale factor) is held by exactly the
// lanes that hold O^T's columns for those heads, and P^T's MMA fragment is one
// movmatrix.trans of the packed probabilities.
__device__ __forceinline__ void compute_slab(const uint8_t* st, int valid, const uint4 (&qb)[2][2], float sc, int g,
                                             int t, float (&m_run)[2], float (&l_run)[2], float (&oacc)[8][4]) {
    // ---- S^T: A = K rows g (tokens 0-7) and g+8 (tokens 8-15), 16 channels per k-step;
    // lane t reads chunks 2t, 2t+1 of each 64-channel box (swizzled by row % 8 = g)
    float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const uint8_t* r0 = st + b * kBoxBytes + g * 128;
        const uint8_t* r8 = r0 + 8 * 128;
        const uint4 a0 = lds128(r0 + (((2 * t) ^ g) << 4));
        const uint4 a1 = lds128(r0 + (((2 * t + 1) ^ g) << 4));
        const uint4 c0 = lds128(r8 + (((2 * t) ^ g) << 4));
        const uint4 c1 = lds128(r8 + (((2 * t + 1) ^ g) << 4));
        mma16816(s, a0.x, c0.x, a0.y, c0.y, qb[b][0].x, qb[b][0].y);
        mma16816(s, a0.z, c0.z, a0.w, c0.w, qb[b][0].z, qb[b][0].w);
        mma16816(s, a1.x, c1.x, a1.y, c1.y, qb[b][1].x, qb[b][1].y);
        mma16816(s, a1.z, c1.z, a1.w, c1.w, qb[b][1].z, qb[b][1].w);
    }
    // s[0], s[1]: token g, heads 2t, 2t+1; s[2], s[3]: token g+8
    float x[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int tok = g + (e >> 1) * 8;
        x[e] = tok < valid ? s[e] * sc : -INFINITY;
    }
    float mx0 = fmaxf(x[0], x[2]), mx1 = fmaxf(x[1], x[3]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {  // over the 8 lanes g with the same t
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const float mn0 = fmaxf(m_run[0], mx0), mn1 = fmaxf(m_run[1], mx1);
    const float al0 = (mn0 == -INFINITY) ? 1.0f : exp2f(m_run[0] - mn0);
    const float al1 = (mn1 == -INFINITY) ? 1.0f : exp2f(m_run[1] - mn1);
    float pv[4];
    pv[0] = (mn0 == -INFINITY) ? 0.0f : exp2f(x[0] - mn0);
    pv[1] = (mn1 == -INFINITY) ? 0.0f : exp2f(x[1] - mn1);
    pv[2] = (mn0 == -INFINITY) ? 0.0f : exp2f(x[2] - mn0);
    pv[3] = (mn1 == -INFINITY) ? 0.0f : exp2f(x[3] - mn1);
    l_run[0] = l_run[0] * al0 + pv[0] + pv[2];
    l_run[1] = l_run[1] * al1 + pv[1] + pv[3];
    m_run[0] = mn0;
    m_run[1] = mn1;
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
        oacc[mt][0] *= al0;
        oacc[mt][1] *= al1;
        oacc[mt][2] *= al0;
        oacc[mt][3] *= al1;
    }
    // ---- P^T fragments (hi + lo bf16 split): pack (token g, heads 2t, 2t+1) then transpose the
    // 8x8 (token x head) tiles so lane (g, t) holds P[tokens 2t, 2t+1][head g]
    const uint32_t ph0 = pack_bf16(pv[0], pv[1]);
    const uint32_t ph8 = pack_bf16(pv[2], pv[3]);
    const __nv_bfloat162 h0 = *reinterpret_cast<const __nv_bfloat162*>(&ph0);
    const __nv_bfloat162 h8 = *reinterpret_cast<const __nv_bfloat162*>(&ph8);
    const uint32_t pl0 = pack_bf16(pv[0] - __low2float(h0), pv[1] - __high2float(h0));
    const uint32_t pl8 = pack_bf16(pv[2] - __low2float(h8), pv[3] - __high2float(h8));
    const uint32_t bh0 = movmatrix_trans(ph0), bh1 = movmatrix_trans(ph8);
    const uint32_t bl0 = movmatrix_trans(pl0), bl1 = movmatrix_trans(pl8);
    // ---- V fragments: lane (g, t) reads tokens 2t, 2t+1, 2t+8, 2t+9 and, in box g / 4, the
    // chunks g % 4 (m-tiles 0-3) and g % 4 + 4 (m-tiles 4-7), swizzled by row % 8
    uint4 vr[4][2];
    {
        const uint8_t* vb = st + 2 * kBoxBytes + (g >> 2) * kBoxBytes;
        const int c0 = g & 3;
#pragma unroll
        for (int ri = 0; ri < 4; ++ri) {
            const int r = 2 * t + (ri & 1) + (ri >> 1) * 8;
            vr[ri][0] = lds128(vb + r * 128 + ((c0 ^ (r & 7)) << 4));
            vr[ri][1] = lds128(vb + r * 128 + (((c0 + 4) ^ (r & 7)) << 4));
        }
    }
    // ---- O^T += V^T P^T over 8 m-tiles of 16 channels
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
        const uint32_t x0 = u4get(vr[0][mt >> 2], mt & 3);  // token 2t
        const uint32_t x1 = u4get(vr[1][mt >> 2], mt & 3);  // token 2t+1
        const uint32_t x8 = u4get(vr[2][mt >> 2], mt & 3);  // token 2t+8
        const uint32_t x9 = u4get(vr[3][mt >> 2], mt & 3);  // token 2t+9
        const uint32_t A0 = __byte_perm(x0, x1, 0x5410);
        const uint32_t A1 = __byte_perm(x0, x1, 0x7632);
        const uint32_t A2 = __byte_perm(x8, x9, 0x5410);
        const uint32_t A3 = __byte_perm(x8, x9, 0x7632);
        mma16816(oacc[mt], A0, A1, A2, A3, bh0, bh1);
        mma16816(oacc[mt], A0, A1, A2, A3, bl0, bl1);
    }
}

// Page sources of attend_pages: entry i of unit u's page list -> (first K row in the arena
// or host tensor, valid tokens | 0x80 for a host row, write-back row).
struct TableSrc {  // the list written by the select (or prep) kernel of this step
    const int32_t* rows;
    const uint8_t* valid;
    const int32_t* dst;
    __device__ __forceinline__ void load(int i, int& r, int& v, int& d) const {
        r = rows[i];
        v = valid[i];
        d = dst[i];
    }
};
struct SpecSrc {  // sink pages, then the resident set R of step i-1 (all full pages)
    int sink_row0, slot_row0, page_rows, n_sink;
    const int32_t* res_slot;
    int p;
    __device__ __forceinline__ void load(int i, int& r, int& v, int& d) const {
        r = i < n_sink ? sink_row0 + i * page_rows : slot_row0 + res_slot[i - n_sink] * page_rows;
        v = p;
        d = 0;
    }
};

// Q fragments: lane (g, t) holds Q[head g][64b + 16t + 8e .. +8] (heads >= G are zero)
__device__ __forceinline__ void load_q_frags(const FkvDims& D, const uint16_t* __restrict__ q, int u,
                                             uint4 (&qa)[2][2]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int b = u / D.n_kv, m = u % D.n_kv;
    const bool hv = g < D.G;
    const uint16_t* qrow = q + ((size_t)b * D.n_qo + m * D.G + (hv ? g : 0)) * kHeadDim;
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 2; ++e)
            qa[bb][e] = hv ? *reinterpret_cast<const uint4*>(qrow + 64 * bb + 16 * t + 8 * e) : make_uint4(0u, 0u, 0u, 0u);
}

// Attend entries [pa, pb) of a page list: online softmax over every token of those pages
// into (m_run, l_run, oacc) -- lane (g, t) holds heads 2t, 2t+1.  One warp; ring/bar are
// the warp's NST slab stages, phase_bits their parities (carried across calls).
template <int NST, class Src>
__device__ __forceinline__ void attend_pages(const FkvDims& D, const FkvScratch& X, const uint4 (&qa)[2][2],
                                             const CUtensorMap* tmap_p, const CUtensorMap* tmap_hp, const Src& src,
                                             int pa, int pb, uint8_t* ring, uint64_t* bars, uint32_t& phase_bits,
                                             float (&m_run)[2], float (&l_run)[2], float (&oacc)[8][4], int tcls,
                                             int w, int pre = 0, int skip = 0, int trim = 0) {
    // pre: the first `pre` slabs of this range are already in flight in stages 0..pre-1 (issued
    // from the same rows before the PDL wait).  skip / trim: the range starts `skip` slabs into
    // entry pa and ends `trim` slabs before the end of entry pb - 1 (slab-granular split)
    constexpr int kStages = NST;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int spp = D.p >> 4, lspp = spp == 1 ? 0 : (spp == 2 ? 1 : 2);
    const float sc = D.attn_c;
    const CUtensorMap& tmap = *tmap_p;
    const CUtensorMap& tmap_h = *tmap_hp;
    // the segment's pages in chunks of <= 32 (one page-table entry per lane)
    for (int cb = pa; cb < pb; cb += 32) {
        const int np = min(32, pb - cb);
        // page list of the segment, one page per lane: first K row and valid tokens -- one
        // batch of independent loads instead of a dependent load per slab
        int my_row = 0, my_valid = 0, my_dst = 0;
        if (lane < np) src.load(cb + lane, my_row, my_valid, my_dst);
        const unsigned host_mask = __ballot_sync(0xffffffffu, my_valid & 0x80);  // pages read from the host pool
        const int nx = np * spp - (cb + 32 >= pb ? trim : 0);  // last chunk: drop the trimmed slabs
        const int i0 = cb == pa ? skip : 0;
        if (lane == 0) trace_stamp(X.trace, tcls, w, 1);
        auto slab_of = [&](int x, int& row) {  // warp-uniform; spp = 1 << lspp
            const int pi = x >> lspp, sl = x & (spp - 1);
            row = __shfl_sync(0xffffffffu, my_row, pi) + sl * 16;
            return (__shfl_sync(0xffffffffu, my_valid, pi) & 0x7f) - sl * 16;
        };
        auto is_host = [&](int x) { return (host_mask >> (x >> lspp)) & 1u; };
        // prologue: first kStages slabs of this segment in flight
        int rows[kStages], valids[kStages];
#pragma unroll
        for (int i = 0; i < kStages; ++i) valids[i] = i0 + i < nx ? slab_of(i0 + i, rows[i]) : 0;
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < kStages; ++i)
                if (valids[i] > 0 && !(cb == pa && i < pre))
                    issue_slab(is_host(i0 + i) ? &tmap_h : &tmap, ring + i * kSlabBytes, &bars[i], rows[i], D.p);
        }
        for (int i = i0; i < nx; ++i) {
            const int stg = (i - i0) % kStages;
            int row;
            const int valid = slab_of(i, row);
            int row2 = 0, valid2 = 0;
            if (i + kStages < nx) valid2 = slab_of(i + kStages, row2);
            const int dst = host_mask ? __shfl_sync(0xffffffffu, my_dst, i >> lspp) + (i & (spp - 1)) * 16 : 0;
            if (valid > 0) {
                mbar_wait(&bars[stg], (phase_bits >> stg) & 1u);
                phase_bits ^= 1u << stg;
                if (i == 0 && lane == 0) trace_stamp(X.trace, tcls, w, 2);
                compute_slab(ring + stg * kSlabBytes, valid, qa, sc, g, t, m_run, l_run, oacc);
            }
            __syncwarp();  // every lane is done with this stage before it is refilled
            if (lane == 0) {
                if (valid > 0 && is_host(i)) {
                    store_slab(&tmap, ring + stg * kSlabBytes, dst, D.p);  // recall fused: cache the page
                    if (valid2 > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
                if (valid2 > 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue_slab(is_host(i + kStages) ? &tmap_h : &tmap, ring + stg * kSlabBytes, &bars[stg],
                               row2, D.p);
                }
            }
        }
        if (host_mask && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

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

// ---- clustered attention: one cluster of C CTAs (4 warps each) per unit; warp k of the
// 4C warps attends pages [k P_max / 4C, (k+1) P_max / 4C) of the unit's list, leaves its
// partial record (unnormalised o, running max m, sum l per head) in its own shared memory,
// and after one cluster barrier the leader CTA merges the 4C records over DSMEM, writes
// the output and commits the speculative advance (row a8) -- no global records, no second
// kernel.  Units have (almost) equal page counts, so the per-unit split stays balanced.
template <int NST, int C>
__global__ void __launch_bounds__(kAttnWarpsPerCta * 32, NST == 2 ? 3 : 2)
    fkv_attn_cluster_kernel(FkvDims D, FkvLayer L, FkvScratch X, const uint16_t* __restrict__ q,
                            float* __restrict__ out, int phase, const __grid_constant__ CUtensorMap tmap,
                            const __grid_constant__ CUtensorMap tmap_h, int commit) {
    constexpr int kStages = NST, W = kAttnWarpsPerCta, NW = W * C;
    extern __shared__ __align__(1024) uint8_t s_stage[];  // [W][kStages][8 KiB]; then the records
    __shared__ __align__(8) uint64_t bar[W][kStages];
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const int rk = blockIdx.x / C;  // rank of this cluster's unit among the phase's units
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int g = lane >> 2, t = lane & 3;
    const int G = D.G;
    pdl_trigger();
    const int tcls = 4 + phase;
    const int w = rk * NW + crank * W + warp;  // trace entity
    if (lane == 0) trace_stamp(X.trace, tcls, w, 0);
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
    // slabs; whole entries [pa, pbc) minus `skip` slabs at the front and `trim` at the back).
    // The speculative-attention mode splits by whole entries.
    const int spp = D.p >> 4, TS = D.attn_spec ? D.P_max : D.P_max * spp, gran = D.attn_spec ? 1 : spp;
    const int sa = (int)((long long)k * TS / NW), sb = (int)((long long)(k + 1) * TS / NW);
    const int pa = sa / gran, pbc = (sb + gran - 1) / gran;
    const int skip = sa - pa * gran, trim = pbc * gran - sb;
    float oacc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) oacc[i][j] = 0.0f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.0f, 0.0f};
    uint4 qa[2][2];
    // ---- speculative attention (phase 0), before the PDL wait: the sink pages and the
    // resident set R of step i-1 form the head of every page list a unit without a
    // correction attends at step i -- R is state the select kernel does not modify,
    // so this warp streams its part of it while the select is still running.  After the wait
    // a corrected unit discards that work and starts over from its new page list; the rest
    // continue with the local pages (which include this step's token).  The select triggers
    // this launch only after its own PDL wait, so the previous layer is complete and q_i may
    // be read here.
    int spec_end = pa;  // entries [pa, spec_end) attended speculatively
    int pre = 0;        // slabs of entry pa prefetched speculatively (default mode)
    if (phase == 0 && rk < D.U && pa < pbc && !D.attn_spec && !(D.dbg & 8)) {
        // default: only prefetch this warp's first slabs if they lie in the sink + R head of the
        // list (rows from state the select does not modify); a corrected unit drains them
        const int u0 = rk;
        const int rv = L.res_valid[u0], rc = L.res_cnt[u0], ctx_any = L.ctx[u0];
        int slot_of[kStages];
#pragma unroll
        for (int x = 0; x < kStages; ++x) {
            const int a = pa + (skip + x) / spp - D.n_sink;
            slot_of[x] = (a >= 0 && a < D.K) ? L.res_slot[(size_t)u0 * D.K + a] : 0;
        }
        if (rv && !D.full_refresh && ctx_any >= D.S_tok) {
            const int n_spec = D.n_sink + rc, pr = 2 * D.p;
            int row[kStages];
#pragma unroll
            for (int x = 0; x < kStages; ++x) {
                const int pi = pa + (skip + x) / spp;
                row[x] = -1;
                if (pa * spp + skip + x < sb && pi < n_spec)
                    row[x] = (pi < D.n_sink ? (int)((L.sink - L.arena) / kHeadDim) + (u0 * D.n_sink + pi) * pr
                                            : (int)((L.slots - L.arena) / kHeadDim) + (u0 * 2 * D.K + slot_of[x]) * pr) +
                             ((skip + x) % spp) * 16;
            }
            while (pre < kStages && row[pre] >= 0) ++pre;
            if (lane == 0)
                for (int x = 0; x < pre; ++x) issue_slab(&tmap, ring + x * kSlabBytes, &bar[warp][x], row[x], D.p);
        }
    }
    if (phase == 0 && rk < D.U && pa < pbc && D.attn_spec) {  // FREEKV_ATTN_SPEC=1 (off by default: measured
                                                               // slower, it competes with the select)
        const int u0 = rk;
        const int rv = L.res_valid[u0], rc = L.res_cnt[u0], ctx_any = L.ctx[u0];
        load_q_frags(D, q, u0, qa);
        if (rv && !D.full_refresh && ctx_any >= D.S_tok) {
            spec_end = min(pbc, D.n_sink + rc);
            if (spec_end > pa) {
                const int pr = 2 * D.p;  // arena rows per page
                const SpecSrc ssrc{(int)((L.sink - L.arena) / kHeadDim) + u0 * D.n_sink * pr,
                                   (int)((L.slots - L.arena) / kHeadDim) + u0 * 2 * D.K * pr, pr, D.n_sink,
                                   L.res_slot + (size_t)u0 * D.K, D.p};
                attend_pages<NST>(D, X, qa, &tmap, &tmap_h, ssrc, pa, spec_end, ring, bar[warp], phase_bits, m_run,
                                  l_run, oacc, tcls, w);
            } else {
                spec_end = pa;
            }
        }
    }
    pdl_wait();  // the select kernel's page lists and flags are complete
    int u = rk, nu = D.U;
    if (phase != 0) {
        int d1;
        nu = phase_units(D, L, phase, rk, lane, u, d1);
    }
    if (rk >= nu) return;  // cluster-uniform: no unit for this cluster in this phase
    if (spec_end > pa && L.flags[u]) {  // corrected unit: its pages are S_i, not R -- start over
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) oacc[i][j] = 0.0f;
        m_run[0] = m_run[1] = -INFINITY;
        l_run[0] = l_run[1] = 0.0f;
        spec_end = pa;
    }
    if (spec_end == pa) load_q_frags(D, q, u, qa);
    if (pre > 0 && L.flags[u]) {  // corrected unit: the prefetched slabs are not its pages
        for (int x = 0; x < pre; ++x) {
            mbar_wait(&bar[warp][x], (phase_bits >> x) & 1u);
            phase_bits ^= 1u << x;
        }
        pre = 0;
    }
    {
        const TableSrc tsrc{X.page_rows + (size_t)u * D.P_max, X.page_valid + (size_t)u * D.P_max,
                            X.page_dst + (size_t)u * D.P_max};
        const int pe = min(pbc, X.page_cnt[u]);
        attend_pages<NST>(D, X, qa, &tmap, &tmap_h, tsrc, spec_end, pe, ring, bar[warp], phase_bits, m_run, l_run,
                          oacc, tcls, w, pre, spec_end == pa ? skip : 0, pe == pbc ? trim : 0);
    }
    if (lane == 0) trace_stamp(X.trace, tcls, w, 3);
    // ---- this warp's record, in its own (now idle) ring: o [G][128], then m [G], l [G]
    __syncwarp();
    float* rec = reinterpret_cast<float*>(ring);
    float l0 = l_run[0], l1 = l_run[1];
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    if (g == 0) {
        if (2 * t < G) {
            rec[G * kHeadDim + 2 * t] = m_run[0];
            rec[G * kHeadDim + G + 2 * t] = l0;
        }
        if (2 * t + 1 < G) {
            rec[G * kHeadDim + 2 * t + 1] = m_run[1];
            rec[G * kHeadDim + G + 2 * t + 1] = l1;
        }
    }
    const int base0 = 64 * (g >> 2) + 8 * (g & 3);  // see the split kernel's record layout
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        const int h = 2 * t + hh;
        if (h < G) {
            float* dst = rec + h * kHeadDim + base0;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                float4* d4 = reinterpret_cast<float4*>(dst + 32 * half);
                const int mb = 4 * half;
                d4[0] = make_float4(oacc[mb][hh], oacc[mb][2 + hh], oacc[mb + 1][hh], oacc[mb + 1][2 + hh]);
                d4[1] = make_float4(oacc[mb + 2][hh], oacc[mb + 2][2 + hh], oacc[mb + 3][hh], oacc[mb + 3][2 + hh]);
            }
        }
    }
    // the leader's commit / q_prev inputs, loaded before the barrier (independent of the records)
    constexpr int kQv = (kMaxG * (kHeadDim / 4) + kAttnWarpsPerCta * 32 - 1) / (kAttnWarpsPerCta * 32);
    uint2 qv[kQv];
    int cp_page = 0, cp_slot = 0, cp_front = 0, cp_cnt = 0;
    if (crank == 0) {
        const int b = u / D.n_kv, m = u % D.n_kv;
#pragma unroll
        for (int i = 0; i < kQv; ++i) {
            const int e = tid + i * (int)blockDim.x;
            if (e < G * (kHeadDim / 4)) {
                const size_t row = (size_t)b * D.n_qo + m * G + e / (kHeadDim / 4);
                qv[i] = reinterpret_cast<const uint2*>(q + row * kHeadDim)[e % (kHeadDim / 4)];
            }
        }
        if (commit == 0 && tid < D.K) {
            cp_page = L.pend_pages[(size_t)u * D.K + tid];
            cp_slot = L.pend_slot[(size_t)u * D.K + tid];
        }
        if (commit == 0 && tid == 0) {
            cp_front = L.pend_front[u];
            cp_cnt = L.pend_cnt[u];
        }
    }
    cl.sync();  // every record of the unit is in its CTA's shared memory
    if (crank == 0) {
        if (tid == 0) trace_stamp(X.trace, 7, rk, 0);
        // thread -> (head h, 4 channels); records read over DSMEM, merged with an online max
        const int b = u / D.n_kv, m = u % D.n_kv;
#pragma unroll
        for (int qi = 0; qi < kQv; ++qi) {
            const int e = tid + qi * (int)blockDim.x;
            if (e >= G * (kHeadDim / 4)) break;
            const int h = e / (kHeadDim / 4), c4 = e % (kHeadDim / 4);
            constexpr int RB = NW < 8 ? NW : 8;  // records per batch (loads in flight together)
            float M = -INFINITY, Ls = 0.0f;
            float4 O = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
            for (int r0 = 0; r0 < NW; r0 += RB) {
                float mv[RB], lv[RB];
                float4 ov[RB];
#pragma unroll
                for (int i = 0; i < RB; ++i) {
                    const int r = r0 + i;
                    const float* rr = cl.map_shared_rank(
                        reinterpret_cast<float*>(s_stage + (r % W) * (kStages * kSlabBytes)), r / W);
                    mv[i] = rr[G * kHeadDim + h];
                    lv[i] = rr[G * kHeadDim + G + h];
                    ov[i] = reinterpret_cast<const float4*>(rr + h * kHeadDim)[c4];
                }
                float Mb = M;
#pragma unroll
                for (int i = 0; i < RB; ++i) Mb = fmaxf(Mb, mv[i]);
                if (Mb != -INFINITY) {
                    const float scl = exp2f(M - Mb);  // M = -inf -> 0
                    Ls *= scl;
                    O.x *= scl;
                    O.y *= scl;
                    O.z *= scl;
                    O.w *= scl;
#pragma unroll
                    for (int i = 0; i < RB; ++i) {
                        const float wgt = mv[i] == -INFINITY ? 0.0f : exp2f(mv[i] - Mb);
                        Ls += wgt * lv[i];
                        O.x += wgt * ov[i].x;
                        O.y += wgt * ov[i].y;
                        O.z += wgt * ov[i].z;
                        O.w += wgt * ov[i].w;
                    }
                    M = Mb;
                }
            }
            const size_t row = (size_t)b * D.n_qo + m * G + h;
            reinterpret_cast<float4*>(out + row * kHeadDim)[c4] = make_float4(O.x / Ls, O.y / Ls, O.z / Ls, O.w / Ls);
            reinterpret_cast<uint2*>(L.q_prev + row * kHeadDim)[c4] = qv[qi];  // q_prev := q_i
        }
        if (commit == 0) {  // commit: R := S_i
            if (tid < D.K) {
                L.res_pages[(size_t)u * D.K + tid] = cp_page;
                L.res_slot[(size_t)u * D.K + tid] = cp_slot;
            }
            for (int i = tid + (int)blockDim.x; i < D.K; i += blockDim.x) {  // K > block size
                L.res_pages[(size_t)u * D.K + i] = L.pend_pages[(size_t)u * D.K + i];
                L.res_slot[(size_t)u * D.K + i] = L.pend_slot[(size_t)u * D.K + i];
            }
            if (tid == 0) {
                L.res_front[u] = cp_front;
                L.res_cnt[u] = cp_cnt;
                L.res_valid[u] = 1;
            }
        }
        if (tid == 0) trace_stamp(X.trace, 7, rk, 1);
    }
    cl.sync();  // the leader has read every record: the other CTAs may exit
}

template <int NST, int C>
static cudaError_t launch_cluster_c(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                    float* out, int phase, const CUtensorMap& tmap, const CUtensorMap& tmap_h,
                                    int commit, bool pdl, cudaStream_t s) {
    auto kern = fkv_attn_cluster_kernel<NST, C>;
    const int smem = kAttnWarpsPerCta * NST * kSlabBytes;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.U * C);
    cfg.blockDim = dim3(kAttnWarpsPerCta * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, D, L, X, q, out, phase, tmap, tmap_h, commit);
}

// Clustered attention + merge + commit (replaces split + combine); c = CTAs per unit (1..8)
cudaError_t launch_attn_cluster(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                float* out, int phase, const CUtensorMap& tmap, const CUtensorMap& tmap_h,
                                int commit, int c, bool pdl, cudaStream_t s) {
    const int nst = attn_stages();
#define FKV_CL(NS)                                                                                          \
    do {                                                                                                    \
        if (c == 1) return launch_cluster_c<NS, 1>(D, L, X, q, out, phase, tmap, tmap_h, commit, pdl, s); \
        if (c == 2) return launch_cluster_c<NS, 2>(D, L, X, q, out, phase, tmap, tmap_h, commit, pdl, s); \
        if (c == 4) return launch_cluster_c<NS, 4>(D, L, X, q, out, phase, tmap, tmap_h, commit, pdl, s); \
        return launch_cluster_c<NS, 8>(D, L, X, q, out, phase, tmap, tmap_h, commit, pdl, s);             \
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

template <int NST, int WPC>
static cudaError_t attn_config() {
    const int smem = WPC * NST * kSlabBytes;
    cudaError_t e = cudaFuncSetAttribute(fkv_attn_split_kernel<NST, WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    // every kernel of the path prefers the max-shared carveout, so consecutive kernels never
    // force an L1/shared-memory reconfiguration of the SMs
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fkv_attn_split_kernel<NST, WPC>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
    return e;
}

template <int NST>
static cudaError_t attn_setup(int cps_want, int* warps) {
    const int smem = kAttnWarpsPerCta * NST * kSlabBytes;
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = attn_config<NST, 4>();
    if (e == cudaSuccess) e = NST == 2 ? attn_config<2, 8>() : attn_config<3, 8>();
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fkv_attn_combine_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fkv_attn_split_kernel<NST, 4>,
                                                          kAttnWarpsPerCta * 32, smem);
    // CTAs per SM (FREEKV_ATTN_CTAS_PER_SM overrides the caller's choice): 2 when the attention
    // runs alone (8 warps per SM hide the per-slab MMA/softmax latency); 1 in the pipelined
    // step, where it leaves shared memory and registers to the select kernels running beside it
    const char* ce = getenv("FREEKV_ATTN_CTAS_PER_SM");
    const int cps = std::max(1, std::min(per_sm, ce ? atoi(ce) : cps_want));
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

// wpc = 8 (phase 1 of the overlapped step): one 8-warp CTA per SM, which cannot share an SM
// with a select CTA, so the two kernels split the SMs between them
cudaError_t launch_attn_split(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              int phase, const CUtensorMap& tmap, const CUtensorMap& tmap_h, const uint16_t* arena,
                              bool pdl, cudaStream_t s, int wpc) {
    const int T = phase == 1 ? D.attn_warps_p1 : D.attn_warps;
    const int nst = attn_stages();
#define FKV_ATTN(NS, W)                                                                                         \
    return launch_ex(fkv_attn_split_kernel<NS, W>, dim3((T + W - 1) / W), dim3(W * 32), W * NS * kSlabBytes, s, \
                     pdl, D, L, X, q, phase, tmap, tmap_h, arena)
    if (wpc == 8) {
        if (nst == 2) FKV_ATTN(2, 8);
        FKV_ATTN(3, 8);
    }
    if (nst == 2) FKV_ATTN(2, 4);
    if (nst == 4) FKV_ATTN(4, 4);
    FKV_ATTN(3, 4);
#undef FKV_ATTN
}

cudaError_t launch_attn_combine(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                float* out, int split, int commit, bool pdl, cudaStream_t s) {
    return launch_ex(fkv_attn_combine_kernel, dim3(D.U), dim3(kCombThreads), 0, s, pdl, D, L, X, q, out, split,
                     commit);
}

}  // namespace fkv
