// attn_core.cuh -- row a7 building blocks of the attention kernels (attn.cu): TMA slab staging
// of head-major (2, p, d) pages, the per-slab online-softmax step on mma.sync micro-tiles (S^T = K Q^T, O^T += V^T P^T), page-list sources
// and the per-warp page loop.  PAPER.md P:95-97 (sparse decode attention over the selected pages).
#pragma once
#include "fkv_internal.cuh"

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

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint32_t u4get(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
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

__device__ __forceinline__ void issue_slab(const CUtensorMap* map, uint8_t* st, uint64_t* bar, int row, int p,
                                           const uint16_t* arena = nullptr) {
    mbar_expect_tx(bar, kSlabBytes);
#ifdef FKV_ATTN_BULK  // A/B timing experiment only (unswizzled, wrong results): two 1D 4 KB copies
    if (arena) {
        bulk_g2s(st, arena + (size_t)row * 128, 2 * kBoxBytes, bar);
        bulk_g2s(st + 2 * kBoxBytes, arena + (size_t)(row + p) * 128, 2 * kBoxBytes, bar);
        return;
    }
#endif
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
        r = __ldcg(rows + i);  // L2: written by the concurrently running select kernel (mode 1)
        v = __ldcg(valid + i);
        d = __ldcg(dst + i);
    }
};
// The page list of a unit that attends its resident set R (not corrected this step),
// computed in the attention kernel from state the select kernel does not modify: sink pages,
// R's slots, local pages [f_R p, Lc) of the ring (reading A-9) -- the same entries the select
// kernel writes for a corrected unit's S_i.
struct ResSrc {
    int n_sp, n_sel, f, Lc, sink_tok, p, R_loc;
    int sink_row0, slot_row0, ring_row0, page_rows;  // arena rows of the unit's regions; rows per page
    const int32_t* res_slot;
    __device__ __forceinline__ void load(int i, int& r, int& v, int& d) const {
        d = 0;
        if (i < n_sp) {
            r = sink_row0 + i * page_rows;
            v = min(p, sink_tok - i * p);
        } else if (i < n_sp + n_sel) {
            r = slot_row0 + res_slot[i - n_sp] * page_rows;
            v = p;
        } else {
            const int j = f + (i - n_sp - n_sel);
            r = ring_row0 + (j % R_loc) * page_rows;
            v = min(p, Lc - j * p);
        }
    }
    __device__ __forceinline__ int count() const {
        const int n_last = (Lc - 1) / p;
        return n_sp + n_sel + ((Lc > f * p) ? (n_last - f + 1) : 0);
    }
};

// The dense page list of a unit (first_layer_dense, layer 0, O-7 / P:560): every page [0, Lc)
// from the dense pool
struct DenseSrc {
    int row0, p, Lc, page_rows;
    __device__ __forceinline__ void load(int i, int& r, int& v, int& d) const {
        d = 0;
        r = row0 + i * page_rows;
        v = min(p, Lc - i * p);
    }
    __device__ __forceinline__ int count() const { return (Lc + p - 1) / p; }
};

__device__ __forceinline__ ResSrc res_src(const FkvDims& D, const FkvLayer& L, int u, int Lc) {
    ResSrc s;
    s.p = D.p;
    s.R_loc = D.R_loc;
    s.Lc = Lc;
    s.sink_tok = min(D.S_tok, Lc);
    s.n_sp = (s.sink_tok + D.p - 1) / D.p;
    s.n_sel = L.res_cnt[u];
    s.f = L.res_front[u];
    s.page_rows = 2 * D.p;
    s.sink_row0 = (int)((L.sink - L.arena) / kHeadDim) + u * D.n_sink * s.page_rows;
    s.slot_row0 = (int)((L.slots - L.arena) / kHeadDim) + u * 2 * D.K * s.page_rows;
    s.ring_row0 = (int)((L.ring - L.arena) / kHeadDim) + u * D.R_loc * s.page_rows;
    s.res_slot = L.res_slot + (size_t)u * D.K;
    return s;
}

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
                    issue_slab(is_host(i0 + i) ? &tmap_h : &tmap, ring + i * kSlabBytes, &bars[i], rows[i], D.p,
                               is_host(i0 + i) ? nullptr : X.arena);
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
#ifndef FKV_ATTN_NOCOMPUTE
                compute_slab(ring + stg * kSlabBytes, valid, qa, sc, g, t, m_run, l_run, oacc);
#else
                oacc[0][0] += (float)ring[stg * kSlabBytes + lane];
#endif
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
                               row2, D.p, is_host(i + kStages) ? nullptr : X.arena);
                }
            }
        }
        if (host_mask && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// This warp's partial record of a unit: unnormalised o [G][128] (channel order of the MMA
// fragments, see the split kernel), then the running max m [G] and sum l [G] (relative to m).
// Lane (g, t) holds heads 2t, 2t+1; l is summed over the 8 lanes g of the same t.
__device__ __forceinline__ void write_record(float* rec, int G, const float (&oacc)[8][4], const float (&m_run)[2],
                                             const float (&l_run)[2]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
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
    const int base0 = 64 * (g >> 2) + 8 * (g & 3);
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
}

// Merge of the NW partial records of a unit (record r = warp r % W of CTA r / W, at `rec_of(r)`,
// possibly in another CTA's shared memory) into (o / l) for float4 e of the G x 128 output:
// online max over batches of records loaded together.
template <int NW, class RecOf>
__device__ __forceinline__ float4 merge_records(int G, int e, RecOf rec_of) {
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
            const float* rr = rec_of(r0 + i);
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
    return make_float4(O.x / Ls, O.y / Ls, O.z / Ls, O.w / Ls);
}

}  // namespace fkv
