// attn.cu -- rows a7/a8: sparse decode attention over the gathered pages and
// the speculative advance.
//
// PAPER.md P:95-97 (§2.1): o_h = softmax(q_h K^T / sqrt(d)) V over the token
// set T = sink tokens U selected pages U local region (reading A-9),
// with the pages of S_i for corrected units and the resident set otherwise
// (P:223).  After attention the step commits R := S_i, q_prev := q_i
// (fig:algo1).
//
// Split-KV flash decode: each warp owns a chunk of pages of one unit and keeps
// an online softmax; a combine kernel merges the chunks.  The G <= 8 heads of a
// GQA group ride as one MMA tile so every KV byte is loaded once, straight
// from HBM into registers in MMA fragment order (no shared memory):
//   S = Q K^T  : mma.m16n8k16  A = Q (16 rows, heads 0..7 real), B = K^T
//   O^T = V^T P^T : mma.m16n8k16  A = V^T (d rows), B = P^T (heads as N = 8)
// The contraction order over d and over tokens is free, so the channel and
// token orders are permuted such that every lane issues contiguous 16-byte
// loads; V^T fragments are built with byte permutes.  P is split into bf16
// hi + lo parts (two PV MMAs) so its rounding stays ~2^-17, far inside the
// 2e-3 output tolerance (reading A-19/A-21).
#include "fkv_internal.cuh"

namespace fkv {

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

struct PageRef {
    const uint16_t* ptr;
    int valid;
};

// Resolve entry i of unit u's page list: sink pages, selected slots, local ring.
__device__ __forceinline__ PageRef page_at(const FkvDims& D, const FkvLayer& L, int u, int i, int Lc, int n_sp,
                                           int n_sel, const int32_t* sel_slot, int f, int n_loc) {
    const size_t pe = page_elems(D);
    PageRef r{nullptr, 0};
    const int sink_tok = min(D.S_tok, Lc);
    if (i < n_sp) {
        r.ptr = L.sink + ((size_t)u * D.n_sink + i) * pe;
        r.valid = min(D.p, sink_tok - i * D.p);
        return r;
    }
    i -= n_sp;
    if (i < n_sel) {
        r.ptr = L.slots + ((size_t)u * 2 * D.K + sel_slot[i]) * pe;
        r.valid = D.p;
        return r;
    }
    i -= n_sel;
    if (i < n_loc) {
        const int j = f + i;
        r.ptr = L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe;
        r.valid = min(D.p, Lc - j * D.p);
    }
    return r;
}

__global__ void __launch_bounds__(128) fkv_attn_split_kernel(FkvDims D, FkvLayer L, FkvScratch X,
                                                             const uint16_t* __restrict__ q) {
    const int u = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int ci = blockIdx.y * (blockDim.x >> 5) + warp;  // chunk index
    if (ci >= D.n_chunks) return;
    const int b = u / D.n_kv, m = u % D.n_kv, G = D.G, p = D.p;

    const int flag = L.flags[u];
    const int32_t* sel_pages = (flag ? L.pend_pages : L.res_pages) + (size_t)u * D.K;
    const int32_t* sel_slot = (flag ? L.pend_slot : L.res_slot) + (size_t)u * D.K;
    const int f = flag ? L.pend_front[u] : L.res_front[u];
    const int Lc = L.ctx[u];
    int n_sel = 0;
    for (int i = 0; i < D.K; ++i) n_sel += sel_pages[i] >= 0;
    const int n_sp = (min(D.S_tok, Lc) + p - 1) / p;
    const int n_last = (Lc - 1) / p;
    const int n_loc = (Lc > f * p) ? (n_last - f + 1) : 0;
    const int n_pages = n_sp + n_sel + n_loc;

    // Q fragments: lane (g, t) holds Q[head g][32c + 8t .. 8t+7] for c = 0..3
    uint4 qa[4];
    {
        const bool hv = g < G;
        const uint16_t* qrow = q + ((size_t)b * D.n_qo + m * G + (hv ? g : 0)) * kHeadDim;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            qa[c] = hv ? *reinterpret_cast<const uint4*>(qrow + 32 * c + 8 * t) : make_uint4(0u, 0u, 0u, 0u);
        }
    }
    float oacc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) oacc[i][k] = 0.0f;
    float m_run = -INFINITY, l_run = 0.0f;
    const float sc = D.attn_c;

    const int pg0 = ci * D.pages_per_chunk;
    const int pg1 = min(n_pages, pg0 + D.pages_per_chunk);
    for (int pi = pg0; pi < pg1; ++pi) {
        const PageRef pr = page_at(D, L, u, pi, Lc, n_sp, n_sel, sel_slot, f, n_loc);
        const uint16_t* Kp = pr.ptr;
        const uint16_t* Vp = pr.ptr + (size_t)p * kHeadDim;
        for (int slab = 0; slab < p / 16; ++slab) {
            // ---- loads: K rows (tokens slab*16 + nt*8 + g), V rows (2t, 2t+1, 2t+8, 2t+9)
            uint4 kr[2][4], vr[4][2];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    kr[nt][c] = ldg_stream(Kp + (size_t)(slab * 16 + nt * 8 + g) * kHeadDim + 32 * c + 8 * t);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int tok = slab * 16 + 2 * t + (r & 1) + (r >> 1) * 8;
#pragma unroll
                for (int h = 0; h < 2; ++h) vr[r][h] = ldg_stream(Vp + (size_t)tok * kHeadDim + 16 * g + 8 * h);
            }
            // ---- S = Q K^T for two n-tiles of 8 tokens
            float s[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
                for (int k = 0; k < 4; ++k) s[nt][k] = 0.0f;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int sh = 0; sh < 2; ++sh)
                        mma16816(s[nt], u4get(qa[c], 2 * sh), 0u, u4get(qa[c], 2 * sh + 1), 0u,
                                 u4get(kr[nt][c], 2 * sh), u4get(kr[nt][c], 2 * sh + 1));
            }
            // ---- online softmax (row = head g; 4 lanes of a quad share a row)
            float x[2][2];
            float smax = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int tok = slab * 16 + nt * 8 + 2 * t + e;
                    x[nt][e] = tok < pr.valid ? s[nt][e] * sc : -INFINITY;
                    smax = fmaxf(smax, x[nt][e]);
                }
            smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, 1));
            smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, 2));
            const float m_new = fmaxf(m_run, smax);
            const float alpha = (m_new == -INFINITY) ? 1.0f : exp2f(m_run - m_new);
            float pv[2][2];
            float psum = 0.0f;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    pv[nt][e] = (m_new == -INFINITY) ? 0.0f : exp2f(x[nt][e] - m_new);
                    psum += pv[nt][e];
                }
            l_run = l_run * alpha + psum;
            m_run = m_new;
            const float a0 = __shfl_sync(0xffffffffu, alpha, (2 * t) * 4);
            const float a1 = __shfl_sync(0xffffffffu, alpha, (2 * t + 1) * 4);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                oacc[mt][0] *= a0;
                oacc[mt][1] *= a1;
                oacc[mt][2] *= a0;
                oacc[mt][3] *= a1;
            }
            // ---- P^T fragments, hi + lo bf16 split
            const uint32_t bh0 = pack_bf16(pv[0][0], pv[0][1]);
            const uint32_t bh1 = pack_bf16(pv[1][0], pv[1][1]);
            const __nv_bfloat162 h0 = *reinterpret_cast<const __nv_bfloat162*>(&bh0);
            const __nv_bfloat162 h1 = *reinterpret_cast<const __nv_bfloat162*>(&bh1);
            const uint32_t bl0 = pack_bf16(pv[0][0] - __low2float(h0), pv[0][1] - __high2float(h0));
            const uint32_t bl1 = pack_bf16(pv[1][0] - __low2float(h1), pv[1][1] - __high2float(h1));
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
    }
    // ---- partial results of this chunk (unnormalised, relative to m_run)
    float l_tot = l_run;
    l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 1);
    l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
    const size_t cbase = (size_t)u * D.n_chunks + ci;
    if (t == 0 && g < G) {
        X.part_ml[(cbase * G + g) * 2 + 0] = m_run;
        X.part_ml[(cbase * G + g) * 2 + 1] = l_tot;
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        const int h = 2 * t + hh;
        if (h < G) {
            float4* dst = reinterpret_cast<float4*>(X.part_o + (cbase * G + h) * kHeadDim + 16 * g);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
                dst[q4] = make_float4(oacc[2 * q4][hh], oacc[2 * q4][2 + hh], oacc[2 * q4 + 1][hh],
                                      oacc[2 * q4 + 1][2 + hh]);
        }
    }
}

// Merge chunk partials and commit the speculative advance (row a8).
__global__ void __launch_bounds__(1024) fkv_attn_combine_kernel(FkvDims D, FkvLayer L, FkvScratch X,
                                                                const uint16_t* __restrict__ q,
                                                                float* __restrict__ out) {
    const int u = blockIdx.x, b = u / D.n_kv, m = u % D.n_kv, G = D.G;
    const int h = threadIdx.x / kHeadDim, c = threadIdx.x % kHeadDim;
    if (h < G) {
        float M = -INFINITY;
        for (int ci = 0; ci < D.n_chunks; ++ci)
            M = fmaxf(M, X.part_ml[(((size_t)u * D.n_chunks + ci) * G + h) * 2]);
        float Ls = 0.0f, O = 0.0f;
        for (int ci = 0; ci < D.n_chunks; ++ci) {
            const size_t cb = ((size_t)u * D.n_chunks + ci) * G + h;
            const float mc = X.part_ml[cb * 2];
            if (mc == -INFINITY) continue;
            const float w = exp2f(mc - M);
            Ls += w * X.part_ml[cb * 2 + 1];
            O += w * X.part_o[cb * kHeadDim + c];
        }
        const size_t row = (size_t)b * D.n_qo + m * G + h;
        out[row * kHeadDim + c] = O / Ls;
        L.q_prev[row * kHeadDim + c] = q[row * kHeadDim + c];  // q_prev := q_i
    }
    for (int i = threadIdx.x; i < D.K; i += blockDim.x) {
        L.res_pages[(size_t)u * D.K + i] = L.pend_pages[(size_t)u * D.K + i];
        L.res_slot[(size_t)u * D.K + i] = L.pend_slot[(size_t)u * D.K + i];
    }
    if (threadIdx.x == 0) {
        L.res_front[u] = L.pend_front[u];
        L.res_valid[u] = 1;
    }
}

cudaError_t launch_attn_split(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              cudaStream_t s) {
    const int warps = 4;
    const dim3 grid(D.U, (D.n_chunks + warps - 1) / warps);
    fkv_attn_split_kernel<<<grid, warps * 32, 0, s>>>(D, L, X, q);
    return cudaGetLastError();
}

cudaError_t launch_attn_combine(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                float* out, cudaStream_t s) {
    fkv_attn_combine_kernel<<<D.U, D.G * kHeadDim, 0, s>>>(D, L, X, q, out);
    return cudaGetLastError();
}

}  // namespace fkv
