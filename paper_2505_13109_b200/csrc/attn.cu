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

struct Slab {
    uint4 k[2][4];  // K rows slab*16 + nt*8 + g, channels 32c + 8t .. +7
    uint4 v[4][2];  // V rows 2t, 2t+1, 2t+8, 2t+9; channels 16g + 8h .. +7
    int valid;      // valid tokens of this slab (<= 0: empty)
};

__device__ __forceinline__ void load_slab(const FkvDims& D, const FkvLayer& L, int u, const UnitMeta& M, int x,
                                          int g, int t, Slab& S) {
    const int spp = D.p >> 4;
    const int pi = x / spp, slab = x - pi * spp;
    int pv;
    const uint16_t* base = page_ptr(D, L, u, M, pi, pv);
    S.valid = pv - slab * 16;
    if (S.valid <= 0) return;
    const uint16_t* Kp = base + (size_t)slab * 16 * kHeadDim;
    const uint16_t* Vp = base + (size_t)D.p * kHeadDim + (size_t)slab * 16 * kHeadDim;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int c = 0; c < 4; ++c) S.k[nt][c] = ldg_stream(Kp + (size_t)(nt * 8 + g) * kHeadDim + 32 * c + 8 * t);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int tok = 2 * t + (r & 1) + (r >> 1) * 8;
#pragma unroll
        for (int h = 0; h < 2; ++h) S.v[r][h] = ldg_stream(Vp + (size_t)tok * kHeadDim + 16 * g + 8 * h);
    }
}

__device__ __forceinline__ void compute_slab(const Slab& S, const uint4 (&qa)[4], float sc, int t, float& m_run,
                                             float& l_run, float (&oacc)[8][4]) {
    if (S.valid <= 0) return;
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
                mma16816(s[nt], u4get(qa[c], 2 * sh), 0u, u4get(qa[c], 2 * sh + 1), 0u, u4get(S.k[nt][c], 2 * sh),
                         u4get(S.k[nt][c], 2 * sh + 1));
    }
    // ---- online softmax (row = head g; the 4 lanes of a quad share a row)
    float x[2][2];
    float smax = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int tok = nt * 8 + 2 * t + e;
            x[nt][e] = tok < S.valid ? s[nt][e] * sc : -INFINITY;
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
        const uint32_t x0 = u4get(S.v[0][mt >> 2], mt & 3);  // token 2t
        const uint32_t x1 = u4get(S.v[1][mt >> 2], mt & 3);  // token 2t+1
        const uint32_t x8 = u4get(S.v[2][mt >> 2], mt & 3);  // token 2t+8
        const uint32_t x9 = u4get(S.v[3][mt >> 2], mt & 3);  // token 2t+9
        const uint32_t A0 = __byte_perm(x0, x1, 0x5410);
        const uint32_t A1 = __byte_perm(x0, x1, 0x7632);
        const uint32_t A2 = __byte_perm(x8, x9, 0x5410);
        const uint32_t A3 = __byte_perm(x8, x9, 0x7632);
        mma16816(oacc[mt], A0, A1, A2, A3, bh0, bh1);
        mma16816(oacc[mt], A0, A1, A2, A3, bl0, bl1);
    }
}

__device__ __forceinline__ long long range_start(long long w, long long V, long long T) { return w * V / T; }

// phase: 0 = every unit; 1 = unflagged units only (their pages are resident, so this
// half runs while the synchronous recall of the corrected units is in flight);
// 2 = corrected units only (after that recall).  Each unit is attended in exactly
// one phase, so every partial record is written once per step.
__global__ void __launch_bounds__(kAttnWarpsPerCta * 32, 2) fkv_attn_split_kernel(FkvDims D, FkvLayer L,
                                                                                   FkvScratch X,
                                                                                   const uint16_t* __restrict__ q,
                                                                                   int phase) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int w = blockIdx.x * kAttnWarpsPerCta + warp;
    const int T = D.attn_warps;
    if (w >= T) return;
    const long long V = (long long)D.U * D.P_max;
    const long long s0 = range_start(w, V, T), s1 = range_start(w + 1, V, T);
    const int G = D.G, spp = D.p >> 4;
    const float sc = D.attn_c;
    int k_rec = 0;
    for (long long seg = s0; seg < s1; ++k_rec) {
        const int u = (int)(seg / D.P_max);
        const long long seg_end = min(s1, (long long)(u + 1) * D.P_max);
        if (phase != 0 && ((L.flags[u] != 0) != (phase == 2))) {
            seg = seg_end;  // this unit is attended in the other phase
            continue;
        }
        const UnitMeta M = load_meta(D, L, u);
        const int pa = (int)(seg - (long long)u * D.P_max);
        const int pb = min((int)(seg_end - (long long)u * D.P_max), M.n_pages);
        seg = seg_end;
        const int b = u / D.n_kv, m = u % D.n_kv;
        // Q fragments: lane (g, t) holds Q[head g][32c + 8t .. 8t+7], c = 0..3 (heads >= G are zero)
        uint4 qa[4];
        {
            const bool hv = g < G;
            const uint16_t* qrow = q + ((size_t)b * D.n_qo + m * G + (hv ? g : 0)) * kHeadDim;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                qa[c] = hv ? *reinterpret_cast<const uint4*>(qrow + 32 * c + 8 * t) : make_uint4(0u, 0u, 0u, 0u);
        }
        float oacc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) oacc[i][k] = 0.0f;
        float m_run = -INFINITY, l_run = 0.0f;
        const int x0 = pa * spp, nx = pb > pa ? (pb - pa) * spp : 0;
        Slab A, B;
        if (nx > 0) load_slab(D, L, u, M, x0, g, t, A);
        for (int x = 0; x < nx; x += 2) {
            if (x + 1 < nx) load_slab(D, L, u, M, x0 + x + 1, g, t, B);
            compute_slab(A, qa, sc, t, m_run, l_run, oacc);
            if (x + 1 < nx) {
                if (x + 2 < nx) load_slab(D, L, u, M, x0 + x + 2, g, t, A);
                compute_slab(B, qa, sc, t, m_run, l_run, oacc);
            }
        }
        // ---- partial record (w, k_rec) of unit u: unnormalised, relative to m_run
        float l_tot = l_run;
        l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 1);
        l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
        const size_t rec = (size_t)w * 2 + k_rec;
        if (t == 0 && g < G) {
            X.part_ml[(rec * G + g) * 2 + 0] = m_run;
            X.part_ml[(rec * G + g) * 2 + 1] = l_tot;
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int h = 2 * t + hh;
            if (h < G) {
                float4* dst = reinterpret_cast<float4*>(X.part_o + (rec * G + h) * kHeadDim + 16 * g);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    dst[q4] = make_float4(oacc[2 * q4][hh], oacc[2 * q4][2 + hh], oacc[2 * q4 + 1][hh],
                                          oacc[2 * q4 + 1][2 + hh]);
            }
        }
    }
}

// Merge a unit's partial records and commit the speculative advance (row a8).
// Phase 1 stages every record's (m, l) in shared memory, phase 2 turns them
// into weights 2^(m_r - M) / L per head, phase 3 has thread (h, c) reduce the
// weighted partial outputs.
constexpr int kMaxRecs = 256;

__global__ void __launch_bounds__(1024) fkv_attn_combine_kernel(FkvDims D, FkvLayer L, FkvScratch X,
                                                                const uint16_t* __restrict__ q,
                                                                float* __restrict__ out) {
    __shared__ int s_rec[kMaxRecs];
    __shared__ int s_nrec, s_first;
    __shared__ float s_ml[kMaxRecs * kMaxG * 2];
    __shared__ float s_w[kMaxRecs * kMaxG];
    const int u = blockIdx.x, b = u / D.n_kv, m = u % D.n_kv, G = D.G;
    const long long V = (long long)D.U * D.P_max, T = D.attn_warps;
    const long long x0 = (long long)u * D.P_max, x1 = x0 + D.P_max;
    // Records of unit u: the warps whose range [start(w), start(w+1)) intersects
    // [x0, x1).  Every warp owns >= 1 page (T <= V), so they are the contiguous run
    // w_first..w_last; candidates are tested in parallel with 32-bit arithmetic
    // (T * V < 2^31 and records <= kMaxRecs are guaranteed on the host).
    if (threadIdx.x == 0) {
        s_nrec = 0;
        s_first = 0x7fffffff;
    }
    __syncthreads();
    {
        const unsigned Ti = (unsigned)T, Vi = (unsigned)V;
        const int w_lo = max(0, (int)(((long long)x0 * Ti) / Vi) - 1);
        for (int w = w_lo + (int)threadIdx.x; w < (int)Ti && w < w_lo + kMaxRecs + 2; w += blockDim.x) {
            const int a = (int)((unsigned)w * Vi / Ti), e = (int)((unsigned)(w + 1) * Vi / Ti);
            if (e > (int)x0 && a < (int)x1) {
                atomicMin(&s_first, w);
                atomicAdd(&s_nrec, 1);
            }
        }
        __syncthreads();
        for (int w = w_lo + (int)threadIdx.x; w < (int)Ti && w < w_lo + kMaxRecs + 2; w += blockDim.x) {
            const int a = (int)((unsigned)w * Vi / Ti), e = (int)((unsigned)(w + 1) * Vi / Ti);
            if (e > (int)x0 && a < (int)x1) s_rec[w - s_first] = w * 2 + ((a / D.P_max == u) ? 0 : 1);
        }
    }
    __syncthreads();
    const int nr = s_nrec;
    for (int i = threadIdx.x; i < nr * G * 2; i += blockDim.x) {
        const int r = i / (G * 2), rem = i % (G * 2);
        s_ml[i] = X.part_ml[(size_t)s_rec[r] * G * 2 + rem];
    }
    __syncthreads();
    if (threadIdx.x < G) {
        const int h = threadIdx.x;
        float M = -INFINITY;
        for (int r = 0; r < nr; ++r) M = fmaxf(M, s_ml[(r * G + h) * 2]);
        float Ls = 0.0f;
        for (int r = 0; r < nr; ++r) {
            const float mr = s_ml[(r * G + h) * 2];
            const float wgt = mr == -INFINITY ? 0.0f : exp2f(mr - M);
            s_w[r * G + h] = wgt;
            Ls += wgt * s_ml[(r * G + h) * 2 + 1];
        }
        const float inv = 1.0f / Ls;
        for (int r = 0; r < nr; ++r) s_w[r * G + h] *= inv;
    }
    __syncthreads();
    const int h = threadIdx.x / kHeadDim, c = threadIdx.x % kHeadDim;
    if (h < G) {
        // unconditional, unrolled loads keep all records' reads in flight (every listed
        // record was written this step; empty segments carry weight 0 and o = 0)
        float O = 0.0f;
        int r = 0;
        for (; r + 8 <= nr; r += 8) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = X.part_o[((size_t)s_rec[r + i] * G + h) * kHeadDim + c];
#pragma unroll
            for (int i = 0; i < 8; ++i) O += s_w[(r + i) * G + h] * v[i];
        }
        for (; r < nr; ++r) O += s_w[r * G + h] * X.part_o[((size_t)s_rec[r] * G + h) * kHeadDim + c];
        const size_t row = (size_t)b * D.n_qo + m * G + h;
        out[row * kHeadDim + c] = O;
        L.q_prev[row * kHeadDim + c] = q[row * kHeadDim + c];  // q_prev := q_i
    }
    for (int i = threadIdx.x; i < D.K; i += blockDim.x) {
        L.res_pages[(size_t)u * D.K + i] = L.pend_pages[(size_t)u * D.K + i];
        L.res_slot[(size_t)u * D.K + i] = L.pend_slot[(size_t)u * D.K + i];
    }
    if (threadIdx.x == 0) {
        L.res_front[u] = L.pend_front[u];
        L.res_cnt[u] = L.pend_cnt[u];
        L.res_valid[u] = 1;
    }
}

// Resident warps of the split kernel, minus headroom of ~1/8 of the CTA slots so
// the recall kernels (other streams) can be scheduled while attention runs.
cudaError_t attn_resident_warps(int* warps) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fkv_attn_split_kernel, kAttnWarpsPerCta * 32, 0);
    const int ctas = sms * per_sm;
    *warps = (ctas - ctas / 8) * kAttnWarpsPerCta;
    return e;
}

cudaError_t launch_attn_split(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              int phase, cudaStream_t s) {
    const int ctas = (D.attn_warps + kAttnWarpsPerCta - 1) / kAttnWarpsPerCta;
    fkv_attn_split_kernel<<<ctas, kAttnWarpsPerCta * 32, 0, s>>>(D, L, X, q, phase);
    return cudaGetLastError();
}

cudaError_t launch_attn_combine(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                float* out, cudaStream_t s) {
    fkv_attn_combine_kernel<<<D.U, D.G * kHeadDim, 0, s>>>(D, L, X, q, out);
    return cudaGetLastError();
}

}  // namespace fkv
