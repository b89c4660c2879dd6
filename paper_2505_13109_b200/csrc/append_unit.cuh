// append_unit.cuh -- row a9 for one unit, executed by one CTA: append new token
// rows, and when a page completes build its channel-wise min/max summary
// and store it to the pinned host pool as one (2, p, d) page
// (the NHD -> HND transpose at offload).
//
// Offload happens when a page COMPLETES (not when it later leaves the window):
// the page's bytes and summary are the same either way, and doing it early
// means the selection of the step at which the page becomes a candidate never
// waits for this step's append (requires W >= p, i.e. n_win >= 1; with W = 0
// the caller runs the append before scoring).  Pages are processed in
// ascending order by one CTA, so ring reuse (page j and j + R_loc share a
// slot) is race-free.
#pragma once
#include "fkv_internal.cuh"

namespace fkv {

// total order on finite bf16 with -0 < +0 (reading R-5)
__device__ __forceinline__ uint16_t sort_key(uint16_t b) {
    return (b & 0x8000u) ? (uint16_t)~b : (uint16_t)(b | 0x8000u);
}
__device__ __forceinline__ uint16_t from_key(uint16_t k) {
    return (k & 0x8000u) ? (uint16_t)(k & 0x7fffu) : (uint16_t)~k;
}

__device__ __forceinline__ void summarize_smem_page(const FkvDims& D, const FkvLayer& L, int u, int j,
                                                    const uint16_t* ks) {
    for (int c = threadIdx.x; c < D.d; c += blockDim.x) {
        uint16_t lo = sort_key(ks[c]), hi = lo;
        for (int r = 1; r < D.p; ++r) {
            const uint16_t kk = sort_key(ks[r * D.d + c]);
            lo = kk < lo ? kk : lo;
            hi = kk > hi ? kk : hi;
        }
        L.summ[summ_off(D, u, c >> 3, 0, j) + (c & 7)] = from_key(lo);
        L.summ[summ_off(D, u, c >> 3, 1, j) + (c & 7)] = from_key(hi);
    }
}

// Append n_new tokens (k, v: [nb][n_new][n_kv][d] bf16) to unit u.  L0 = context
// before the append.  sm: 2*p*d bf16 of shared memory.  Every thread of the CTA
// must call this (it synchronises on page completion).  Does not update ctx/n_off.
__device__ __forceinline__ void append_unit(const FkvDims& D, const FkvLayer& L, int u, int L0,
                                            const uint16_t* __restrict__ k, const uint16_t* __restrict__ v,
                                            int n_new, uint4* sm) {
    const int b = u / D.n_kv, m = u % D.n_kv;
    const int p = D.p, d = D.d, row_u4 = d / 8, page_u4 = 2 * p * row_u4;
    const int L1 = L0 + n_new;
    const int n_last = (L1 - 1) / p;
    const int ring_lo = max(D.n_sink, n_last - D.R_loc + 1);
    const size_t pe = page_elems(D);
    for (int j = L0 / p; j <= n_last; ++j) {
        const int t0 = j * p;
        uint4* dst = nullptr;  // resident home of page j after this append (sink area or local ring)
        if (j < D.n_sink)
            dst = reinterpret_cast<uint4*>(L.sink + ((size_t)u * D.n_sink + j) * pe);
        else if (j >= ring_lo)
            dst = reinterpret_cast<uint4*>(L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe);
        const bool completes = j >= D.n_sink && t0 + p <= L1;
        // dense layer (first_layer_dense): every page also in its dense-pool home
        uint4* dn = L.dense ? reinterpret_cast<uint4*>(L.dense + ((size_t)u * D.n_page_max + j) * pe) : nullptr;
        if (!completes) {
            // fast path (most decode steps): copy the new token rows straight to their page
            if (dst || dn) {
                const int ta = max(t0, L0), tb = min(t0 + p, L1);
                const int n_u4 = (tb - ta) * row_u4;
                for (int i = threadIdx.x; i < 2 * n_u4; i += blockDim.x) {
                    const int kv = i / n_u4, rem = i % n_u4, r = rem / row_u4, c = rem % row_u4;
                    const int t = ta + r;
                    const uint16_t* src = (kv == 0 ? k : v) + (((size_t)b * n_new + (t - L0)) * D.n_kv + m) * d;
                    const uint4 val = reinterpret_cast<const uint4*>(src)[c];
                    if (dst) dst[((size_t)kv * p + (t - t0)) * row_u4 + c] = val;
                    if (dn) dn[((size_t)kv * p + (t - t0)) * row_u4 + c] = val;
                }
            }
            continue;
        }
        // page j completes: assemble (2, p, d) in shared memory from its old rows (ring)
        // and the new input rows, summarise, offload with zero-copy 128-bit stores
        const uint4* old_src = reinterpret_cast<const uint4*>(L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe);
        for (int i = threadIdx.x; i < page_u4; i += blockDim.x) {
            const int kv = i / (p * row_u4), rem = i % (p * row_u4), r = rem / row_u4, c = rem % row_u4;
            const int t = t0 + r;
            uint4 val;
            if (t < L0) {
                val = old_src[i];
            } else {
                const uint16_t* src = (kv == 0 ? k : v) + (((size_t)b * n_new + (t - L0)) * D.n_kv + m) * d;
                val = reinterpret_cast<const uint4*>(src)[c];
            }
            sm[i] = val;
        }
        __syncthreads();
        summarize_smem_page(D, L, u, j, reinterpret_cast<const uint16_t*>(sm));
        uint4* host = reinterpret_cast<uint4*>(L.host + (((size_t)b * D.n_page_host + j) * D.n_kv + m) * pe);
        for (int i = threadIdx.x; i < page_u4; i += blockDim.x) {
            host[i] = sm[i];
            if (dn) dn[i] = sm[i];
            if (dst) {
                const int r = (i % (p * row_u4)) / row_u4;
                if (t0 + r >= L0) dst[i] = sm[i];
            }
        }
        __syncthreads();
    }
}


}  // namespace fkv
