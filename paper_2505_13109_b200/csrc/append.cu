// append.cu -- row a9: append new tokens, build page summaries, offload pages
// leaving the window to the pinned host pool ("the NHD-HND
// transpose is only required when offloading a KV page", P:231 summaries).
//
// One CTA per unit (b, kv head).  Pages touched by the new tokens or crossing
// the frontier n_off = max(S/p, floor(Lc/p) - W/p) are processed in ascending
// order: the page is assembled in shared memory as (2, p, d) from the local
// ring (old tokens) and the NHD input (new tokens); a crossing page gets its
// channel-wise min/max summary and is stored as one 16 KiB page into the host
// pool with zero-copy 128-bit stores; new tokens are written to the sink area
// or the local ring.  Sequential page order inside one CTA makes ring reuse
// (page j and j + R_loc share a slot) race-free.
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
            uint16_t kk = sort_key(ks[r * D.d + c]);
            lo = kk < lo ? kk : lo;
            hi = kk > hi ? kk : hi;
        }
        L.summ[summ_chunk_offset(D, u, j, c >> 3, 0) + (c & 7)] = from_key(lo);
        L.summ[summ_chunk_offset(D, u, j, c >> 3, 1) + (c & 7)] = from_key(hi);
    }
}

__global__ void __launch_bounds__(256) fkv_append_kernel(FkvDims D, FkvLayer L, const uint16_t* __restrict__ k,
                                                         const uint16_t* __restrict__ v, int n_new) {
    extern __shared__ uint4 sm[];  // one page (2, p, d) bf16
    const int u = blockIdx.x, b = u / D.n_kv, m = u % D.n_kv;
    const int p = D.p, d = D.d, row_u4 = d / 8, page_u4 = 2 * p * row_u4;
    const int L0 = L.ctx[u];
    const int L1 = L0 + n_new;
    const int old_off = L.n_off[u];
    const int new_off = max(D.n_sink, L1 / p - D.n_win);
    const int n_last = (L1 - 1) / p;
    const int ring_lo = max(D.n_sink, n_last - D.R_loc + 1);
    const int jA = min(L0 / p, old_off);
    const size_t pe = page_elems(D);
    for (int j = jA; j <= n_last; ++j) {
        const bool touched = (j + 1) * p > L0;
        const bool crossing = j >= old_off && j < new_off;
        if (!touched && !crossing) continue;
        const int t0 = j * p;
        if (!crossing) {
            // fast path (every decode step): copy the new token rows straight to their page
            uint4* dst = nullptr;
            if (j < D.n_sink)
                dst = reinterpret_cast<uint4*>(L.sink + ((size_t)u * D.n_sink + j) * pe);
            else if (j >= ring_lo)
                dst = reinterpret_cast<uint4*>(L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe);
            if (dst) {
                const int ta = max(t0, L0), tb = min(t0 + p, L1);
                const int n_u4 = (tb - ta) * row_u4;
                for (int i = threadIdx.x; i < 2 * n_u4; i += blockDim.x) {
                    const int kv = i / n_u4, rem = i % n_u4, r = rem / row_u4, c = rem % row_u4;
                    const int t = ta + r;
                    const uint16_t* src = (kv == 0 ? k : v) + (((size_t)b * n_new + (t - L0)) * D.n_kv + m) * d;
                    dst[((size_t)kv * p + (t - t0)) * row_u4 + c] = reinterpret_cast<const uint4*>(src)[c];
                }
            }
            continue;  // no __syncthreads needed: distinct pages never alias within this branch
        }
        const uint4* old_src =
            j < D.n_sink ? reinterpret_cast<const uint4*>(L.sink + ((size_t)u * D.n_sink + j) * pe)
                         : reinterpret_cast<const uint4*>(L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe);
        for (int i = threadIdx.x; i < page_u4; i += blockDim.x) {
            const int kv = i / (p * row_u4), rem = i % (p * row_u4), r = rem / row_u4, c = rem % row_u4;
            const int t = t0 + r;
            uint4 val = make_uint4(0u, 0u, 0u, 0u);
            if (t < L0) {
                val = old_src[i];
            } else if (t < L1) {
                const uint16_t* src = (kv == 0 ? k : v) + (((size_t)b * n_new + (t - L0)) * D.n_kv + m) * d;
                val = reinterpret_cast<const uint4*>(src)[c];
            }
            sm[i] = val;
        }
        __syncthreads();
        if (crossing) {
            summarize_smem_page(D, L, u, j, reinterpret_cast<const uint16_t*>(sm));
            uint4* dst = reinterpret_cast<uint4*>(L.host + (((size_t)b * D.n_page_host + j) * D.n_kv + m) * pe);
            for (int i = threadIdx.x; i < page_u4; i += blockDim.x) dst[i] = sm[i];
        }
        if (touched) {
            uint4* dst = nullptr;
            if (j < D.n_sink)
                dst = reinterpret_cast<uint4*>(L.sink + ((size_t)u * D.n_sink + j) * pe);
            else if (j >= ring_lo)
                dst = reinterpret_cast<uint4*>(L.ring + ((size_t)u * D.R_loc + (j % D.R_loc)) * pe);
            if (dst)
                for (int i = threadIdx.x; i < page_u4; i += blockDim.x) {
                    const int r = (i % (p * row_u4)) / row_u4;
                    const int t = t0 + r;
                    if (t >= L0 && t < L1) dst[i] = sm[i];
                }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        L.ctx[u] = L1;
        L.n_off[u] = max(old_off, new_off);
        if (n_new > 1) L.res_valid[u] = 0;  // reading R-9: bulk append restarts speculation
    }
}

// Rebuild summaries of pages [pb, pe) from the host pool (zero-copy reads).
__global__ void __launch_bounds__(128) fkv_summarize_kernel(FkvDims D, FkvLayer L, int pb) {
    extern __shared__ uint4 sm[];
    const int u = blockIdx.x, j = pb + blockIdx.y;
    const int b = u / D.n_kv, m = u % D.n_kv;
    const size_t pe = page_elems(D);
    const uint4* src = reinterpret_cast<const uint4*>(L.host + (((size_t)b * D.n_page_host + j) * D.n_kv + m) * pe);
    const int k_u4 = D.p * D.d / 8;
    for (int i = threadIdx.x; i < k_u4; i += blockDim.x) sm[i] = src[i];
    __syncthreads();
    summarize_smem_page(D, L, u, j, reinterpret_cast<const uint16_t*>(sm));
}

cudaError_t launch_append(const FkvDims& D, const FkvLayer& L, const uint16_t* k, const uint16_t* v,
                          int n_new, cudaStream_t s) {
    const size_t smem = page_elems(D) * sizeof(uint16_t);
    fkv_append_kernel<<<D.U, 256, smem, s>>>(D, L, k, v, n_new);
    return cudaGetLastError();
}

cudaError_t launch_summarize(const FkvDims& D, const FkvLayer& L, int page_begin, int page_end, cudaStream_t s) {
    if (page_end <= page_begin) return cudaSuccess;
    const size_t smem = (size_t)D.p * D.d * sizeof(uint16_t);
    fkv_summarize_kernel<<<dim3(D.U, page_end - page_begin), 128, smem, s>>>(D, L, page_begin);
    return cudaGetLastError();
}

}  // namespace fkv
