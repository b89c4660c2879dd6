// append.cu -- row a9 kernels: bulk/standalone append (append_unit per CTA) and
// the summary rebuild from the host pool.  See append_unit.cuh.
#include "append_unit.cuh"

namespace fkv {

__global__ void __launch_bounds__(256) fkv_append_kernel(FkvDims D, FkvLayer L, const uint16_t* __restrict__ k,
                                                         const uint16_t* __restrict__ v, int n_new) {
    extern __shared__ uint4 sm[];  // one page (2, p, d) bf16
    const int u = blockIdx.x;
    const int L0 = L.ctx[u];
    append_unit(D, L, u, L0, k, v, n_new, sm);
    if (threadIdx.x == 0) {
        const int L1 = L0 + n_new;
        L.ctx[u] = L1;
        L.n_off[u] = max(L.n_off[u], frontier_for(D, L1));
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
    cudaError_t e = func_smem((const void*)fkv_append_kernel, smem);
    if (e != cudaSuccess) return e;
    fkv_append_kernel<<<D.U, 256, smem, s>>>(D, L, k, v, n_new);
    return cudaGetLastError();
}

cudaError_t launch_summarize(const FkvDims& D, const FkvLayer& L, int page_begin, int page_end, cudaStream_t s) {
    if (page_end <= page_begin) return cudaSuccess;
    const size_t smem = (size_t)D.p * D.d * sizeof(uint16_t);
    cudaError_t e = func_smem((const void*)fkv_summarize_kernel, smem);
    if (e != cudaSuccess) return e;
    fkv_summarize_kernel<<<dim3(D.U, page_end - page_begin), 128, smem, s>>>(D, L, page_begin);
    return cudaGetLastError();
}

}  // namespace fkv
