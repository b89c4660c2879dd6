// recall.cu -- rows a5/a6: recall of selected pages from the pinned host pool.
//
// the host pool is (n_page, n_kv, 2, p, d), so one (page, KV
// head) is 2*p*d contiguous elements (16 KiB at p=32, d=128) and one transfer
// moves a whole page.  P:255-256: corrected units are recalled before this
// step's attention, the others in the background for reuse at step i+1.
//
// B200 design: the fetch list is produced on the GPU by the
// select kernel, so the copy is a zero-copy gather: one CTA per fetched page
// reads the device-mapped pinned host page over PCIe with 128-bit loads and
// writes it into its free cache slot (slot double-buffering: the slot is not
// read by any attention until the next commit).  Synchronous mode runs on the
// compute stream for flagged units; background mode runs on the dedicated
// recall stream for the others.
#include <algorithm>
#include <cstdlib>

#include "fkv_internal.cuh"

namespace fkv {

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// The grid strides over the flattened (unit, fetch) pairs with 16 KiB of PCIe
// reads in flight per CTA.  Measured on B200: zero-copy read bandwidth scales
// with the number of SMs issuing (8 CTAs reach ~4 GB/s; one CTA per SM reaches
// the host link), while a grid of thousands of CTAs (one per pair) crowds the
// block scheduler and delays the attention kernels running concurrently -- so by
// default one CTA per SM (FREEKV_RECALL_{SYNC,BG}_CTAS overrides).
__global__ void __launch_bounds__(128) fkv_recall_kernel(FkvDims D, FkvLayer L, int sync_mode,
                                                         unsigned long long* __restrict__ trace) {
    if (threadIdx.x == 0) trace_stamp(trace, 2 + (sync_mode ? 0 : 1), blockIdx.x, 0);
    const size_t pe = page_elems(D);
    const int n = (int)(pe / 8);  // uint4 per page
    for (int pair = blockIdx.x; pair < D.U * D.K; pair += gridDim.x) {
        const int u = pair / D.K, f = pair % D.K;
        if ((L.flags[u] != 0) != (sync_mode != 0)) continue;
        if (f >= L.n_fetch[u]) continue;
        const int b = u / D.n_kv, m = u % D.n_kv;
        const int j = L.fetch_page[(size_t)u * D.K + f];
        const int slot = L.fetch_slot[(size_t)u * D.K + f];
        const uint4* src =
            reinterpret_cast<const uint4*>(L.host + (((size_t)b * D.n_page_host + j) * D.n_kv + m) * pe);
        uint4* dst = reinterpret_cast<uint4*>(L.slots + ((size_t)u * 2 * D.K + slot) * pe);
        for (int base = 0; base < n; base += 8 * 128) {
            uint4 r[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int idx = base + i * 128 + threadIdx.x;
                if (idx < n) r[i] = ld_stream(src + idx);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int idx = base + i * 128 + threadIdx.x;
                if (idx < n) dst[idx] = r[i];
            }
        }
    }
    if (threadIdx.x == 0) trace_stamp(trace, 2 + (sync_mode ? 0 : 1), blockIdx.x, 1);
}

static int recall_ctas(int sync_mode) {
    static int c[2] = {0, 0};
    if (!c[sync_mode]) {
        const char* e = getenv(sync_mode ? "FREEKV_RECALL_SYNC_CTAS" : "FREEKV_RECALL_BG_CTAS");
        const int v = e ? atoi(e) : 0;
        c[sync_mode] = v > 0 ? v : 148;  // default: one CTA per SM (zero-copy bandwidth scales with SMs)
    }
    return c[sync_mode];
}

cudaError_t launch_recall(const FkvDims& D, const FkvLayer& L, int sync_mode, cudaStream_t s,
                          unsigned long long* trace) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(fkv_recall_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        configured = true;
    }
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int want = recall_ctas(sync_mode ? 1 : 0);
    const int grid = std::min(want == 148 ? sms : want, D.U * D.K);
    fkv_recall_kernel<<<grid, 128, 0, s>>>(D, L, sync_mode, trace);
    return cudaGetLastError();
}

}  // namespace fkv
