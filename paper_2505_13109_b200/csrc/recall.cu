// recall.cu -- rows a5/a6: recall of selected pages from the pinned host pool.
//
// the host pool is (n_page, n_kv, 2, p, d), so one (page, KV
// head) is 2*p*d contiguous elements (16 KiB at p=32, d=128) and one transfer
// moves a whole page.  P:255-256: corrected units are recalled before this
// step's attention, the others in the background for reuse at step i+1.
//
// B200 design: the fetch list is produced on the GPU by the
// select kernel, so the copy is a kernel: each fetched page moves from the
// device-mapped pinned host pool into its free cache slot with TMA bulk copies
// (slot double-buffering: the slot is not read by any attention until the next
// commit).  Synchronous mode runs on the
// compute stream for flagged units; background mode runs on the dedicated
// recall stream for the others.
#include <algorithm>
#include <cstdlib>

#include "fkv_internal.cuh"

namespace fkv {

// The fetch lists of the units of this mode (sync: corrected units, background: the
// others) are concatenated: every CTA loads all units' counts in one batch, builds the
// exclusive prefix in shared memory, and then strides over the fetched pages only (one
// 16 KiB page per CTA iteration, 16 KiB of PCIe reads in flight per CTA).  Measured on
// B200: zero-copy read bandwidth scales with the number of SMs issuing, while a grid of
// thousands of CTAs (one per pair) crowds the block scheduler and delays the attention
// kernels running concurrently -- so by default one CTA per SM (FREEKV_RECALL_{SYNC,BG}_CTAS).
constexpr int kRecallThreads = 128;
constexpr int kRecallMaxU = 4096;

__global__ void __launch_bounds__(kRecallThreads) fkv_recall_kernel(FkvDims D, FkvLayer L, int sync_mode,
                                                                    unsigned long long* __restrict__ trace,
                                                                    int frag, const uint8_t* __restrict__ mask) {
    __shared__ int s_off[kRecallMaxU + 1];  // exclusive prefix of the eligible units' fetch counts
    __shared__ int s_wsum[kRecallThreads / 32];
    if (threadIdx.x == 0) trace_stamp(trace, 2 + (sync_mode ? 0 : 1), blockIdx.x, 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // counts: thread t owns units [t * per, (t + 1) * per), loads issued together
    const int per = (D.U + kRecallThreads - 1) / kRecallThreads;
    int local = 0;
    for (int i = 0; i < per; ++i) {
        const int u = tid * per + i;
        int n = 0;
        if (u < D.U) {
            // which units are synchronous: the correction flags, or the caller's sync_mask
            const int f = mask ? mask[u] : L.flags[u], nf = L.n_fetch[u];
            n = ((f != 0) == (sync_mode != 0)) ? nf : 0;
        }
        s_off[u < D.U ? u : D.U] = n;  // temporarily the count
        local += n;
    }
    // block exclusive scan of the per-thread totals
    int x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp; ++w) base += s_wsum[w];
    int run = base + x - local;
    for (int i = 0; i < per; ++i) {
        const int u = tid * per + i;
        if (u < D.U) {
            const int n = s_off[u];
            s_off[u] = run;
            run += n;
        }
    }
    __syncthreads();
    if (tid == kRecallThreads - 1) s_off[D.U] = run;  // total (the last thread's running sum)
    __syncthreads();
    const int total = s_off[D.U];
    const size_t pe = page_elems(D);
    // one elected thread moves each page with two bulk copies through shared memory (host pool ->
    // smem over the link, smem -> slot in HBM): the TMA engine carries the PCIe reads, not the SM's
    // load/store pipeline
    extern __shared__ __align__(128) uint8_t s_page[];
    __shared__ __align__(8) uint64_t bar;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        uint32_t ph = 0;
        const uint32_t bytes = (uint32_t)(pe * sizeof(uint16_t));
        for (int f = blockIdx.x; f < total; f += gridDim.x) {
            int lo = 0, hi = D.U - 1;  // unit of the f-th fetched page: the last u with s_off[u] <= f
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_off[mid] <= f) lo = mid;
                else hi = mid - 1;
            }
            const int u = lo, k = f - s_off[u];
            const int b = u / D.n_kv, m = u % D.n_kv;
            const int j = L.fetch_page[(size_t)u * D.K + k];
            const int slot = L.fetch_slot[(size_t)u * D.K + k];
            const uint16_t* src = L.host + (((size_t)b * D.n_page_host + j) * D.n_kv + m) * pe;
            uint16_t* dst = L.slots + ((size_t)u * 2 * D.K + slot) * pe;
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // s_page free again
            mbar_expect_tx(&bar, bytes);
            if (frag > 0 && frag < (int)bytes) {  // ablation (f2): many small transfers per page
                for (uint32_t off = 0; off < bytes; off += (uint32_t)frag)
                    bulk_g2s(s_page + off, reinterpret_cast<const uint8_t*>(src) + off, (uint32_t)frag, &bar);
            } else {
                bulk_g2s(s_page, src, bytes, &bar);
            }
            mbar_wait(&bar, ph);
            ph ^= 1u;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(s_page)),
                         "r"(bytes)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    if (threadIdx.x == 0) trace_stamp(trace, 2 + (sync_mode ? 0 : 1), blockIdx.x, 1);
}

static int recall_ctas(int sync_mode) {
    static int c[2] = {0, 0};
    if (!c[sync_mode]) {
        const char* e = getenv(sync_mode ? "FREEKV_RECALL_SYNC_CTAS" : "FREEKV_RECALL_BG_CTAS");
        const int v = e ? atoi(e) : 0;
        // defaults: synchronous recall one CTA per SM (it is on the critical path); background
        // recall 16 CTAs -- fewer outstanding host reads measurably disturb the HBM-bound kernels
        // of the next layers less, and the link is never the bottleneck of this path
        c[sync_mode] = v > 0 ? v : (sync_mode ? 148 : 16);
    }
    return c[sync_mode];
}

cudaError_t launch_recall(const FkvDims& D, const FkvLayer& L, int sync_mode, cudaStream_t s,
                          unsigned long long* trace, const uint8_t* mask) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int want = recall_ctas(sync_mode ? 1 : 0);
    const int grid = std::min(want == 148 ? sms : want, D.U * D.K);
    const size_t smem = page_elems(D) * sizeof(uint16_t);
    cudaError_t e = func_smem((const void*)fkv_recall_kernel, smem);
    if (e != cudaSuccess) return e;
    // FREEKV_RECALL_FRAG=<bytes> (ablation): move each page as <bytes>-sized
    // transfers, e.g. 256 = one (token, head) row of an NHD host layout, instead of one 16 KiB page
    static int frag = -1;
    if (frag < 0) {
        const char* fe = getenv("FREEKV_RECALL_FRAG");
        int v = fe ? std::max(0, atoi(fe)) : 0;
        frag = (v % 16) ? 0 : v;  // bulk copies move multiples of 16 bytes
    }
    fkv_recall_kernel<<<grid, kRecallThreads, smem, s>>>(D, L, sync_mode, trace, frag, mask);
    return cudaGetLastError();
}

}  // namespace fkv
