// fkv_internal.cuh -- shared definitions of the CUDA path (NOT shared with oracle/).
//
// Layout of one layer's state in the device arena and the host pool
// (DESIGN.md §4).  All kernels receive a FkvDims and a FkvLayer by value.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace fkv {

constexpr int kHeadDim = 128;   // d (P:557 models: 128)
constexpr int kMaxG = 8;        // GQA group size supported (Llama 4, Qwen 7, 70B 8)
// pages scored by one score CTA (score.cu): the throughput variant (4 pages per thread) of the
// serial step and the side chain, and the latency variant (1 page per thread, 4x more CTAs) that
// scores the corrected units on the critical path
#ifndef FKV_SC_WARPS
#define FKV_SC_WARPS 4  // warps per score CTA (A/B builds: -DFKV_SC_WARPS=2)
#endif
constexpr int kScoreCtaPages = FKV_SC_WARPS * 128;
constexpr int kScoreCtaPagesFast = FKV_SC_WARPS * 32;

struct FkvDims {
    int nb, n_qo, n_kv, G, d, p;
    int K;            // selectable pages per unit
    int n_sink;       // sink pages (S/p)
    int n_win;        // window pages (W/p)
    int S_tok;        // sink tokens
    int R_loc;        // local ring pages = n_win + 2
    int n_page_max;   // device page capacity per unit (multiple of 128; summaries, scores)
    int n_page_host;  // host pool pages per sequence (max_ctx/p + 1)
    int max_ctx;
    int U;            // nb * n_kv
    int mode;
    int full_refresh; // diagnostics (env FREEKV_DEBUG_FULL_REFRESH=1): no slot reuse, all pages re-fetched
    int attn_early;   // serial step: uncorrected units attend before the wait for the select (FREEKV_ATTN_EARLY)
    int score_warps;  // warps per score CTA (parts -1/-2): 4 or 8 (1024 pages per CTA)
    int score_stages; // ring depth per warp of the 4-warp score CTAs (parts -1/-2): 4, 6 or 8
    int attn_nst;     // slab stages per warp of the clustered attention (2 or 3; 0 = env / default 3)
    int pool;         // FREEKV_POOL_* group pooling of the selection (f3); 0 = MeanS
    int corr_pool;    // 0 = mean of the cosines, 1 = corrected when the least similar head is below tau
    float tau;
    float score_r;    // CFR-3: fl32(log2(e)/sqrt(d))
    float attn_c;     // log2(e)/sqrt(d) for attention softmax (not CFR)
    int P_max;        // upper bound of attention pages per unit: n_sink + K + R_loc
    int attn_warps;   // T: warps of the balanced split-KV attention grid (<= resident warps)
    int attn_warps_p1;  // T of attention phase 1 (recall mode: units attending R)
    int direct;       // 1: corrected units' fetched pages are read by the attention kernel straight
                      // from the host pool (and written back to their slots); 0: synchronous recall
                      // before a second attention phase
};

struct FkvLayer {
    uint16_t* summ;       // [U][d/8][2][n_page_max][8]: channel group c8, {min, max}, page, 8 channels
    uint16_t* sink;       // [U][n_sink][2][p][d]
    uint16_t* slots;      // [U][2K][2][p][d]
    uint16_t* ring;       // [U][R_loc][2][p][d]
    uint16_t* q_prev;     // [nb][n_qo][d]
    int32_t* res_pages;   // [U][K]  resident selection R (ascending, -1 pad)
    int32_t* res_slot;    // [U][K]
    int32_t* res_front;   // [U]     frontier f_R of R
    int32_t* res_valid;   // [U]     0 until the first commit (bootstrap, A-12)
    int32_t* res_cnt;     // [U]     number of valid entries of res_pages
    int32_t* pend_cnt;    // [U]     number of valid entries of pend_pages
    int32_t* pend_pages;  // [U][K]  pending S_i
    int32_t* pend_slot;   // [U][K]
    int32_t* pend_front;  // [U]
    uint8_t* flags;       // [U]     correction flags of this step
    float* cbar;          // [U]
    int32_t* fetch_page;  // [U][K]  S_i \ R, ascending
    int32_t* fetch_slot;  // [U][K]
    int32_t* n_fetch;     // [U]
    int32_t* ctx;         // [U]     context length Lc (tokens)
    int32_t* n_off;       // [U]     pages [0, n_off) are offloaded; candidates [n_sink, n_off)
    uint16_t* q_cur;      // [nb][n_qo][d] this step's q, copied by the pre kernel (read by the side chain)
    float* scores;        // [U][G][n_page_max] page scores of this step (CFR-3 base-2 logits)
    int32_t* pend_valid;  // [U]     1: pend_* holds a selection not yet committed to R
    int32_t* order;       // [U]     units in scoring/selection priority order (corrected units first)
    int32_t* ord_cnt;     // [2][2]  per step parity (ctx & 1): fill counters of `order` (corrected from the
                          //         front, the others from the back)
    uint8_t* sync_mask;   // [U]     freekv_recall_pages' sync_mask, copied (read by the background part)
    int32_t* score_done;  // [U]     score items of the unit finished this step (release/acquire hand-off)
    unsigned long long* trace;  // diagnostics (FREEKV_TRACE=1): %globaltimer stamps, else NULL
    uint16_t* host;       // device-mapped host pool of this layer: [nb][n_page_host][n_kv][2][p][d]
    const uint16_t* arena;  // base of the device arena (row 0 of the attention TMA tensor)
    uint16_t* dense;      // first_layer_dense, layer 0 only: [U][n_page_max][2][p][d] every page resident
                          // (dense attention); NULL otherwise
    int host_row0;        // first row of this layer's host pool in the host TMA tensor (256-byte rows)
};

struct FkvScratch {
    int32_t* page_rows;   // [U][P_max] attention page list of this step: arena row of the page's K block
    uint8_t* page_valid;  // [U][P_max] valid tokens of each listed page; bit 7: the row is a host
                          // pool row (direct mode), to be written back to arena row page_dst
    int32_t* page_dst;    // [U][P_max] arena row of the slot a host-read page is written back to
    unsigned long long* trace;  // diagnostics (FREEKV_TRACE=1): %globaltimer stamps, else NULL
    int32_t* page_cnt;    // [U]
    float* part_o;        // [2 phases][attn_warps][2 segments][G][d] per-warp, per-unit-segment partial outputs
    float* part_ml;       // [2 phases][attn_warps][2 segments][G][2] (running max, running sum)
    float* cosv;          // [U][kMaxG] per-head correction cosines from the score kernel
    const uint16_t* arena;  // base of the device arena (row 0 of the attention TMA tensor)
    int32_t* ready;       // [U] 1 once the select kernel has published unit u's selection (S_i, pend_*,
                          // fetch list, corrected units' page list); reset by the attention's commit
};

__host__ __device__ inline size_t page_elems(const FkvDims& D) { return (size_t)2 * D.p * D.d; }

// summary element offset (in uint16) of the 8 channels [8 c8, 8 c8 + 8) of page j, which (0 = min,
// 1 = max).  Channel-group-major: the c8 slice of consecutive pages is contiguous, so a scoring
// warp streams {8 channels x 128 pages} as two 2 KiB bulk copies and lane l reads page l with
// conflict-free 16-byte shared loads.
__host__ __device__ __forceinline__ size_t summ_off(const FkvDims& D, int u, int c8, int which, int j) {
    return ((((size_t)u * (kHeadDim / 8) + c8) * 2 + which) * D.n_page_max + j) * 8;
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ float bf16f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream
// serialization may start while its predecessor drains; it runs its prologue, then
// waits for the predecessor's completion (and memory) at pdl_wait().
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// trace slots: [kernel class 0..11][entity < 4096][stamp < 8]
constexpr int kTraceClasses = 12;
constexpr int kTraceEnt = 4096, kTraceStamps = 8;
__device__ __forceinline__ void trace_stamp(unsigned long long* tr, int cls, int ent, int i) {
    if (tr && ent < kTraceEnt) tr[((size_t)cls * kTraceEnt + ent) * kTraceStamps + i] = gtimer();
}

// ---- TMA bulk copy (cp.async.bulk, SASS UBLKCP) + mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Warp-wide max of a float (exact, order-free): one redux.sync (sm_100a)
__device__ __forceinline__ float warp_max_f32(float v) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}

// CFR-10 for one head: sequential fp32 channel sums of x*y, x*x and y*y over d = 128
// bf16 channels (fma = exact product + one rounding), then dot / (sqrt(n1) * sqrt(n2)),
// 0 when either norm is 0.  All 2 x 256 bytes are loaded first (16-byte vectors), so the
// chain runs from registers.
__device__ __forceinline__ float cos_cfr10(const uint16_t* qa, const uint16_t* qb) {
    uint4 va[16], vb[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        va[i] = reinterpret_cast<const uint4*>(qa)[i];
        vb[i] = reinterpret_cast<const uint4*>(qb)[i];
    }
    float dot = 0.0f, n1 = 0.0f, n2 = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const uint32_t wa[4] = {va[i].x, va[i].y, va[i].z, va[i].w};
        const uint32_t wb[4] = {vb[i].x, vb[i].y, vb[i].z, vb[i].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // channel 8i + 2k + h: low half first
                const float x = h ? bf16_hi(wa[k]) : bf16_lo(wa[k]);
                const float y = h ? bf16_hi(wb[k]) : bf16_lo(wb[k]);
                dot = __fmaf_rn(x, y, dot);
                n1 = __fmaf_rn(x, x, n1);
                n2 = __fmaf_rn(y, y, n2);
            }
        }
    }
    return (n1 == 0.0f || n2 == 0.0f) ? 0.0f : __fdiv_rn(dot, __fmul_rn(__fsqrt_rn(n1), __fsqrt_rn(n2)));
}

// Group pooling of the heads' cosines (CFR-10): 0 = mean (sequential sum / G, FreeKV);
// 1 = minimum, the "max pooling over group C_i" of tab:abl-g-corr (reading R-11)
__device__ __forceinline__ float pool_cos(const float* c, int G, int corr_pool) {
    float acc = c[0];
    for (int g = 1; g < G; ++g) acc = corr_pool ? (c[g] < acc ? c[g] : acc) : __fadd_rn(acc, c[g]);
    return corr_pool ? acc : __fdiv_rn(acc, (float)G);
}

// Correction decision of one unit (readings A-12, A-13): step 0 (no resident set) is
// always corrected; ALWAYS / tau >= 1 always, NEVER / tau <= 0 never; else pooled cosine < tau.
__device__ __forceinline__ int correction_flag(const FkvDims& D, float pooled, int res_valid) {
    int flag;
    if (D.mode == 1 || D.tau >= 1.0f) flag = 1;
    else if (D.mode == 2 || D.tau <= 0.0f) flag = 0;
    else flag = pooled < D.tau;
    return res_valid ? flag : 1;
}

// Unit at index i of a part of the speculative step (-1 if none): part 0 = the corrected units
// L.order[0, n0), part 1 = the others L.order[n0, U); the counters of this step's parity (ctx & 1,
// the batch shares one context length) were filled by the pre kernel.  part < 0: unit i.
// end of the candidate range [n_sink, n_off) once the context holds ctx tokens
__device__ __forceinline__ int frontier_for(const FkvDims& D, int ctx) { return max(D.n_sink, ctx / D.p - D.n_win); }

__device__ __forceinline__ int part_unit(const FkvDims& D, const FkvLayer& L, int part, int i) {
    if (part < 0) return i;
    const int n0 = L.ord_cnt[(L.ctx[0] & 1) * 2];
    const int base = part == 0 ? 0 : n0, n = part == 0 ? n0 : D.U - n0;
    return i < n ? L.order[base + i] : -1;
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Spin until *p >= v (acquire).  Bounded: a hand-off that never comes (a bug) traps -- the launch
// fails with an error instead of hanging the GPU (~4 s at 64 ns per poll).
__device__ __forceinline__ void spin_until_ge(const int32_t* p, int v) {
    for (long long i = 0; ld_acquire(p) < v; ++i) {
        if (i > (1ll << 26)) __trap();
        __nanosleep(64);
    }
}

__device__ __forceinline__ void st_release(int32_t* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Kernel attribute set-up, once per (kernel, device): dynamic shared memory opt-in and the
// max-shared carveout (every kernel of the path prefers it, so consecutive kernels never force
// an L1/shared reconfiguration).  Thread-safe; defined in api.cu.
cudaError_t func_smem(const void* kern, size_t dyn_smem);

// prio: 0 = the stream's, else a CUDA priority value (kernel-node priority inside captured graphs)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                             int prio, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
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
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace fkv

// kernel launchers (defined in the .cu files), return the launch status
namespace fkv {
cudaError_t launch_append(const FkvDims& D, const FkvLayer& L, const uint16_t* k, const uint16_t* v,
                          int n_new, cudaStream_t s);
cudaError_t launch_summarize(const FkvDims& D, const FkvLayer& L, int page_begin, int page_end,
                             cudaStream_t s);
// decode-step prologue of one layer (one CTA per unit): deferred commit R := pend, q_cur := q,
// correction flag (CFR-10), append of this step's token, ctx / n_off publish; ordered: also the
// order of the units (corrected first) that the two parts of the speculative step use
cudaError_t launch_pre(const FkvDims& D, const FkvLayer& L, const uint16_t* q, const uint16_t* k_new,
                       const uint16_t* v_new, int ordered, bool pdl, int prio, cudaStream_t s);
// page scoring.  part -1: every unit; -2: every unit plus one CTA per unit for the correction check
// and the append of k_new/v_new (serial step, the token pending); 0: the corrected units (latency
// variant, critical path); 1: the others (throughput variant, side chain); parts 0/1 count
// finished items per unit
cudaError_t launch_score(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                         int max_n_off, int part, bool pdl, int prio, cudaStream_t s,
                         const uint16_t* k_new = nullptr, const uint16_t* v_new = nullptr);
// softmax + pooling + top-K + delta (nc CTAs per unit, lpt leaves per thread); flag_src 1: flags from
// the score kernel; list_all: attention page lists of every unit (else of the corrected ones)
// part as for the score kernel; parts 0/1 wait per unit for its score items (no PDL wait).
// pending: this step's token was appended by the score grid but not yet published (serial step)
cudaError_t launch_select(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                          int32_t* pages_out, uint8_t* corrected_out, int flag_src, int list_all, int part,
                          int nc, int lpt, bool pdl, int prio, cudaStream_t s, int pending = 0, int nt = 256);
// mask (device [U], nullable): the units recalled synchronously (sync_mode 1) / not (0) instead of
// the correction flags (freekv_recall_pages' sync_mask)
cudaError_t launch_recall(const FkvDims& D, const FkvLayer& L, int sync_mode, cudaStream_t s,
                          unsigned long long* trace = nullptr, const uint8_t* mask = nullptr);
cudaError_t attn_resident_warps(int cps, int* warps);  // warps of the split kernel's grid (cps CTAs per SM)
cudaError_t launch_attn_split(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                              int phase, const CUtensorMap& tmap, const CUtensorMap& tmap_host,
                              const uint16_t* arena, bool pdl, cudaStream_t s);
// mode 0: page lists of every unit from the select kernel (waits for it), commits every unit;
// mode 1: speculative decode step (FREEKV_STEP=spec); mode 2: serial decode step (see attn.cu)
cudaError_t launch_attn_cluster(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                float* out, const CUtensorMap& tmap, const CUtensorMap& tmap_h, int mode, int c,
                                bool pdl, int prio, cudaStream_t s, int pending = 0);
cudaError_t launch_attn_combine(const FkvDims& D, const FkvLayer& L, const FkvScratch& X, const uint16_t* q,
                                float* out, int split, int commit, bool pdl, cudaStream_t s);
}  // namespace fkv
