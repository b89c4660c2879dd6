// api.cu -- the C ABI of include/freekv.h: handle, config validation, arena
// layout, stream/event choreography of the per-layer decode step.
//
// Per layer l, step i (SURVEY §8(a) choreography):
//   compute stream:  wait(recall_done[l]) -> append -> score -> finalize
//                    -> recall(sync, flagged units) -> record(select_done[l])
//                    -> attention split -> combine + commit
//   recall stream:   wait(select_done[l]) -> recall(background, unflagged units)
//                    -> record(recall_done[l])
// Background recall of layer l overlaps the rest of step i and the start of
// step i+1 (PAPER.md P:221-225 speculative retrieval; P:320-324 streamed
// recall).  No host synchronisation on the path.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/freekv.h"
#include "fkv_internal.cuh"

using namespace fkv;

static thread_local std::string g_last_error;

namespace fkv {
// once per (kernel, device, size): opt-in dynamic shared memory + max-shared carveout
cudaError_t func_smem(const void* kern, size_t dyn_smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find({kern, dev});
    if (it != done.end() && it->second >= dyn_smem) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess) done[{kern, dev}] = dyn_smem;
    return e;
}
}  // namespace fkv

static freekv_status fail(freekv_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

#define FKV_CUDA(call)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(FREEKV_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)

struct freekv_handle {
    alignas(64) CUtensorMap tmap_kv;  // the device arena as a 2D tensor of 256-byte rows (TMA)
    alignas(64) CUtensorMap tmap_host;  // the device-mapped host pool, same row geometry (direct mode)
    const uint16_t* arena = nullptr;
    freekv_config cfg;
    FkvDims D;
    std::vector<FkvLayer> layers;
    FkvScratch X;
    int device = 0;
    cudaStream_t cs = nullptr, rs = nullptr;
    cudaStream_t ss = nullptr;  // library-owned high-priority stream for the synchronous recall (recall mode)
    std::vector<cudaEvent_t> ev_select, ev_recall, ev_sync, ev_sync_x;
    bool one_graph = false;      // direct mode: recalls are forked branches of the one step graph
    bool spec = false;           // speculative decode step: attention beside the side chain (attn.cu mode 1)
    std::vector<cudaStream_t> side;  // side streams of the speculative step (score -> select -> recall)
    std::vector<cudaEvent_t> ev_pre;  // fork point of each layer's side chain (after its pre kernel)
    int prio_hi = 0;             // kernel priority of the critical path (pre, attention)
    int attn_cluster = 1;        // CTAs per unit of the clustered attention
    int sms = 148;               // SM count of the handle's device
    int graph_p2 = 0;            // the captured step graph's select tree (leaves)
    int graph_ctx_limit = 0;     // ... covers contexts up to this many tokens (re-captured beyond)
    struct {
        int n_virtual = 0, profile = 0;
        const void *q = nullptr, *k = nullptr, *v = nullptr;
        float* out = nullptr;
    } cap;                       // arguments of the last step-graph capture
    int fsel_nc = 1, fsel_lpt = 1;  // the corrected units' select on the critical path (speculative step)
    int bsel_nc = 1, bsel_lpt = 1;  // the other units' select in the side chain (speculative step)
    std::vector<int> ctx_host;
    std::vector<int> recall_pending;
    bool pdl = true;                    // programmatic dependent launch (FREEKV_PDL=0 disables)
    bool serial_recall = false;  // f2 ablation: FREEKV_SERIAL_RECALL=1 runs background recall on the compute stream
    bool no_bg_recall = false;   // measurement only (FREEKV_DEBUG_NO_RECALL=1, read per capture / call): skip the
                                 // background recall -- selections unchanged, the next step's resident pages stale
                                 // (bench.py exposed_recall_us: step time with minus without)
    // profiling (freekv_profile_begin/end)
    bool prof = false;
    uint32_t prof_mask = ~0u;  // kernel classes bracketed by events while profiling
    std::vector<cudaEvent_t> prof_pool;
    size_t prof_used = 0;
    struct Rec { int cls; cudaEvent_t a, b; };
    std::vector<Rec> prof_recs;
    // whole-step graphs (freekv_step_graph_capture / launch)
    bool capturing = false;
    cudaGraphExec_t g_compute = nullptr, g_recall = nullptr;
    std::vector<Rec> graph_recs;  // event pairs captured into the step graph (profile mode)
    std::vector<int> graph_tokens;  // tokens one replay appends to each layer (> 1 with layer cycling)
    // multi-GPU: this rank's NCCL communicator over the kv-head / batch shards and
    // the gathered per-layer output [n_layers][n_ranks][nb][n_qo][d] fp32 (the one exchange step)
    ncclComm_t comm = nullptr;
    int n_ranks = 1, rank = 0;
    float* gather_all = nullptr;
};

namespace {

constexpr size_t kAlign = 256;
constexpr int kMaxAttnWarps = 148 * 16;
size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

struct Sizes {
    size_t layer_bytes, scratch_bytes, dense_bytes, dev_bytes, host_layer_bytes, host_bytes;
    // offsets inside one layer block
    size_t o_summ, o_sink, o_slots, o_ring, o_qprev, o_res_pages, o_res_slot, o_res_front, o_res_valid, o_res_cnt,
        o_pend_cnt,
        o_pend_pages, o_pend_slot, o_pend_front, o_flags, o_cbar, o_fetch_page, o_fetch_slot, o_n_fetch, o_ctx,
        o_n_off, o_qcur, o_scores, o_pend_valid, o_order, o_ord_cnt, o_score_done, o_sync_mask;
    size_t o_part_o, o_part_ml, o_page_rows, o_page_cnt, o_page_valid, o_page_dst, o_ready;
};

freekv_status validate(const freekv_config* c, FkvDims* D) {
    if (!c) return fail(FREEKV_EINVAL, "config is NULL");
    if (c->n_layers <= 0 || c->batch <= 0 || c->n_qo <= 0 || c->n_kv <= 0)
        return fail(FREEKV_EINVAL, "n_layers, batch, n_qo, n_kv must be positive");
    if (c->n_qo % c->n_kv != 0) return fail(FREEKV_EINVAL, "n_qo % n_kv != 0 (GQA group size G = n_qo/n_kv, P:98)");
    if (c->head_dim != kHeadDim) return fail(FREEKV_EUNSUPPORTED, "head_dim must be 128");
    if (!(c->page_size == 16 || c->page_size == 32 || c->page_size == 64))
        return fail(FREEKV_EUNSUPPORTED, "page_size must be 16, 32 or 64");
    const int G = c->n_qo / c->n_kv;
    if (G > kMaxG) return fail(FREEKV_EUNSUPPORTED, "group size G > 8");
    const int p = c->page_size;
    if (c->sink_tokens < 0 || c->window_tokens < 0) return fail(FREEKV_EINVAL, "sink/window must be >= 0");
    if (c->sink_tokens % p) return fail(FREEKV_EINVAL, "sink_tokens % page_size != 0 (reading A-7)");
    if (c->window_tokens % p) return fail(FREEKV_EINVAL, "window_tokens % page_size != 0 (reading A-7)");
    if (c->budget_tokens < c->sink_tokens + c->window_tokens)
        return fail(FREEKV_EINVAL, "budget < sink + window (P:101)");
    if ((c->budget_tokens - c->sink_tokens - c->window_tokens) % p)
        return fail(FREEKV_EINVAL, "(budget - sink - window) % page_size != 0 (K = (B-S-W)/p, reading A-6)");
    const int K = (c->budget_tokens - c->sink_tokens - c->window_tokens) / p;
    if (K < 1 || K > 256) return fail(FREEKV_EUNSUPPORTED, "K = (B-S-W)/p must be in [1, 256]");
    if (c->sink_tokens / p + K + c->window_tokens / p + 2 > 254)
        return fail(FREEKV_EUNSUPPORTED, "attention pages per unit (S/p + K + W/p + 2) must be <= 254");
    if (c->max_ctx_tokens <= 0) return fail(FREEKV_EINVAL, "max_ctx_tokens must be positive");
    const int n_page_host = c->max_ctx_tokens / p + 1;
    if (n_page_host > 8192) return fail(FREEKV_EUNSUPPORTED, "max_ctx_tokens / page_size > 8191 pages");
    if (!(c->mode == 0 || c->mode == 1 || c->mode == 2)) return fail(FREEKV_EINVAL, "mode must be 0, 1 or 2");
    if (!std::isfinite(c->tau)) return fail(FREEKV_EINVAL, "tau must be finite");
    if (!(c->first_layer_dense == 0 || c->first_layer_dense == 1)) return fail(FREEKV_EINVAL, "first_layer_dense must be 0 or 1");
    if ((long long)c->batch * c->n_kv > 4096) return fail(FREEKV_EUNSUPPORTED, "batch * n_kv must be <= 4096");
    if (c->pool < 0 || c->pool > 5) return fail(FREEKV_EINVAL, "pool must be a FREEKV_POOL_* value");
    if (c->corr_pool < 0 || c->corr_pool > 1) return fail(FREEKV_EINVAL, "corr_pool must be 0 or 1");
    FkvDims d{};
    d.nb = c->batch;
    d.n_qo = c->n_qo;
    d.n_kv = c->n_kv;
    d.G = G;
    d.d = kHeadDim;
    d.p = p;
    d.K = K;
    d.n_sink = c->sink_tokens / p;
    d.n_win = c->window_tokens / p;
    d.S_tok = c->sink_tokens;
    d.R_loc = d.n_win + 2;
    d.n_page_host = n_page_host;
    d.n_page_max = (n_page_host + 127) / 128 * 128;
    d.max_ctx = c->max_ctx_tokens;
    d.U = c->batch * c->n_kv;
    d.mode = c->mode;
    d.tau = c->tau;
    d.score_r = (float)(1.4426950408889634074 / std::sqrt((double)kHeadDim));  // CFR-3
    d.attn_c = (float)(1.4426950408889634074 / std::sqrt((double)kHeadDim));
    d.P_max = d.n_sink + K + d.R_loc;
    d.pool = c->pool;
    d.corr_pool = c->corr_pool;
    d.attn_warps = std::min(kMaxAttnWarps, d.U * d.P_max);
    *D = d;
    return FREEKV_OK;
}

Sizes compute_sizes(const freekv_config* c, const FkvDims& D) {
    Sizes s{};
    const size_t U = D.U, K = D.K, pe_b = page_elems(D) * 2;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = o;
        o = align_up(o + bytes);
        return at;
    };
    s.o_summ = take(U * D.n_page_max * 2 * D.d * 2);
    s.o_sink = take(U * D.n_sink * pe_b);
    s.o_slots = take(U * 2 * K * pe_b);
    s.o_ring = take(U * D.R_loc * pe_b);
    s.o_qprev = take((size_t)D.nb * D.n_qo * D.d * 2);
    s.o_res_pages = take(U * K * 4);
    s.o_res_slot = take(U * K * 4);
    s.o_res_front = take(U * 4);
    s.o_res_valid = take(U * 4);
    s.o_res_cnt = take(U * 4);
    s.o_pend_cnt = take(U * 4);
    s.o_pend_pages = take(U * K * 4);
    s.o_pend_slot = take(U * K * 4);
    s.o_pend_front = take(U * 4);
    s.o_flags = take(U);
    s.o_cbar = take(U * 4);
    s.o_fetch_page = take(U * K * 4);
    s.o_fetch_slot = take(U * K * 4);
    s.o_n_fetch = take(U * 4);
    s.o_ctx = take(U * 4);
    s.o_n_off = take(U * 4);
    s.o_qcur = take((size_t)D.nb * D.n_qo * D.d * 2);
    s.o_scores = take(U * D.G * D.n_page_max * 4);
    s.o_pend_valid = take(U * 4);
    s.o_order = take(U * 4);
    s.o_ord_cnt = take(4 * 4);
    s.o_score_done = take(U * 4);
    s.o_sync_mask = take(U);
    s.layer_bytes = o;
    o = 0;
    s.o_part_o = take((size_t)4 * kMaxAttnWarps * D.G * D.d * 4);
    s.o_part_ml = take((size_t)4 * kMaxAttnWarps * D.G * 2 * 4);
    s.o_page_rows = take(U * D.P_max * 4);
    s.o_page_cnt = take(U * 4);
    s.o_page_valid = take(U * D.P_max);
    s.o_page_dst = take(U * D.P_max * 4);
    s.o_ready = take(U * 4);
    s.scratch_bytes = o;
    // first_layer_dense (O-7): layer 0 keeps every page of every unit resident for its dense
    // attention, [U][n_page_max][2][p][d] after the scratch block
    s.dense_bytes = c->first_layer_dense ? align_up(U * D.n_page_max * pe_b) : 0;
    s.dev_bytes = s.layer_bytes * c->n_layers + s.scratch_bytes + s.dense_bytes;
    s.host_layer_bytes = (size_t)D.nb * D.n_page_host * D.n_kv * pe_b;
    s.host_bytes = s.host_layer_bytes * c->n_layers;
    return s;
}

freekv_status check_layer(freekv_handle* h, int layer) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    if (layer < 0 || layer >= h->cfg.n_layers) return fail(FREEKV_EINVAL, "layer out of range");
    return FREEKV_OK;
}

cudaStream_t pick(freekv_handle* h, void* s) { return s ? (cudaStream_t)s : h->cs; }

int max_n_off(const FkvDims& D, int ctx) { return std::max(D.n_sink, ctx / D.p - D.n_win); }

enum { K_APPEND = 0, K_SCORE, K_FINALIZE, K_RECALL_SYNC, K_RECALL_BG, K_ATTN_SPLIT, K_ATTN_COMBINE, K_ATTN_P2, K_PRE };

template <class F>
cudaError_t timed(freekv_handle* h, int cls, cudaStream_t s, F&& launch) {
    if (!h->prof || !((h->prof_mask >> cls) & 1u) || h->prof_used + 2 > h->prof_pool.size()) return launch();
    cudaEvent_t a = h->prof_pool[h->prof_used++], b = h->prof_pool[h->prof_used++];
    // under stream capture only "external" records become real event-record graph nodes
    const unsigned fl = h->capturing ? cudaEventRecordExternal : 0u;
    cudaError_t e = cudaEventRecordWithFlags(a, s, fl);
    if (e == cudaSuccess) e = launch();
    if (e == cudaSuccess) e = cudaEventRecordWithFlags(b, s, fl);
    h->prof_recs.push_back({cls, a, b});
    return e;
}

freekv_status do_append(freekv_handle* h, int layer, const void* k, const void* v, int n_new, cudaStream_t s) {
    if (!k || !v) return fail(FREEKV_EINVAL, "k/v is NULL");
    if (n_new <= 0) return fail(FREEKV_EINVAL, "n_new must be positive");
    if (h->ctx_host[layer] + n_new > h->D.max_ctx)
        return fail(FREEKV_ERANGE, "context would exceed max_ctx_tokens");
    if (h->recall_pending[layer] && !h->capturing) FKV_CUDA(cudaStreamWaitEvent(s, h->ev_recall[layer], 0));
    FKV_CUDA(timed(h, K_APPEND, s, [&] {
        return launch_append(h->D, h->layers[layer], (const uint16_t*)k, (const uint16_t*)v, n_new, s);
    }));
    h->ctx_host[layer] += n_new;
    return FREEKV_OK;
}

// Rows a2-a4 on stream s (primitive API and the serial decode step): page scoring, then the
// select kernel.  flag_src 1: the pre kernel decided the correction flags; list_all: page lists of
// every unit for the attention.
static bool env_on(const char* name) {
    const char* v = getenv(name);
    return v && v[0] == '1';
}

// The select kernel's instance for a CFR-6 tree of P2 leaves (page ids [0, P2), zero-padded; any
// P2 >= next_pow2(n_off) gives the same Z).  CTAs per unit: the widest cluster (<= 4) with one CTA
// per SM and >= 256 leaves per CTA, or one 1024-thread CTA when there are many units; leaves per
// thread fill the tree.  (<= 4: at c3 4- and 8-CTA clusters measure the same, 44.6 / 44.4 us per
// layer; the smaller cluster leaves the attention's clusters more room.)  Returns false above 8192
// leaves.
struct SelCfg {
    int nc, lpt, nt;
};
static bool select_config(const FkvDims& D, int sms, int P2, SelCfg* out) {
    int nc = 4;
    while (nc > 1 && (D.U * nc > sms || nc * 256 > P2)) nc >>= 1;
    // many units (<= 2 CTAs each would fit): one wide 1024-thread CTA per unit instead
    // (A/B on B200 at c2: 42.3 us/layer vs 50.3 with 2-CTA clusters of 256 threads)
    if (nc <= 2 && P2 >= 1024 && P2 / 1024 <= 8) nc = 1;
    const char* ne = getenv("FREEKV_SELECT_NC");  // A/B: force the cluster width (1, 2, 4, 8)
    if (ne && (atoi(ne) == 1 || atoi(ne) == 2 || atoi(ne) == 4 || atoi(ne) == 8)) nc = atoi(ne);
    int lpt = std::max(1, P2 / (nc * 256));
    if (nc > 1 && lpt > 4) {  // cluster instances are built for <= 4 leaves per thread
        nc = 1;
        lpt = P2 / 256;
    }
    if (lpt > 32) return false;
    // one 1024-thread CTA per unit when there are enough units to fill the GPU with clusters of
    // one (the wide CTA's short per-thread chains beat the 256-thread CTA and a 2-CTA cluster at
    // c2); FREEKV_SELECT_NT=256|512|1024 overrides
    const char* nte = getenv("FREEKV_SELECT_NT");
    int nt = (nc == 1 && P2 >= 1024 && P2 / 1024 <= 8) ? 1024 : 256;
    if (nte && (atoi(nte) == 256 || atoi(nte) == 512 || atoi(nte) == 1024)) nt = atoi(nte);
    if (nt > 256 && (nc != 1 || P2 < nt || P2 / nt > 8)) nt = 256;
    if (nt > 256) lpt = P2 / nt;
    *out = SelCfg{nc, lpt, nt};
    return true;
}

// Leaves of the tree for contexts up to ctx tokens
static int tree_leaves(const FkvDims& D, int ctx) {
    const int n_off = std::max(D.n_sink, ctx / D.p - D.n_win);
    int P2 = 256;
    while (P2 < n_off) P2 <<= 1;
    return P2;
}

freekv_status do_select(freekv_handle* h, int layer, const void* q, int32_t* pages_out, uint8_t* corr_out,
                        cudaStream_t s, int flag_src, int list_all, const void* k_new = nullptr,
                        const void* v_new = nullptr) {
    // k_new/v_new given (serial step, W >= 1 page): the score grid also runs the correction check
    // and the append of every unit (its first U CTAs); the token stays pending until the attention
    const int pending = k_new ? 1 : 0;
    if (!q) return fail(FREEKV_EINVAL, "q is NULL");
    if (h->ctx_host[layer] <= 0) return fail(FREEKV_ESTATE, "select before any token was appended");
    // the background recall of the previous step reads this layer's fetch list (one-graph
    // capture: the previous graph launch, which joins its recalls, has completed)
    if (h->capturing && h->one_graph) {
    } else if (h->capturing)
        FKV_CUDA(cudaStreamWaitEvent(s, h->ev_recall[layer], cudaEventWaitExternal));
    else if (h->recall_pending[layer])
        FKV_CUDA(cudaStreamWaitEvent(s, h->ev_recall[layer], 0));
    const int mno = h->capturing ? max_n_off(h->D, h->D.max_ctx) : max_n_off(h->D, h->ctx_host[layer]);
    FkvLayer& L = h->layers[layer];
    const bool scoring = h->capturing || mno - h->D.n_sink > h->D.K;
    if (scoring || pending)
        FKV_CUDA(timed(h, K_SCORE, s, [&] {
            return launch_score(h->D, L, h->X, (const uint16_t*)q, scoring ? mno : 0, pending ? -2 : -1, h->pdl,
                                0, s, (const uint16_t*)k_new, (const uint16_t*)v_new);
        }));
    FKV_CUDA(timed(h, K_FINALIZE, s, [&] {
        // the smallest CFR-6 tree covering this step's candidates (the graph's: its capture's)
        const int P2 = h->capturing ? h->graph_p2 : tree_leaves(h->D, h->ctx_host[layer]);
        SelCfg sc;
        if (!select_config(h->D, h->sms, P2, &sc)) return cudaErrorInvalidValue;
        return launch_select(h->D, L, h->X, (const uint16_t*)q, pages_out, corr_out, flag_src, list_all, -1,
                             sc.nc, sc.lpt, h->pdl, 0, s, pending, sc.nt);
    }));
    return FREEKV_OK;
}

freekv_status do_recall(freekv_handle* h, int layer, cudaStream_t s, const uint8_t* sync_mask = nullptr) {
    const FkvLayer& L = h->layers[layer];
    const uint8_t* mk = nullptr;
    if (sync_mask) {  // the caller's mask, copied on s into the layer's own [U] (the background part reads it later)
        FKV_CUDA(cudaMemcpyAsync(L.sync_mask, sync_mask, h->D.U, cudaMemcpyDeviceToDevice, s));
        mk = L.sync_mask;
    }
    FKV_CUDA(timed(h, K_RECALL_SYNC, s, [&] { return launch_recall(h->D, L, 1, s, nullptr, mk); }));
    if (h->serial_recall) {
        FKV_CUDA(timed(h, K_RECALL_BG, s, [&] { return launch_recall(h->D, L, 0, s, nullptr, mk); }));
        return FREEKV_OK;
    }
    FKV_CUDA(cudaEventRecord(h->ev_select[layer], s));
    FKV_CUDA(cudaStreamWaitEvent(h->rs, h->ev_select[layer], 0));
    FKV_CUDA(timed(h, K_RECALL_BG, h->rs, [&] { return launch_recall(h->D, L, 0, h->rs, nullptr, mk); }));
    FKV_CUDA(cudaEventRecord(h->ev_recall[layer], h->rs));
    h->recall_pending[layer] = 1;
    return FREEKV_OK;
}

// primitive attention: every unit's page list comes from select_pages (mode 0)
freekv_status do_attn(freekv_handle* h, int layer, const void* q, float* out, cudaStream_t s) {
    if (!q || !out) return fail(FREEKV_EINVAL, "q/out is NULL");
    if (h->layers[layer].dense) {  // first_layer_dense: dense attention over [0, Lc)
        FKV_CUDA(timed(h, K_ATTN_SPLIT, s, [&] {
            return launch_attn_cluster(h->D, h->layers[layer], h->X, (const uint16_t*)q, out, h->tmap_kv,
                                       h->tmap_host, 3, h->attn_cluster, false, 0, s);
        }));
        return FREEKV_OK;
    }
    if (h->D.direct) {
        FKV_CUDA(timed(h, K_ATTN_SPLIT, s, [&] {
            return launch_attn_cluster(h->D, h->layers[layer], h->X, (const uint16_t*)q, out, h->tmap_kv, h->tmap_host,
                                       0, h->attn_cluster, false, 0, s);
        }));
        return FREEKV_OK;
    }
    FKV_CUDA(timed(h, K_ATTN_SPLIT, s, [&] {
        return launch_attn_split(h->D, h->layers[layer], h->X, (const uint16_t*)q, 0, h->tmap_kv, h->tmap_host,
                                 h->arena, false, s);
    }));
    FKV_CUDA(timed(h, K_ATTN_COMBINE, s, [&] {
        return launch_attn_combine(h->D, h->layers[layer], h->X, (const uint16_t*)q, out, 0, 0, h->pdl, s);
    }));
    return FREEKV_OK;
}

// Composite step tail (decode_step and the step graph).
//
// Direct mode (default): one attention launch.  Corrected units' fetched pages are read by the
// attention kernel straight from the host pool and written back into their slots, so the
// synchronous recall and a second attention phase leave the critical path; with `mode` 1 the
// units that are not corrected attend their resident set while the select still runs.  The
// background recall (unflagged units, for step i+1) runs on rs, forked after the attention.
//
// Recall mode (FREEKV_CORR=recall, the paper's order): the corrected units' synchronous recall
// runs on the high-priority stream ss while the attention of every other unit (whose pages are
// resident) runs on the compute stream; the corrected units are attended once their pages have
// landed.  The background recall follows the synchronous one.
freekv_status do_step_tail(freekv_handle* h, int layer, const void* q, float* out, int pending = 0) {
    cudaStream_t cs = h->cs;
    const FkvDims& D = h->D;
    FkvLayer& L = h->layers[layer];
    if (D.direct) {
        FKV_CUDA(timed(h, K_ATTN_SPLIT, cs, [&] {
            return launch_attn_cluster(D, L, h->X, (const uint16_t*)q, out, h->tmap_kv, h->tmap_host, 2,
                                       h->attn_cluster, h->pdl, h->prio_hi, cs, pending);
        }));
        // the background recall of this layer starts after its attention (which completes only after
        // the select); it overlaps the next layers
        if (h->serial_recall) {  // f2 ablation: no overlap at all
            FKV_CUDA(timed(h, K_RECALL_BG, cs, [&] { return launch_recall(D, L, 0, cs, h->X.trace); }));
            if (!h->capturing) {
                FKV_CUDA(cudaEventRecord(h->ev_recall[layer], cs));
                h->recall_pending[layer] = 1;
            }
        } else {  // forked branch (graph capture: joined at the graph's end)
            FKV_CUDA(cudaEventRecord(h->ev_select[layer], cs));
            FKV_CUDA(cudaStreamWaitEvent(h->rs, h->ev_select[layer], 0));
            if (!h->no_bg_recall)
                FKV_CUDA(timed(h, K_RECALL_BG, h->rs, [&] { return launch_recall(D, L, 0, h->rs, h->X.trace); }));
            FKV_CUDA(cudaEventRecord(h->ev_recall[layer], h->rs));
            if (!h->capturing) h->recall_pending[layer] = 1;
        }
        return FREEKV_OK;
    }
    FKV_CUDA(cudaEventRecord(h->ev_select[layer], cs));
    FKV_CUDA(cudaStreamWaitEvent(h->ss, h->ev_select[layer], 0));
    FKV_CUDA(timed(h, K_RECALL_SYNC, h->ss, [&] { return launch_recall(D, L, 1, h->ss, h->X.trace); }));
    if (h->capturing)  // external record first: the internal record below joins every ss node back into cs
        FKV_CUDA(cudaEventRecordWithFlags(h->ev_sync_x[layer], h->ss, cudaEventRecordExternal));
    FKV_CUDA(cudaEventRecord(h->ev_sync[layer], h->ss));
    if (h->capturing) {
    } else if (h->serial_recall) {
        FKV_CUDA(timed(h, K_RECALL_BG, h->ss, [&] { return launch_recall(D, L, 0, h->ss); }));
        FKV_CUDA(cudaEventRecord(h->ev_recall[layer], h->ss));
        h->recall_pending[layer] = 1;
    } else {
        FKV_CUDA(cudaStreamWaitEvent(h->rs, h->ev_sync[layer], 0));
        FKV_CUDA(timed(h, K_RECALL_BG, h->rs, [&] { return launch_recall(D, L, 0, h->rs, h->X.trace); }));
        FKV_CUDA(cudaEventRecord(h->ev_recall[layer], h->rs));
        h->recall_pending[layer] = 1;
    }
    FKV_CUDA(timed(h, K_ATTN_SPLIT, cs, [&] {
        return launch_attn_split(D, L, h->X, (const uint16_t*)q, 1, h->tmap_kv, h->tmap_host, h->arena, h->pdl, cs);
    }));
    FKV_CUDA(cudaStreamWaitEvent(cs, h->ev_sync[layer], 0));
    FKV_CUDA(timed(h, K_ATTN_P2, cs, [&] {
        return launch_attn_split(D, L, h->X, (const uint16_t*)q, 2, h->tmap_kv, h->tmap_host, h->arena, false, cs);
    }));
    FKV_CUDA(timed(h, K_ATTN_COMBINE, cs, [&] {
        return launch_attn_combine(D, L, h->X, (const uint16_t*)q, out, 1, 0, h->pdl, cs);
    }));
    return FREEKV_OK;
}

// One layer of the decode step (decode_step and the step graph).  Every mode starts with the pre
// kernel (deferred commit, append, correction flags, new context length) on the compute stream.
//
// Speculative step (default, direct mode), PAPER.md P:221-225 and P:254-258:
//   compute stream: pre -> attention (mode 1: units that are not corrected attend R = S_{i-1} at
//                   once; corrected units wait for their S_i)
//   side stream:    [fork after pre] score -> select (units in priority order, corrected first;
//                   each waits for its own score items) -> background recall of S_i minus R
// The side chain of layer l overlaps the attention of layer l and the following layers; it is
// joined before the same layer's next step (graph end / ev_recall).  With W = 0 the pre kernel's
// append makes the completed page a candidate before the scoring, as the order requires.
//
// Serial step (FREEKV_OVERLAP=0, and the paper-order recall mode FREEKV_CORR=recall): pre ->
// score -> select (every unit's page list) -> attention / recall tail on the compute stream.
freekv_status do_layer_step_core(freekv_handle* h, int layer, const void* q, const void* k_new, const void* v_new,
                            float* out) {
    cudaStream_t cs = h->cs;
    const FkvDims& D = h->D;
    FkvLayer& L = h->layers[layer];
    if (!q || !out) return fail(FREEKV_EINVAL, "q/out is NULL");
    // the previous step's side chain / recall of this layer (its selection, its slots)
    if (!h->capturing && h->recall_pending[layer]) FKV_CUDA(cudaStreamWaitEvent(cs, h->ev_recall[layer], 0));
    if (L.dense) {
        // first_layer_dense (O-7): layer 0 appends its token and attends every page [0, Lc)
        // from its dense pool -- no scoring, selection or recall.  The attention launches without
        // PDL (it reads the context length the append wrote before its prologue).
        FKV_CUDA(timed(h, K_APPEND, cs, [&] {
            return launch_append(D, L, (const uint16_t*)k_new, (const uint16_t*)v_new, 1, cs);
        }));
        if (!h->capturing) h->ctx_host[layer] += 1;
        FKV_CUDA(timed(h, K_ATTN_SPLIT, cs, [&] {
            return launch_attn_cluster(D, L, h->X, (const uint16_t*)q, out, h->tmap_kv, h->tmap_host, 3,
                                       h->attn_cluster, false, h->prio_hi, cs);
        }));
        if (h->capturing) FKV_CUDA(cudaEventRecord(h->ev_recall[layer], cs));  // joined at the graph's end
        return FREEKV_OK;
    }
    if (!h->spec && D.direct && D.n_win >= 1) {
        // serial step, three launches: score grid (+ correction check and append per unit, the token
        // pending) -> select (every unit's page list) -> attention (mode 2; its commit publishes the
        // new context length).  A window of >= 1 page keeps the page the append completes out of
        // this step's candidates, so the append may run beside the scoring.
        if (!h->capturing) h->ctx_host[layer] += 1;
        // page lists only for the corrected units when the others attend R early (they build theirs)
        const int list_all = (D.attn_early && !getenv("FREEKV_LIST_ALL")) ? 0 : 1;
        freekv_status st = do_select(h, layer, q, nullptr, nullptr, cs, 1, list_all, k_new, v_new);
        if (st != FREEKV_OK) return st;
        return do_step_tail(h, layer, q, out, 1);
    }
    FKV_CUDA(timed(h, K_PRE, cs, [&] {
        return launch_pre(D, L, (const uint16_t*)q, (const uint16_t*)k_new, (const uint16_t*)v_new, h->spec ? 1 : 0,
                          h->pdl, h->prio_hi, cs);
    }));
    if (!h->capturing) h->ctx_host[layer] += 1;
    if (!h->spec) {
        freekv_status st = do_select(h, layer, q, nullptr, nullptr, cs, 1, 1);
        if (st != FREEKV_OK) return st;
        return do_step_tail(h, layer, q, out);
    }
    const int mno = h->capturing ? max_n_off(D, D.max_ctx) : max_n_off(D, h->ctx_host[layer]);
    // the corrected units' scoring and selection (latency variants) on the high-priority stream,
    // beside the attention, which waits for them per unit
    FKV_CUDA(cudaEventRecord(h->ev_pre[layer], cs));
    FKV_CUDA(cudaStreamWaitEvent(h->ss, h->ev_pre[layer], 0));
    FKV_CUDA(timed(h, K_SCORE, h->ss, [&] { return launch_score(D, L, h->X, L.q_cur, mno, 0, false, h->prio_hi, h->ss); }));
    FKV_CUDA(timed(h, K_FINALIZE, h->ss, [&] {
        return launch_select(D, L, h->X, L.q_cur, nullptr, nullptr, 1, 0, 0, h->fsel_nc, h->fsel_lpt, h->pdl,
                             h->prio_hi, h->ss);
    }));
    // critical path: the attention of every unit (the others attend R at once)
    FKV_CUDA(timed(h, K_ATTN_SPLIT, cs, [&] {
        return launch_attn_cluster(D, L, h->X, (const uint16_t*)q, out, h->tmap_kv, h->tmap_host, 1, h->attn_cluster,
                                   h->pdl, h->prio_hi, cs);
    }));
    // side chain of the units that are not corrected (their S_i is used at step i+1), after this
    // layer's attention: it overlaps the next layers
    cudaStream_t ss2 = h->side[layer % h->side.size()];
    FKV_CUDA(cudaEventRecord(h->ev_select[layer], cs));
    FKV_CUDA(cudaStreamWaitEvent(ss2, h->ev_select[layer], 0));
    FKV_CUDA(timed(h, K_SCORE, ss2, [&] { return launch_score(D, L, h->X, L.q_cur, mno, 1, false, 0, ss2); }));
    FKV_CUDA(timed(h, K_FINALIZE, ss2, [&] {
        return launch_select(D, L, h->X, L.q_cur, nullptr, nullptr, 1, 0, 1, h->bsel_nc, h->bsel_lpt, h->pdl, 0, ss2);
    }));
    if (h->serial_recall) {  // f2 ablation: the background recall on the compute stream (no overlap)
        FKV_CUDA(cudaEventRecord(h->ev_sync[layer], ss2));
        FKV_CUDA(cudaStreamWaitEvent(cs, h->ev_sync[layer], 0));
        FKV_CUDA(timed(h, K_RECALL_BG, cs, [&] { return launch_recall(D, L, 0, cs, h->X.trace); }));
        FKV_CUDA(cudaEventRecord(h->ev_recall[layer], cs));
    } else {
        FKV_CUDA(timed(h, K_RECALL_BG, ss2, [&] { return launch_recall(D, L, 0, ss2, h->X.trace); }));
        FKV_CUDA(cudaEventRecord(h->ev_recall[layer], ss2));
    }
    if (!h->capturing) h->recall_pending[layer] = 1;
    return FREEKV_OK;
}

// One layer of the decode step, then (multi-GPU) the per-layer all-gather of the head outputs of
// every rank on the compute stream -- inside the step graph when capturing.
freekv_status do_layer_step(freekv_handle* h, int layer, const void* q, const void* k_new, const void* v_new,
                            float* out, int gather_slot = -1) {
    freekv_status st = do_layer_step_core(h, layer, q, k_new, v_new, out);
    if (st != FREEKV_OK || !h->comm || !h->gather_all) return st;
    const size_t count = (size_t)h->D.nb * h->D.n_qo * h->D.d;
    // slice of the gathered output: the layer, or the virtual layer of a cycled step graph
    float* dst = h->gather_all + (size_t)(gather_slot >= 0 ? gather_slot : layer) * h->n_ranks * count;
    const ncclResult_t r = ncclAllGather(out, dst, count, ncclFloat, h->comm, h->cs);
    if (r != ncclSuccess) return fail(FREEKV_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    return FREEKV_OK;
}

freekv_status sync_both(freekv_handle* h) {
    FKV_CUDA(cudaStreamSynchronize(h->cs));
    FKV_CUDA(cudaStreamSynchronize(h->ss));
    FKV_CUDA(cudaStreamSynchronize(h->rs));
    for (cudaStream_t s : h->side) FKV_CUDA(cudaStreamSynchronize(s));
    return FREEKV_OK;
}

}  // namespace

extern "C" {

int32_t freekv_abi_version(void) { return FREEKV_ABI_VERSION; }

const char* freekv_last_error(void) { return g_last_error.c_str(); }

freekv_status freekv_query_sizes(const freekv_config* cfg, size_t* dev_bytes, size_t* host_bytes) {
    FkvDims D;
    freekv_status st = validate(cfg, &D);
    if (st != FREEKV_OK) return st;
    Sizes s = compute_sizes(cfg, D);
    if (dev_bytes) *dev_bytes = s.dev_bytes;
    if (host_bytes) *host_bytes = s.host_bytes;
    return FREEKV_OK;
}

freekv_status freekv_init(const freekv_config* cfg, const freekv_buffers* bufs, void* compute_stream,
                          void* recall_stream, freekv_handle** out) {
    if (!out) return fail(FREEKV_EINVAL, "out is NULL");
    *out = nullptr;
    FkvDims D;
    freekv_status st = validate(cfg, &D);
    if (st != FREEKV_OK) return st;
    if (!bufs || !bufs->dev || !bufs->host) return fail(FREEKV_EINVAL, "buffers are NULL");
    Sizes s = compute_sizes(cfg, D);
    if (bufs->dev_bytes < s.dev_bytes) return fail(FREEKV_ENOMEM, "device arena smaller than freekv_query_sizes()");
    if (bufs->host_bytes < s.host_bytes) return fail(FREEKV_ENOMEM, "host pool smaller than freekv_query_sizes()");
    if ((uintptr_t)bufs->dev % kAlign) return fail(FREEKV_EINVAL, "device arena must be 256-byte aligned");
    if ((uintptr_t)bufs->host % 16) return fail(FREEKV_EINVAL, "host pool must be 16-byte aligned");
    void* host_dev = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&host_dev, bufs->host, 0);
    if (e != cudaSuccess)
        return fail(FREEKV_EINVAL, std::string("host pool is not pinned/device-mapped: ") + cudaGetErrorString(e));

    freekv_handle* h = new freekv_handle();
    cudaGetDevice(&h->device);
    h->cfg = *cfg;
    h->D = D;
    h->cs = (cudaStream_t)compute_stream;
    h->rs = (cudaStream_t)recall_stream;
    if (!h->rs || h->rs == h->cs) {
        delete h;
        return fail(FREEKV_EINVAL, "recall_stream must be a distinct non-NULL stream");
    }
    uint8_t* dev = (uint8_t*)bufs->dev;
    uint8_t* hd = (uint8_t*)host_dev;
    {
        // TMA descriptor: the arena as [rows][128] bf16, box {64 ch, 16 rows}, 128-byte swizzle
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn) {
            delete h;
            return fail(FREEKV_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
        }
        const cuuint64_t dims[2] = {(cuuint64_t)kHeadDim, (cuuint64_t)(s.dev_bytes / (kHeadDim * 2))};
        const cuuint64_t strides[1] = {(cuuint64_t)kHeadDim * 2};
        const cuuint32_t box[2] = {64, 16};
        const cuuint32_t estr[2] = {1, 1};
        CUresult cr = ((PFN_cuTensorMapEncodeTiled)fn)(
            &h->tmap_kv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dev, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) {
            delete h;
            return fail(FREEKV_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
        }
        h->arena = (const uint16_t*)dev;
        // the host pool with the same row geometry: corrected units' fetched pages are read by the
        // attention kernel straight from here (direct mode); needs < 2^31 rows
        const cuuint64_t hrows = (cuuint64_t)(s.host_bytes / (kHeadDim * 2));
        const char* cm = getenv("FREEKV_CORR");
        h->D.direct = (hrows < (1ull << 31) && !(cm && cm[0] == 'r')) ? 1 : 0;
        if (h->D.direct) {
            const cuuint64_t hdims[2] = {(cuuint64_t)kHeadDim, hrows};
            cr = ((PFN_cuTensorMapEncodeTiled)fn)(
                &h->tmap_host, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, host_dev, hdims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) h->D.direct = 0;
        }
        if (!h->D.direct) h->tmap_host = h->tmap_kv;  // never dereferenced for host rows
    }
    h->layers.resize(cfg->n_layers);
    for (int l = 0; l < cfg->n_layers; ++l) {
        uint8_t* base = dev + s.layer_bytes * l;
        FkvLayer& L = h->layers[l];
        L.summ = (uint16_t*)(base + s.o_summ);
        L.sink = (uint16_t*)(base + s.o_sink);
        L.slots = (uint16_t*)(base + s.o_slots);
        L.ring = (uint16_t*)(base + s.o_ring);
        L.q_prev = (uint16_t*)(base + s.o_qprev);
        L.res_pages = (int32_t*)(base + s.o_res_pages);
        L.res_slot = (int32_t*)(base + s.o_res_slot);
        L.res_front = (int32_t*)(base + s.o_res_front);
        L.res_valid = (int32_t*)(base + s.o_res_valid);
        L.res_cnt = (int32_t*)(base + s.o_res_cnt);
        L.pend_cnt = (int32_t*)(base + s.o_pend_cnt);
        L.pend_pages = (int32_t*)(base + s.o_pend_pages);
        L.pend_slot = (int32_t*)(base + s.o_pend_slot);
        L.pend_front = (int32_t*)(base + s.o_pend_front);
        L.flags = (uint8_t*)(base + s.o_flags);
        L.cbar = (float*)(base + s.o_cbar);
        L.fetch_page = (int32_t*)(base + s.o_fetch_page);
        L.fetch_slot = (int32_t*)(base + s.o_fetch_slot);
        L.n_fetch = (int32_t*)(base + s.o_n_fetch);
        L.ctx = (int32_t*)(base + s.o_ctx);
        L.n_off = (int32_t*)(base + s.o_n_off);
        L.q_cur = (uint16_t*)(base + s.o_qcur);
        L.scores = (float*)(base + s.o_scores);
        L.pend_valid = (int32_t*)(base + s.o_pend_valid);
        L.order = (int32_t*)(base + s.o_order);
        L.ord_cnt = (int32_t*)(base + s.o_ord_cnt);
        L.score_done = (int32_t*)(base + s.o_score_done);
        L.sync_mask = (uint8_t*)(base + s.o_sync_mask);
        L.host = (uint16_t*)(hd + s.host_layer_bytes * l);
        L.host_row0 = (int)(s.host_layer_bytes * l / (kHeadDim * 2));
        L.arena = (const uint16_t*)dev;
    }
    if (s.dense_bytes) h->layers[0].dense = (uint16_t*)(dev + s.layer_bytes * cfg->n_layers + s.scratch_bytes);
    uint8_t* sb = dev + s.layer_bytes * cfg->n_layers;
    h->X.part_o = (float*)(sb + s.o_part_o);
    h->X.part_ml = (float*)(sb + s.o_part_ml);
    h->X.page_rows = (int32_t*)(sb + s.o_page_rows);
    h->X.page_cnt = (int32_t*)(sb + s.o_page_cnt);
    h->X.page_valid = (uint8_t*)(sb + s.o_page_valid);
    h->X.page_dst = (int32_t*)(sb + s.o_page_dst);
    h->X.ready = (int32_t*)(sb + s.o_ready);
    h->X.arena = h->layers[0].arena;

    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    {
        // the select's instance is chosen per launch for the tree the current context needs
        // (select_config); here only the largest one (max_ctx) is validated
        const int P2 = tree_leaves(D, D.max_ctx);
        SelCfg sc;
        if (!select_config(D, sms, P2, &sc)) {
            delete h;
            return fail(FREEKV_EUNSUPPORTED, "max_ctx_tokens / page_size > 8192 pages");
        }
        h->sms = sms;
        // speculative step: the corrected units' select (few units, critical path) as wide as the tree
        // allows (<= 8 CTAs, >= 256 leaves each); the side chain's select one CTA per unit (clusters
        // would constrain the placement of the attention's clusters it runs beside)
        int fnc = 8;
        while (fnc > 1 && fnc * 256 > P2) fnc >>= 1;
        h->fsel_nc = fnc;
        h->fsel_lpt = std::max(1, P2 / (fnc * 256));
        if (h->fsel_lpt > 4) {
            h->fsel_nc = 1;
            h->fsel_lpt = P2 / 256;
        }
        h->bsel_nc = 1;
        h->bsel_lpt = P2 / 256;
        const char* fe = getenv("FREEKV_FSELECT_NC");  // A/B of the critical select's width
        if (fe && (atoi(fe) == 1 || atoi(fe) == 2 || atoi(fe) == 4 || atoi(fe) == 8)) {
            h->fsel_nc = atoi(fe);
            h->fsel_lpt = std::max(1, P2 / (h->fsel_nc * 256));
        }
        h->one_graph = h->D.direct;  // recalls are forked branches of the one step graph
        const char* pd = getenv("FREEKV_PDL");
        h->pdl = !(pd && pd[0] == '0');
        // step mode (FREEKV_STEP): serial (default: score grid with the append / correction CTAs,
        // select, attention), spec (the paper's overlap structure: pre kernel, attention beside the
        // scoring / selection side streams; measured slower on B200)
        const char* ov = getenv("FREEKV_STEP");
        const std::string mode = ov ? ov : "serial";
        h->spec = h->D.direct && mode == "spec";
    }
    {
        int warps = 0;
        cudaError_t oe = attn_resident_warps(2, &warps);
        if (oe != cudaSuccess) {
            freekv_destroy(h);
            return fail(FREEKV_ECUDA, std::string("occupancy query: ") + cudaGetErrorString(oe));
        }
        // split kernel (recall mode): T <= V (every warp owns >= 1 page), T * V < 2^31 (32-bit range
        // math), and at most ~254 records per unit (combine kernel capacity)
        const long long V = (long long)D.U * D.P_max;
        long long T = std::min<long long>({(long long)warps, (long long)kMaxAttnWarps, V, 254LL * D.U});
        while (T > 1 && T * V >= (1LL << 31)) T /= 2;
        h->D.attn_warps = (int)std::max(1LL, T);
        h->D.attn_warps_p1 = h->D.attn_warps;
        // clustered attention (direct mode): C CTAs per unit, the largest power of two <= 8 with
        // U * C within one wave of 2 CTAs per SM
        int c = 8;
        while (c > 1 && D.U * c > 2 * sms) c >>= 1;
        const char* ce = getenv("FREEKV_ATTN_CLUSTER");  // A/B: 1, 2, 4, 8 or 16 CTAs per unit
        if (ce && (atoi(ce) == 1 || atoi(ce) == 2 || atoi(ce) == 4 || atoi(ce) == 8 || atoi(ce) == 16)) c = atoi(ce);
        h->attn_cluster = c;
        // slab ring: 2 stages when the attention grid is one CTA per SM or less (its smaller
        // footprint leaves room for the next layer's score CTAs: c3 39.6 vs 40.5 us/layer), else 3
        // (two CTAs per SM: c2 40.0 vs 41.5); FREEKV_ATTN_STAGES overrides
        h->D.attn_nst = getenv("FREEKV_ATTN_STAGES") ? 0 : (D.U * c <= sms ? 2 : 3);
    }
    h->X.trace = nullptr;
    {
        const char* tr = getenv("FREEKV_TRACE");
        if (tr && tr[0] == '1') {
            const size_t n = (size_t)kTraceClasses * kTraceEnt * kTraceStamps;
            if (cudaMalloc(&h->X.trace, n * 8) != cudaSuccess || cudaMemset(h->X.trace, 0, n * 8) != cudaSuccess) {
                freekv_destroy(h);
                return fail(FREEKV_ECUDA, "trace buffer");
            }
        }
        for (auto& L : h->layers) L.trace = h->X.trace;
    }
    {
        const char* fr = getenv("FREEKV_DEBUG_FULL_REFRESH");
        h->D.full_refresh = (fr && fr[0] == '1') ? 1 : 0;
        const char* ae = getenv("FREEKV_ATTN_EARLY");
        h->D.attn_early = ae ? atoi(ae) : 1;
        // score CTAs of 8 warps (1024 pages) when there are many units with few (<= 2048) candidate
        // pages each (A/B on B200, c2: 40.4 vs 41.7 us/layer); with more pages per unit the 4-warp
        // CTAs' larger grid wins (c3 44.0 vs 44.9, c5 145 vs 162); FREEKV_SCORE_WARPS=4|8
        const char* sw = getenv("FREEKV_SCORE_WARPS");
        const int n_off_cap = std::max(h->D.n_sink, h->D.max_ctx / h->D.p - h->D.n_win);
        h->D.score_warps = sw ? (atoi(sw) == 8 ? 8 : 4) : ((h->D.U >= 64 && n_off_cap <= 2048) ? 8 : 4);
        // 4-warp score CTAs: an 8-deep stage ring when the whole scoring grid is resident at once
        // (c3: 128 CTAs, 40.5 vs 44.1 us/layer), else 4 (c5's 1024 CTAs: 146 vs 115.5 -- 128 KiB
        // CTAs leave fewer resident); FREEKV_SCORE_STAGES=4|6|8
        const char* ss = getenv("FREEKV_SCORE_STAGES");
        const long long sc_ctas = (long long)h->D.U * ((n_off_cap + 511) / 512);
        h->D.score_stages = ss ? atoi(ss) : (sc_ctas <= h->sms ? 8 : 4);
    }
    {
        const char* sr = getenv("FREEKV_SERIAL_RECALL");
        h->serial_recall = sr && sr[0] == '1';
    }
    h->ctx_host.assign(cfg->n_layers, 0);
    h->recall_pending.assign(cfg->n_layers, 0);
    h->ev_select.resize(cfg->n_layers);
    h->ev_recall.resize(cfg->n_layers);
    h->ev_sync.resize(cfg->n_layers);
    h->ev_sync_x.resize(cfg->n_layers);
    h->ev_pre.resize(cfg->n_layers);
    {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        h->prio_hi = hi;  // the critical path's kernels outrank the side chains' (graph node priority)
        if (cudaStreamCreateWithPriority(&h->ss, cudaStreamNonBlocking, hi) != cudaSuccess) {
            freekv_destroy(h);
            return fail(FREEKV_ECUDA, "cudaStreamCreateWithPriority failed");
        }
        // side streams of the speculative step (lowest priority), one per layer in rotation so the
        // side chains of consecutive layers may run concurrently
        const char* ns = getenv("FREEKV_SIDE_STREAMS");
        const int n_side = std::max(1, std::min(8, ns ? atoi(ns) : 4));
        for (int i = 0; i < n_side; ++i) {
            cudaStream_t st2;
            if (cudaStreamCreateWithPriority(&st2, cudaStreamNonBlocking, lo) != cudaSuccess) {
                freekv_destroy(h);
                return fail(FREEKV_ECUDA, "cudaStreamCreateWithPriority failed");
            }
            h->side.push_back(st2);
        }
    }
    for (int l = 0; l < cfg->n_layers; ++l) {
        if (cudaEventCreateWithFlags(&h->ev_pre[l], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_select[l], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_recall[l], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_sync[l], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_sync_x[l], cudaEventDisableTiming) != cudaSuccess) {
            freekv_destroy(h);
            return fail(FREEKV_ECUDA, "cudaEventCreate failed");
        }
    }
    e = cudaMemsetAsync(dev, 0, s.dev_bytes, h->cs);
    std::vector<int32_t> n_off(D.U, D.n_sink);
    for (int l = 0; l < cfg->n_layers && e == cudaSuccess; ++l)
        e = cudaMemcpyAsync(h->layers[l].n_off, n_off.data(), D.U * 4, cudaMemcpyHostToDevice, h->cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->cs);
    if (e != cudaSuccess) {
        freekv_destroy(h);
        return fail(FREEKV_ECUDA, std::string("arena init: ") + cudaGetErrorString(e));
    }
    *out = h;
    return FREEKV_OK;
}

freekv_status freekv_append_kv(freekv_handle* h, int32_t layer, const void* k, const void* v, int32_t n_new,
                               void* stream) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    return do_append(h, layer, k, v, n_new, pick(h, stream));
}

freekv_status freekv_summarize_pages(freekv_handle* h, int32_t layer, int32_t page_begin, int32_t page_end,
                                     void* stream) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    const int n_off = max_n_off(h->D, h->ctx_host[layer]);
    if (page_begin < 0 || page_end > n_off || page_begin > page_end)
        return fail(FREEKV_ERANGE, "pages must lie in [0, n_off) (offloaded pages only)");
    FKV_CUDA(launch_summarize(h->D, h->layers[layer], page_begin, page_end, pick(h, stream)));
    return FREEKV_OK;
}

freekv_status freekv_select_pages(freekv_handle* h, int32_t layer, const void* q, int32_t* pages_out,
                                  uint8_t* corrected_out, void* stream) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    return do_select(h, layer, q, pages_out, corrected_out, pick(h, stream), 0, 1);
}

freekv_status freekv_recall_pages(freekv_handle* h, int32_t layer, const uint8_t* sync_mask, void* stream) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    return do_recall(h, layer, pick(h, stream), sync_mask);
}

freekv_status freekv_sparse_decode_attn(freekv_handle* h, int32_t layer, const void* q, float* out, void* stream) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    return do_attn(h, layer, q, out, pick(h, stream));
}

freekv_status freekv_decode_step(freekv_handle* h, int32_t layer, const void* q, const void* k_new,
                                 const void* v_new, float* out) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    if (!k_new || !v_new) return fail(FREEKV_EINVAL, "k_new/v_new is NULL");
    if (h->ctx_host[layer] + 1 > h->D.max_ctx) return fail(FREEKV_ERANGE, "context would exceed max_ctx_tokens");
    h->no_bg_recall = env_on("FREEKV_DEBUG_NO_RECALL");
    return do_layer_step(h, layer, q, k_new, v_new, out);
}


freekv_status freekv_get_selection(freekv_handle* h, int32_t layer, int32_t* pages, int32_t* frontier,
                                   uint8_t* flags, float* cbar) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    if ((st = sync_both(h)) != FREEKV_OK) return st;
    const FkvLayer& L = h->layers[layer];
    const size_t U = h->D.U, K = h->D.K;
    if (pages) FKV_CUDA(cudaMemcpy(pages, L.pend_pages, U * K * 4, cudaMemcpyDeviceToHost));
    if (frontier) FKV_CUDA(cudaMemcpy(frontier, L.pend_front, U * 4, cudaMemcpyDeviceToHost));
    if (flags) FKV_CUDA(cudaMemcpy(flags, L.flags, U, cudaMemcpyDeviceToHost));
    if (cbar) FKV_CUDA(cudaMemcpy(cbar, L.cbar, U * 4, cudaMemcpyDeviceToHost));
    return FREEKV_OK;
}

freekv_status freekv_get_resident(freekv_handle* h, int32_t layer, int32_t* pages, int32_t* frontier) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    if ((st = sync_both(h)) != FREEKV_OK) return st;
    const FkvLayer& L = h->layers[layer];
    const size_t U = h->D.U, K = h->D.K;
    if (pages) FKV_CUDA(cudaMemcpy(pages, L.res_pages, U * K * 4, cudaMemcpyDeviceToHost));
    if (frontier) FKV_CUDA(cudaMemcpy(frontier, L.res_front, U * 4, cudaMemcpyDeviceToHost));
    return FREEKV_OK;
}

freekv_status freekv_get_fetch(freekv_handle* h, int32_t layer, int32_t* n_fetch, int32_t* fetch_pages) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    if ((st = sync_both(h)) != FREEKV_OK) return st;
    const FkvLayer& L = h->layers[layer];
    const size_t U = h->D.U, K = h->D.K;
    if (n_fetch) FKV_CUDA(cudaMemcpy(n_fetch, L.n_fetch, U * 4, cudaMemcpyDeviceToHost));
    if (fetch_pages) FKV_CUDA(cudaMemcpy(fetch_pages, L.fetch_page, U * K * 4, cudaMemcpyDeviceToHost));
    return FREEKV_OK;
}

freekv_status freekv_get_step_stats(freekv_handle* h, int32_t layer, freekv_step_stats* out) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    if (!out) return fail(FREEKV_EINVAL, "out is NULL");
    if ((st = sync_both(h)) != FREEKV_OK) return st;
    const FkvLayer& L = h->layers[layer];
    const size_t U = h->D.U;
    std::vector<uint8_t> fl(U);
    std::vector<int32_t> nf(U);
    FKV_CUDA(cudaMemcpy(fl.data(), L.flags, U, cudaMemcpyDeviceToHost));
    FKV_CUDA(cudaMemcpy(nf.data(), L.n_fetch, U * 4, cudaMemcpyDeviceToHost));
    const int64_t page_bytes = (int64_t)page_elems(h->D) * 2;
    freekv_step_stats s{};
    for (size_t u = 0; u < U; ++u) {
        if (fl[u]) {
            s.corrected_units += 1;
            s.sync_pages += nf[u];
        } else {
            s.bg_pages += nf[u];
        }
    }
    s.sync_bytes = s.sync_pages * page_bytes;
    s.bg_bytes = s.bg_pages * page_bytes;
    *out = s;
    return FREEKV_OK;
}

freekv_status freekv_get_summaries(freekv_handle* h, int32_t layer, int32_t unit, int32_t page_begin,
                                   int32_t page_end, uint16_t* out) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    const FkvDims& D = h->D;
    if (unit < 0 || unit >= D.U || page_begin < 0 || page_end > D.n_page_max || page_begin > page_end || !out)
        return fail(FREEKV_EINVAL, "bad unit/page range/out");
    if ((st = sync_both(h)) != FREEKV_OK) return st;
    const size_t unit_elems = (size_t)D.n_page_max * 2 * D.d;
    std::vector<uint16_t> buf(unit_elems);
    FKV_CUDA(cudaMemcpy(buf.data(), h->layers[layer].summ + unit * unit_elems, unit_elems * 2,
                        cudaMemcpyDeviceToHost));
    for (int j = page_begin; j < page_end; ++j)
        for (int which = 0; which < 2; ++which)
            for (int c = 0; c < D.d; ++c) {
                const size_t off = (((size_t)(c >> 3) * 2 + which) * D.n_page_max + j) * 8 + (c & 7);
                out[((size_t)(j - page_begin) * 2 + which) * D.d + c] = buf[off];
            }
    return FREEKV_OK;
}

freekv_status freekv_get_context(freekv_handle* h, int32_t layer, int32_t* ctx_tokens) {
    freekv_status st = check_layer(h, layer);
    if (st != FREEKV_OK) return st;
    if (ctx_tokens) *ctx_tokens = h->ctx_host[layer];
    return FREEKV_OK;
}

freekv_status freekv_get_dims(freekv_handle* h, int32_t* K, int32_t* n_page_max, int32_t* units) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    if (K) *K = h->D.K;
    if (n_page_max) *n_page_max = h->D.n_page_max;
    if (units) *units = h->D.U;
    return FREEKV_OK;
}

freekv_status freekv_profile_begin(freekv_handle* h, int32_t max_launches) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    if (max_launches <= 0) return fail(FREEKV_EINVAL, "max_launches must be positive");
    while (h->prof_pool.size() < (size_t)max_launches * 2) {
        cudaEvent_t e;
        FKV_CUDA(cudaEventCreate(&e));
        h->prof_pool.push_back(e);
    }
    h->prof_used = 0;
    h->prof_recs.clear();
    h->prof = true;
    return FREEKV_OK;
}

freekv_status freekv_profile_end(freekv_handle* h, float* ms, int32_t* launches) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    h->prof = false;
    freekv_status st = sync_both(h);
    if (st != FREEKV_OK) return st;
    float acc[FREEKV_NUM_KERNEL_CLASSES] = {0};
    int32_t cnt[FREEKV_NUM_KERNEL_CLASSES] = {0};
    for (auto& r : h->prof_recs) {
        float t = 0.0f;
        FKV_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        acc[r.cls] += t;
        cnt[r.cls] += 1;
    }
    for (int i = 0; i < FREEKV_NUM_KERNEL_CLASSES; ++i) {
        if (ms) ms[i] = acc[i];
        if (launches) launches[i] = cnt[i];
    }
    h->prof_recs.clear();
    h->prof_used = 0;
    return FREEKV_OK;
}

freekv_status freekv_synchronize(freekv_handle* h) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    return sync_both(h);
}

freekv_status freekv_debug_trace(freekv_handle* h, uint64_t* out, size_t n) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    if (!h->X.trace) return fail(FREEKV_ESTATE, "tracing is off (set FREEKV_TRACE=1 before freekv_init)");
    freekv_status st = sync_both(h);
    if (st != FREEKV_OK) return st;
    const size_t cap = (size_t)kTraceClasses * kTraceEnt * kTraceStamps;
    FKV_CUDA(cudaMemcpy(out, h->X.trace, std::min(n, cap) * 8, cudaMemcpyDeviceToHost));
    FKV_CUDA(cudaMemset(h->X.trace, 0, cap * 8));
    return FREEKV_OK;
}

static void drop_graphs(freekv_handle* h) {
    if (h->g_compute) cudaGraphExecDestroy(h->g_compute);
    if (h->g_recall) cudaGraphExecDestroy(h->g_recall);
    h->g_compute = h->g_recall = nullptr;
}

freekv_status freekv_step_graph_capture(freekv_handle* h, const void* q_all, const void* k_all, const void* v_all,
                                        float* out_all, int32_t profile) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    return freekv_step_graph_capture_cycle(h, h->cfg.n_layers, q_all, k_all, v_all, out_all, profile);
}

freekv_status freekv_step_graph_capture_cycle(freekv_handle* h, int32_t n_virtual, const void* q_all,
                                              const void* k_all, const void* v_all, float* out_all,
                                              int32_t profile) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    if (n_virtual < h->cfg.n_layers) return fail(FREEKV_EINVAL, "n_virtual < n_layers");
    if (n_virtual != h->cfg.n_layers && (!h->one_graph || h->spec))
        return fail(FREEKV_EUNSUPPORTED, "layer cycling needs the serial direct-mode step");
    {
        // the select tree of the graph: the smallest covering the first replay's contexts; the
        // graph is re-captured (freekv_step_graph_launch) once a context outgrows it
        const int tok = (n_virtual + h->cfg.n_layers - 1) / h->cfg.n_layers;
        int cmax = 0;
        for (int l = 0; l < h->cfg.n_layers; ++l) cmax = std::max(cmax, h->ctx_host[l]);
        h->graph_p2 = tree_leaves(h->D, std::min(h->D.max_ctx, cmax + tok));
        h->graph_ctx_limit = (h->graph_p2 + h->D.n_win + 1) * h->D.p - 1;
        h->cap.n_virtual = n_virtual;
        h->cap.profile = profile;
        h->cap.q = q_all;
        h->cap.k = k_all;
        h->cap.v = v_all;
        h->cap.out = out_all;
    }
    if (!q_all || !k_all || !v_all || !out_all) return fail(FREEKV_EINVAL, "NULL buffer");
    if (h->prof) return fail(FREEKV_ESTATE, "capture while profiling");
    h->no_bg_recall = env_on("FREEKV_DEBUG_NO_RECALL");
    h->graph_recs.clear();
    if (profile) {  // event pool: <= 8 kernels per layer, 2 events each
        freekv_status ps = freekv_profile_begin(h, n_virtual * 8 + 8);
        if (ps != FREEKV_OK) return ps;
        h->prof_mask = profile == 1 ? ~0u : (uint32_t)profile;
    }
    for (int l = 0; l < h->cfg.n_layers; ++l)
        if (h->ctx_host[l] <= 0) return fail(FREEKV_ESTATE, "capture before the first append of every layer");
    freekv_status st = sync_both(h);
    if (st != FREEKV_OK) return st;
    drop_graphs(h);
    const FkvDims& D = h->D;
    const size_t q_stride = (size_t)D.nb * D.n_qo * D.d * 2, kv_stride = (size_t)D.nb * D.n_kv * D.d * 2;
    const size_t o_stride = (size_t)D.nb * D.n_qo * D.d;
    cudaGraph_t gc = nullptr, gr = nullptr;
    h->capturing = true;
    cudaError_t e = cudaStreamBeginCapture(h->cs, cudaStreamCaptureModeThreadLocal);
    for (int vl = 0; vl < n_virtual && e == cudaSuccess && st == FREEKV_OK; ++vl) {
        // virtual layer vl runs instantiated layer vl % n_layers (L_inst cycling for models whose
        // host KV does not fit: SURVEY §7 hard part 9); a layer met again in the same graph first
        // joins its previous background recall (its slots are this occurrence's resident set)
        const int l = vl % h->cfg.n_layers;
        if (vl >= h->cfg.n_layers) e = cudaStreamWaitEvent(h->cs, h->ev_recall[l], 0);
        if (e != cudaSuccess) break;
        if (vl == 0) h->graph_tokens.assign(h->cfg.n_layers, 0);
        h->graph_tokens[l] += 1;
        const uint8_t* q = (const uint8_t*)q_all + q_stride * vl;
        const uint8_t* k = (const uint8_t*)k_all + kv_stride * vl;
        const uint8_t* v = (const uint8_t*)v_all + kv_stride * vl;
        st = do_layer_step(h, l, q, k, v, out_all + o_stride * vl, vl);
    }
    if (h->one_graph) {  // join every layer's recall branch (and the corrected units' chain)
        for (int l = 0; l < h->cfg.n_layers && e == cudaSuccess && st == FREEKV_OK; ++l)
            e = cudaStreamWaitEvent(h->cs, h->ev_recall[l], 0);
        if (h->spec && e == cudaSuccess && st == FREEKV_OK) {
            e = cudaEventRecord(h->ev_sync_x[0], h->ss);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(h->cs, h->ev_sync_x[0], 0);
        }
    }
    cudaError_t e2 = cudaStreamEndCapture(h->cs, &gc);
    if (e == cudaSuccess) e = e2;
    if (e == cudaSuccess && st == FREEKV_OK && !h->one_graph) {
        e = cudaStreamBeginCapture(h->rs, cudaStreamCaptureModeThreadLocal);
        for (int l = 0; l < h->cfg.n_layers && e == cudaSuccess; ++l) {
            // recall mode: after this layer's synchronous recall
            e = cudaStreamWaitEvent(h->rs, h->ev_sync_x[l], cudaEventWaitExternal);
            if (e == cudaSuccess)
                e = timed(h, K_RECALL_BG, h->rs, [&] { return launch_recall(D, h->layers[l], 0, h->rs, h->X.trace); });
            if (e == cudaSuccess) e = cudaEventRecordWithFlags(h->ev_recall[l], h->rs, cudaEventRecordExternal);
        }
        e2 = cudaStreamEndCapture(h->rs, &gr);
        if (e == cudaSuccess) e = e2;
    }
    h->capturing = false;
    if (profile) {
        h->prof = false;
        h->prof_mask = ~0u;
        h->graph_recs = h->prof_recs;
        h->prof_recs.clear();
    }
    // per-node priorities: the critical path's kernels (pre, attention) outrank the side chains'
    if (e == cudaSuccess && st == FREEKV_OK)
        e = cudaGraphInstantiate(&h->g_compute, gc, cudaGraphInstantiateFlagUseNodePriority);
    if (e == cudaSuccess && st == FREEKV_OK && gr) e = cudaGraphInstantiate(&h->g_recall, gr, 0);
    if (gc) cudaGraphDestroy(gc);
    if (gr) cudaGraphDestroy(gr);
    if (st != FREEKV_OK) {
        drop_graphs(h);
        return st;
    }
    if (e != cudaSuccess) {
        drop_graphs(h);
        return fail(FREEKV_ECUDA, std::string("step graph capture: ") + cudaGetErrorString(e));
    }
    return FREEKV_OK;
}

freekv_status freekv_step_graph_profile(freekv_handle* h, float* ms, int32_t* launches) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    if (h->graph_recs.empty()) return fail(FREEKV_ESTATE, "step graph was not captured with profile != 0");
    freekv_status st = sync_both(h);
    if (st != FREEKV_OK) return st;
    float acc[FREEKV_NUM_KERNEL_CLASSES] = {0};
    int32_t cnt[FREEKV_NUM_KERNEL_CLASSES] = {0};
    for (auto& r : h->graph_recs) {
        float t = 0.0f;
        FKV_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        acc[r.cls] += t;
        cnt[r.cls] += 1;
    }
    for (int i = 0; i < FREEKV_NUM_KERNEL_CLASSES; ++i) {
        if (ms) ms[i] = acc[i];
        if (launches) launches[i] = cnt[i];
    }
    return FREEKV_OK;
}

freekv_status freekv_step_graph_launch(freekv_handle* h) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    if (!h->g_compute || (!h->g_recall && !h->one_graph)) return fail(FREEKV_ESTATE, "no captured step graph");
    const auto tok = [&](int l) { return l < (int)h->graph_tokens.size() ? h->graph_tokens[l] : 1; };
    for (int l = 0; l < h->cfg.n_layers; ++l)
        if (h->ctx_host[l] + tok(l) > h->D.max_ctx) return fail(FREEKV_ERANGE, "context would exceed max_ctx_tokens");
    for (int l = 0; l < h->cfg.n_layers; ++l)
        if (h->ctx_host[l] + tok(l) > h->graph_ctx_limit) {  // the select tree must grow: capture again
            const auto c = h->cap;
            freekv_status st = freekv_step_graph_capture_cycle(h, c.n_virtual, c.q, c.k, c.v, c.out, c.profile);
            if (st != FREEKV_OK) return st;
            break;
        }
    FKV_CUDA(cudaGraphLaunch(h->g_compute, h->cs));
    if (h->g_recall) FKV_CUDA(cudaGraphLaunch(h->g_recall, h->rs));
    for (int l = 0; l < h->cfg.n_layers; ++l) {
        h->ctx_host[l] += tok(l);
        // one graph: its recall branches are joined into its end, so the graph's completion
        // on cs stands for them (for callers that later use other streams)
        if (h->one_graph) FKV_CUDA(cudaEventRecord(h->ev_recall[l], h->cs));
        h->recall_pending[l] = 1;
    }
    return FREEKV_OK;
}

freekv_status freekv_comm_unique_id(uint8_t* id_out) {
    if (!id_out) return fail(FREEKV_EINVAL, "id_out is NULL");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(FREEKV_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == FREEKV_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
    return FREEKV_OK;
}

freekv_status freekv_comm_init(freekv_handle* h, const uint8_t* id, int32_t n_ranks, int32_t rank) {
    if (!h || !id) return fail(FREEKV_EINVAL, "handle/id is NULL");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(FREEKV_EINVAL, "bad n_ranks / rank");
    if (h->comm) return fail(FREEKV_ESTATE, "communicator already initialised");
    FKV_CUDA(cudaSetDevice(h->device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    const ncclResult_t r = ncclCommInitRank(&c, n_ranks, uid, rank);
    if (r != ncclSuccess) return fail(FREEKV_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    h->comm = c;
    h->n_ranks = n_ranks;
    h->rank = rank;
    drop_graphs(h);  // a captured step graph has no all-gather nodes
    return FREEKV_OK;
}

freekv_status freekv_set_gather_output(freekv_handle* h, float* gather_all) {
    if (!h) return fail(FREEKV_EINVAL, "handle is NULL");
    if (gather_all && !h->comm) return fail(FREEKV_ESTATE, "freekv_comm_init first");
    h->gather_all = gather_all;
    drop_graphs(h);
    return FREEKV_OK;
}

void freekv_destroy(freekv_handle* h) {
    if (!h) return;
    cudaStreamSynchronize(h->cs);
    if (h->ss) cudaStreamSynchronize(h->ss);
    cudaStreamSynchronize(h->rs);
    drop_graphs(h);
    for (auto e : h->ev_select)
        if (e) cudaEventDestroy(e);
    for (auto e : h->ev_recall)
        if (e) cudaEventDestroy(e);
    for (auto e : h->ev_sync)
        if (e) cudaEventDestroy(e);
    for (auto e : h->ev_sync_x)
        if (e) cudaEventDestroy(e);
    for (auto e : h->ev_pre)
        if (e) cudaEventDestroy(e);
    for (auto e : h->prof_pool) cudaEventDestroy(e);
    for (cudaStream_t s2 : h->side) {
        cudaStreamSynchronize(s2);
        cudaStreamDestroy(s2);
    }
    if (h->ss) cudaStreamDestroy(h->ss);
    if (h->X.trace) cudaFree(h->X.trace);
    if (h->comm) ncclCommDestroy(h->comm);
    delete h;
}

}  // extern "C"
