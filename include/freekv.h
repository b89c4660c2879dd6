/*
 * freekv.h -- C ABI of the B200-native FreeKV decode-step KV-retrieval path
 * (arXiv 2505.13109).  C99-compatible; no CUDA or torch types in signatures.
 *
 * Notation (§2.1): nb batch rows, n_qo attention heads,
 * n_kv KV heads, G = n_qo / n_kv, d head dim, p page size, budget B
 * tokens with S sink and W window tokens kept, K = (B - S - W) / p selectable
 * pages per unit (reading A-6).  A "unit" is one (batch row, KV head)
 * pair, u = b * n_kv + m; all per-unit arrays are u-major.
 *
 * Memory: the caller owns all large memory.  `dev` is one device allocation
 * (e.g. a torch.uint8 CUDA tensor) of freekv_query_sizes()->dev_bytes; `host`
 * is one pinned, device-mapped host allocation (torch pin_memory tensor /
 * cudaHostAlloc) of host_bytes -- the CPU KV pool of P:297 in the combined
 * HND layout (n_page, n_kv, 2, p, d) of P:318.  Both must outlive the handle.
 * Streams are cudaStream_t passed as void*; NULL selects the handle's compute
 * stream.  All bf16 tensors are raw 16-bit patterns.
 *
 * Errors: every call returns FREEKV_OK (0) or a negative status; the message
 * of the last failure on the calling thread is freekv_last_error().  Calls are
 * asynchronous and stream-ordered; asynchronous CUDA faults surface as
 * FREEKV_ECUDA on a later call or freekv_synchronize().  No call allocates
 * device memory after freekv_init and none blocks the host except the
 * freekv_get_* inspection calls and freekv_synchronize.
 */
#ifndef FREEKV_H
#define FREEKV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FREEKV_ABI_VERSION 3

typedef int32_t freekv_status;
enum {
    FREEKV_OK = 0,
    FREEKV_EINVAL = -1,        /* invalid argument / violated config invariant */
    FREEKV_ENOMEM = -2,        /* buffer smaller than freekv_query_sizes() */
    FREEKV_ECUDA = -3,         /* CUDA runtime error (possibly from earlier async work) */
    FREEKV_ENCCL = -4,         /* NCCL (communicator / collective) failure */
    FREEKV_ESTATE = -5,        /* call out of order / handle in wrong state */
    FREEKV_ERANGE = -6,        /* context would exceed max_ctx_tokens */
    FREEKV_EUNSUPPORTED = -7   /* head_dim != 128, page_size not in {16,32,64}, G > 8, batch*n_kv > 4096 */
};

/* Correction modes, P:661-665 (Table tab:abl-tau): tau = 0 "No Correction",
 * tau = 1 "No Speculation".  SPECULATIVE flags a unit iff mean_g C < tau
 * (P:247-250), with tau <= 0 never and tau >= 1 always (reading A-13). */
enum { FREEKV_MODE_SPECULATIVE = 0, FREEKV_MODE_ALWAYS_CORRECT = 1, FREEKV_MODE_NEVER_CORRECT = 2 };

typedef struct freekv_config {
    int32_t n_layers;        /* layers served by this handle */
    int32_t batch;           /* nb: batch rows on this GPU */
    int32_t n_qo, n_kv;      /* heads on this GPU; G = n_qo / n_kv <= 8 */
    int32_t head_dim;        /* d, must be 128 */
    int32_t page_size;       /* p in {16, 32, 64} (P:557 uses 32) */
    int32_t budget_tokens;   /* B */
    int32_t sink_tokens;     /* S, multiple of p (A-7) */
    int32_t window_tokens;   /* W, multiple of p (A-7) */
    int32_t max_ctx_tokens;  /* capacity of the host pool per sequence */
    float tau;               /* correction threshold */
    int32_t mode;            /* FREEKV_MODE_* */
    int32_t first_layer_dense; /* 1: layer 0 is not compressed (O-7): every page stays resident
                                  in a dense device pool and its attention (decode_step,
                                  sparse_decode_attn) covers all Lc tokens; no selection or recall */
    /* multi-GPU shard description; informational in ABI v1 */
    int32_t kv_head_begin, kv_head_end, batch_begin, batch_end;
    int32_t n_ranks, rank;
    /* ABI v2 -- group-consistency variants:
     * pool: FREEKV_POOL_* how the G heads of a group agree on one selection (FreeKV: MeanS);
     * corr_pool: 0 = mean of the heads' cosines < tau (FreeKV), 1 = "max pooling":
     * corrected when the least similar head is below tau (reading R-11). */
    int32_t pool;
    int32_t corr_pool;
} freekv_config;

#define FREEKV_POOL_MEAN_S 0  /* mean of per-head softmax weights (FreeKV) */
#define FREEKV_POOL_MAX_S 1   /* max of per-head softmax weights */
#define FREEKV_POOL_MEAN_QK 2 /* mean of per-head page scores, one softmax */
#define FREEKV_POOL_MAX_QK 3  /* max of per-head page scores, one softmax */
#define FREEKV_POOL_MEAN_Q 4  /* mean query vector of the group, scored once */
#define FREEKV_POOL_MAX_Q 5   /* element-wise max query vector, scored once */

typedef struct freekv_buffers {
    void* dev;          /* device arena, >= dev_bytes, 256-byte aligned */
    size_t dev_bytes;
    void* host;         /* pinned, device-mapped host pool, >= host_bytes, 4 KiB aligned */
    size_t host_bytes;
} freekv_buffers;

typedef struct freekv_handle freekv_handle;

/* Sizes of the two caller-owned buffers for `cfg`.  Validates cfg. */
freekv_status freekv_query_sizes(const freekv_config* cfg, size_t* dev_bytes, size_t* host_bytes);

/* Create a handle over caller buffers.  compute_stream: stream of decode_step;
 * recall_stream: dedicated stream for background recall.  Zeroes
 * the device arena (stream-ordered on compute_stream). */
freekv_status freekv_init(const freekv_config* cfg, const freekv_buffers* bufs,
                          void* compute_stream, void* recall_stream, freekv_handle** out);

/* O-1 / row a9: append n_new tokens to every sequence of `layer`.
 * k, v: device bf16 [nb][n_new][n_kv][d] (NHD, the natural projection layout,
 * P:304-305).  Writes sink/local device pages; every page that leaves the
 * window (page < n_off = max(S/p, floor(Lc/p) - W/p)) gets its channel-wise
 * min/max summary and is stored to the host pool as one (2,p,d) page
 * (the NHD->HND transpose at offload).  n_new > 1 (prefill) restarts
 * speculation (reading R-9).  ERANGE if the context would exceed max_ctx. */
freekv_status freekv_append_kv(freekv_handle* h, int32_t layer, const void* k, const void* v,
                               int32_t n_new, void* stream);

/* Rebuild the summaries of pages [page_begin, page_end) of every unit of
 * `layer` from the host pool.  Pages must already be offloaded. */
freekv_status freekv_summarize_pages(freekv_handle* h, int32_t layer, int32_t page_begin,
                                     int32_t page_end, void* stream);

/* Rows a1-a4: correction flags (vs the stored q_{i-1}) and the
 * selection S_i with q_i for every unit: page scores (Quest bound,
 * P:231), per-head softmax + MeanS group pooling, top-K with
 * lowest-id ties, delta vs the resident set.  The result is pending:
 * it changes neither the resident set nor q_prev.
 * q: device bf16 [nb][n_qo][d].  pages_out (nullable): device int32
 * [nb][n_kv][K], ascending, -1 padded.  corrected_out (nullable): device
 * uint8 [nb][n_kv]. */
freekv_status freekv_select_pages(freekv_handle* h, int32_t layer, const void* q,
                                  int32_t* pages_out, uint8_t* corrected_out, void* stream);

/* Rows a5/a6: recall the pending selection's missing pages (S_i minus
 * resident, reading A-18) from the host pool into free cache slots.  Units
 * whose correction flag is set are recalled synchronously on `stream` (before
 * attention); the others are recalled in the background on the recall
 * stream for use at the next step.  sync_mask (device uint8
 * [nb][n_kv], nullable): the units to recall synchronously instead of the
 * correction flags (copied on `stream`; the caller's buffer may be reused at
 * once).  In direct mode (default) any mask gives the same results -- a
 * corrected unit's attention reads its missing pages from the host pool if
 * they are not resident yet; in the paper-order recall mode (FREEKV_CORR=recall)
 * the mask must include every corrected unit. */
freekv_status freekv_recall_pages(freekv_handle* h, int32_t layer, const uint8_t* sync_mask,
                                  void* stream);

/* Row a7 + a8: sparse decode attention: for each q head of unit u
 * o = softmax(q K_T^T / sqrt(d)) V_T over T = sink tokens U pages U local
 * region (reading A-9), with pages = S_i for corrected units and the resident
 * set otherwise.  out: device fp32 [nb][n_qo][d].  Then commits
 * the speculative advance: resident := S_i, q_prev := q. */
freekv_status freekv_sparse_decode_attn(freekv_handle* h, int32_t layer, const void* q, float* out,
                                        void* stream);

/* The composite decode step of one layer on the compute stream:
 * append_kv(1 token) -> select_pages -> recall_pages -> sparse_decode_attn.
 * q: [nb][n_qo][d], k_new/v_new: [nb][1][n_kv][d] bf16; out: fp32 [nb][n_qo][d]. */
freekv_status freekv_decode_step(freekv_handle* h, int32_t layer, const void* q, const void* k_new,
                                 const void* v_new, float* out);

/* Whole-step CUDA graphs: capture one decode step of every layer (the same
 * sequence as n_layers freekv_decode_step calls) with fixed device buffers
 * q_all [n_layers][nb][n_qo][d], k_all / v_all [n_layers][nb][1][n_kv][d]
 * (bf16) and out_all [n_layers][nb][n_qo][d] (fp32).  In direct mode (default)
 * each layer's background recall is a forked branch of the one step graph,
 * joined at its end; in recall mode (FREEKV_CORR=recall) the compute-stream part
 * and the background-recall part are two graphs joined by external event nodes
 * (recall of layer l waits for its synchronous recall; step i+1's layer l waits
 * for step i's recall of layer l).  Kernel arguments read all step-varying state
 * from device memory, so one capture replays for every later step.
 * step_graph_launch replays one step on the handle's streams (ERANGE when the
 * context would exceed max_ctx_tokens).
 * profile: 0 = none; 1 = an event-record node pair around every kernel node;
 * otherwise a bit mask (bit c = kernel class c, see freekv_profile_end) of the
 * classes to bracket -- fewer event nodes disturb the step less. */
freekv_status freekv_step_graph_capture(freekv_handle* h, const void* q_all, const void* k_all,
                                        const void* v_all, float* out_all, int32_t profile);
/* Replay the captured step on the compute stream (each layer appends one token; with layer
 * cycling n_virtual / n_layers tokens).  The select's CFR-6 tree in the graph is the smallest
 * covering the contexts at capture; a replay whose contexts outgrow it first re-captures the
 * graph with the same buffers (once per power of two of pages).  ERANGE past max_ctx_tokens. */
freekv_status freekv_step_graph_launch(freekv_handle* h);
/* The same with n_virtual >= n_layers virtual layers: virtual layer v runs layer v % n_layers
 * with q_all / k_all / v_all / out_all slices v (buffers sized for n_virtual) -- L_inst
 * cycling, so an 80-layer model's step is timed with a handle of L_inst instantiated layers
 * whose host KV fits (SURVEY §7 hard part 9).  Each instantiated layer then appends
 * n_virtual / n_layers tokens per step. */
freekv_status freekv_step_graph_capture_cycle(freekv_handle* h, int32_t n_virtual, const void* q_all,
                                              const void* k_all, const void* v_all, float* out_all,
                                              int32_t profile);
/* With profile != 0 at capture, the selected kernel nodes are bracketed by event-record
 * nodes; after a replay has completed, this returns per kernel class the summed
 * device milliseconds and launch counts of that replay (classes as in
 * freekv_profile_end).  Blocking. */
freekv_status freekv_step_graph_profile(freekv_handle* h, float* ms /*[11]*/, int32_t* launches /*[11]*/);

/* Inspection (blocking; host outputs).  All arrays u-major. */
freekv_status freekv_get_selection(freekv_handle* h, int32_t layer, int32_t* pages /*[U][K]*/,
                                   int32_t* frontier /*[U]*/, uint8_t* flags /*[U]*/, float* cbar /*[U]*/);
freekv_status freekv_get_resident(freekv_handle* h, int32_t layer, int32_t* pages /*[U][K]*/,
                                  int32_t* frontier /*[U]*/);
freekv_status freekv_get_fetch(freekv_handle* h, int32_t layer, int32_t* n_fetch /*[U]*/,
                               int32_t* fetch_pages /*[U][K]*/);
/* Summaries of pages [page_begin, page_end) of unit u as [n][2][d] bf16 (min, max). */
/* Recall accounting of the last step (or select_pages) of `layer` (blocking): units
 * corrected this step, the pages their synchronous path fetches (in direct mode read by the
 * attention from the host pool), the pages the background recall moves for the others, and
 * the bytes of each (page = 2 * p * d bf16). */
typedef struct {
    int32_t corrected_units, sync_pages, bg_pages;
    int64_t sync_bytes, bg_bytes;
} freekv_step_stats;
freekv_status freekv_get_step_stats(freekv_handle* h, int32_t layer, freekv_step_stats* out);
freekv_status freekv_get_summaries(freekv_handle* h, int32_t layer, int32_t unit, int32_t page_begin,
                                   int32_t page_end, uint16_t* out);
freekv_status freekv_get_context(freekv_handle* h, int32_t layer, int32_t* ctx_tokens);
/* Numbers a caller needs to size its own tensors. */
freekv_status freekv_get_dims(freekv_handle* h, int32_t* K, int32_t* n_page_max, int32_t* units);

/* Per-kernel device timing for roofline reporting: while profiling is on,
 * every kernel launch of the handle is bracketed by CUDA events on the stream
 * it is launched on (at most max_launches launches are recorded).
 * profile_end synchronises and returns, per kernel class, the summed device
 * milliseconds and the launch count.  Classes: 0 append, 1 score, 2 select
 * finalize, 3 synchronous recall, 4 background recall, 5 attention split (all
 * units, or phase 1: units with resident pages), 6 attention combine + commit,
 * 7 attention split phase 2 (corrected units), 8 step prologue (pipelined step:
 * append + correction check + page lists), 9 background score, 10 background
 * select (pipelined step). */
#define FREEKV_NUM_KERNEL_CLASSES 11
freekv_status freekv_profile_begin(freekv_handle* h, int32_t max_launches);
freekv_status freekv_profile_end(freekv_handle* h, float* ms /*[11]*/, int32_t* launches /*[11]*/);

/* Diagnostics: with FREEKV_TRACE=1 in the environment at freekv_init, kernels write
 * %globaltimer stamps [class 12][entity 4096][stamp 8] (ns); this copies n <= 393216
 * of them to host memory `out` and clears the buffer.  Blocking. */
freekv_status freekv_debug_trace(freekv_handle* h, uint64_t* out, size_t n);

/* Wait for all work of the handle (both streams); surfaces async errors. */
freekv_status freekv_synchronize(freekv_handle* h);
void freekv_destroy(freekv_handle* h);
const char* freekv_last_error(void);
int32_t freekv_abi_version(void);

/* ---- multi-GPU: one process per GPU, each handle
 * configured with its kv-head / batch shard.  The units never interact; the
 * one exchange step is gathering every rank's head outputs per layer.
 *
 * freekv_comm_unique_id: rank 0 creates the NCCL id (FREEKV_COMM_ID_BYTES
 * bytes, host) and the caller broadcasts it (e.g. over torch.distributed).
 * freekv_comm_init: every rank builds the communicator on its handle's device
 * (blocking, collective over n_ranks).  freekv_set_gather_output: device fp32
 * [n_layers (n_virtual for a cycled step graph)][n_ranks][nb][n_qo][d]
 * (caller-owned, NULL to stop): every
 * decode step of layer l then ends with an all-gather of `out` into slice l
 * on the compute stream -- a node of the step graph when captured.  Both
 * invalidate a captured step graph (capture again).  ENCCL on NCCL errors. */
#define FREEKV_COMM_ID_BYTES 128
freekv_status freekv_comm_unique_id(uint8_t* id_out);
freekv_status freekv_comm_init(freekv_handle* h, const uint8_t* id, int32_t n_ranks, int32_t rank);
freekv_status freekv_set_gather_output(freekv_handle* h, float* gather_all);

#ifdef __cplusplus
}
#endif
#endif /* FREEKV_H */
