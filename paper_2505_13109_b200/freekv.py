"""ctypes binding of include/freekv.h (argument marshalling only).

Every step of the path runs in ``libfreekv.so``; this module only allocates the
caller-owned buffers with PyTorch (device arena, pinned host pool, streams)
and forwards pointers.  There is no CPU fallback: a missing library or a
missing GPU raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, fields

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfreekv.so")
# A/B measurements only: FREEKV_LIB_SUFFIX=_X loads libfreekv_X.so from the same directory
if os.environ.get("FREEKV_LIB_SUFFIX"):
    LIB_PATH = LIB_PATH.replace("libfreekv.so", "libfreekv" + os.environ["FREEKV_LIB_SUFFIX"] + ".so")

MODE_SPECULATIVE, MODE_ALWAYS_CORRECT, MODE_NEVER_CORRECT = 0, 1, 2

EXPORTED = [
    "freekv_query_sizes", "freekv_init", "freekv_append_kv", "freekv_summarize_pages",
    "freekv_select_pages", "freekv_recall_pages", "freekv_sparse_decode_attn", "freekv_decode_step",
    "freekv_get_selection", "freekv_get_resident", "freekv_get_fetch", "freekv_get_summaries",
    "freekv_get_context", "freekv_get_dims", "freekv_synchronize", "freekv_destroy",
    "freekv_last_error", "freekv_abi_version", "freekv_profile_begin", "freekv_profile_end",
    "freekv_step_graph_capture", "freekv_step_graph_launch", "freekv_step_graph_profile", "freekv_debug_trace",
    "freekv_get_step_stats", "freekv_step_graph_capture_cycle", "freekv_comm_unique_id", "freekv_comm_init", "freekv_set_gather_output",
]
KERNEL_CLASSES = ["append", "score", "select_finalize", "recall_sync", "recall_bg", "attn_split", "attn_combine",
                  "attn_split_phase2", "prep", "score_bg", "select_finalize_bg"]


class FreeKVError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"freekv status {status}: {msg}")
        self.status = status


class _Config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "n_layers", "batch", "n_qo", "n_kv", "head_dim", "page_size", "budget_tokens", "sink_tokens",
        "window_tokens", "max_ctx_tokens")] + [("tau", ctypes.c_float)] + [(n, ctypes.c_int32) for n in (
            "mode", "first_layer_dense", "kv_head_begin", "kv_head_end", "batch_begin", "batch_end",
            "n_ranks", "rank", "pool", "corr_pool")]


class _StepStats(ctypes.Structure):
    _fields_ = [("corrected_units", ctypes.c_int32), ("sync_pages", ctypes.c_int32), ("bg_pages", ctypes.c_int32),
                ("sync_bytes", ctypes.c_int64), ("bg_bytes", ctypes.c_int64)]


class _Buffers(ctypes.Structure):
    _fields_ = [("dev", ctypes.c_void_p), ("dev_bytes", ctypes.c_size_t), ("host", ctypes.c_void_p),
                ("host_bytes", ctypes.c_size_t)]


@dataclass
class FreeKVConfig:
    n_layers: int
    batch: int
    n_qo: int
    n_kv: int
    head_dim: int = 128
    page_size: int = 32
    budget_tokens: int = 2048
    sink_tokens: int = 512
    window_tokens: int = 512
    max_ctx_tokens: int = 32768 + 1024
    tau: float = 0.8
    mode: int = MODE_SPECULATIVE
    first_layer_dense: int = 0
    kv_head_begin: int = 0
    kv_head_end: int = 0
    batch_begin: int = 0
    batch_end: int = 0
    n_ranks: int = 1
    rank: int = 0
    pool: int = 0       # FREEKV_POOL_* (SURVEY §8(f) f3); 0 = MeanS (FreeKV)
    corr_pool: int = 0  # 0 = mean of the cosines (FreeKV), 1 = max pooling of the need to correct

    @property
    def G(self) -> int:
        return self.n_qo // self.n_kv

    @property
    def K(self) -> int:
        return (self.budget_tokens - self.sink_tokens - self.window_tokens) // self.page_size

    @property
    def units(self) -> int:
        return self.batch * self.n_kv

    def to_c(self) -> _Config:
        c = _Config()
        for f in fields(self):
            setattr(c, f.name, getattr(self, f.name))
        if c.kv_head_end == 0:
            c.kv_head_end = self.n_kv
        if c.batch_end == 0:
            c.batch_end = self.batch
        return c


_lib = None


def load_library():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FreeKVError(-3, f"{LIB_PATH} missing: run `python -m paper_2505_13109_b200.build` "
                                  "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
        P = ctypes.POINTER
        sigs = {
            "freekv_query_sizes": [P(_Config), P(sz), P(sz)],
            "freekv_init": [P(_Config), P(_Buffers), vp, vp, P(vp)],
            "freekv_append_kv": [vp, i32, vp, vp, i32, vp],
            "freekv_summarize_pages": [vp, i32, i32, i32, vp],
            "freekv_select_pages": [vp, i32, vp, vp, vp, vp],
            "freekv_recall_pages": [vp, i32, vp, vp],
            "freekv_sparse_decode_attn": [vp, i32, vp, vp, vp],
            "freekv_decode_step": [vp, i32, vp, vp, vp, vp],
            "freekv_get_selection": [vp, i32, vp, vp, vp, vp],
            "freekv_get_resident": [vp, i32, vp, vp],
            "freekv_get_fetch": [vp, i32, vp, vp],
            "freekv_get_step_stats": [vp, i32, P(_StepStats)],
            "freekv_comm_unique_id": [vp],
            "freekv_comm_init": [vp, vp, i32, i32],
            "freekv_set_gather_output": [vp, vp],
            "freekv_get_summaries": [vp, i32, i32, i32, i32, vp],
            "freekv_get_context": [vp, i32, P(i32)],
            "freekv_get_dims": [vp, P(i32), P(i32), P(i32)],
            "freekv_synchronize": [vp],
            "freekv_profile_begin": [vp, i32],
            "freekv_profile_end": [vp, vp, vp],
            "freekv_step_graph_capture": [vp, vp, vp, vp, vp, i32],
            "freekv_step_graph_capture_cycle": [vp, i32, vp, vp, vp, vp, i32],
            "freekv_step_graph_profile": [vp, vp, vp],
            "freekv_debug_trace": [vp, vp, sz],
            "freekv_step_graph_launch": [vp],
        }
        for name, args in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int32
        L.freekv_destroy.argtypes = [vp]
        L.freekv_destroy.restype = None
        L.freekv_last_error.restype = ctypes.c_char_p
        L.freekv_abi_version.restype = ctypes.c_int32
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise FreeKVError(st, load_library().freekv_last_error().decode())


def query_sizes(cfg: FreeKVConfig) -> tuple[int, int]:
    L = load_library()
    d, h = ctypes.c_size_t(), ctypes.c_size_t()
    c = cfg.to_c()
    _check(L.freekv_query_sizes(ctypes.byref(c), ctypes.byref(d), ctypes.byref(h)))
    return d.value, h.value


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class FreeKV:
    """One handle: n_layers of FreeKV state on the current CUDA device."""

    def __init__(self, cfg: FreeKVConfig, compute_stream=None, host_pool=None):
        import torch
        if not torch.cuda.is_available():
            raise FreeKVError(-3, "no CUDA device: the FreeKV path has no CPU fallback")
        self.L = load_library()
        self.cfg = cfg
        self.dev_bytes, self.host_bytes = query_sizes(cfg)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.dev = torch.empty(self.dev_bytes, dtype=torch.uint8, device=self.device)
        if host_pool is None:
            host_pool = torch.empty(self.host_bytes, dtype=torch.uint8, pin_memory=True)
        self.host = host_pool
        # the decode path outranks the background recall when SMs are contended
        self.stream = compute_stream if compute_stream is not None else torch.cuda.Stream(self.device, priority=-1)
        self.recall_stream = torch.cuda.Stream(self.device, priority=0)
        bufs = _Buffers(self.dev.data_ptr(), self.dev_bytes, self.host.data_ptr(), self.host_bytes)
        h = ctypes.c_void_p()
        c = cfg.to_c()
        _check(self.L.freekv_init(ctypes.byref(c), ctypes.byref(bufs), self.stream.cuda_stream,
                                  self.recall_stream.cuda_stream, ctypes.byref(h)))
        self.h = h
        K, npm, U = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(self.L.freekv_get_dims(self.h, ctypes.byref(K), ctypes.byref(npm), ctypes.byref(U)))
        self.K, self.n_page_max, self.U = K.value, npm.value, U.value

    # -- the C-ABI entry points ------------------------------------------------
    def _s(self, stream):
        return (stream or self.stream).cuda_stream

    def append_kv(self, layer, k, v, stream=None):
        n_new = k.shape[1]
        _check(self.L.freekv_append_kv(self.h, layer, k.data_ptr(), v.data_ptr(), n_new, self._s(stream)))

    def summarize_pages(self, layer, page_begin, page_end, stream=None):
        _check(self.L.freekv_summarize_pages(self.h, layer, page_begin, page_end, self._s(stream)))

    def select_pages(self, layer, q, pages_out=None, corrected_out=None, stream=None):
        _check(self.L.freekv_select_pages(self.h, layer, q.data_ptr(), _ptr(pages_out), _ptr(corrected_out),
                                          self._s(stream)))

    def recall_pages(self, layer, sync_mask=None, stream=None):
        """sync_mask: optional device uint8 [nb][n_kv] (units recalled synchronously)."""
        _check(self.L.freekv_recall_pages(self.h, layer, _ptr(sync_mask), self._s(stream)))

    def sparse_decode_attn(self, layer, q, out, stream=None):
        _check(self.L.freekv_sparse_decode_attn(self.h, layer, q.data_ptr(), out.data_ptr(), self._s(stream)))

    def decode_step(self, layer, q, k_new, v_new, out):
        _check(self.L.freekv_decode_step(self.h, layer, q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                                         out.data_ptr()))

    def step_graph_capture(self, q_all, k_all, v_all, out_all, profile=False):
        """Capture one decode step of every layer reading q_all [L][nb][n_qo][d], k_all/v_all
        [L][nb][1][n_kv][d] and writing out_all [L][nb][n_qo][d] (fixed device buffers)."""
        _check(self.L.freekv_step_graph_capture(self.h, q_all.data_ptr(), k_all.data_ptr(), v_all.data_ptr(),
                                                out_all.data_ptr(), int(profile)))
        self._graph_bufs = (q_all, k_all, v_all, out_all)

    def step_graph_capture_cycle(self, n_virtual, q_all, k_all, v_all, out_all, profile=False):
        """L_inst cycling: n_virtual virtual layers over the handle's n_layers (buffers [n_virtual]...)."""
        _check(self.L.freekv_step_graph_capture_cycle(self.h, n_virtual, q_all.data_ptr(), k_all.data_ptr(),
                                                      v_all.data_ptr(), out_all.data_ptr(), int(profile)))
        self._graph_bufs = (q_all, k_all, v_all, out_all)

    def step_graph_launch(self):
        _check(self.L.freekv_step_graph_launch(self.h))

    def step_graph_profile(self):
        """Per kernel class (ms, launches) of the last replay of a profile-mode step graph."""
        ms = np.zeros(len(KERNEL_CLASSES), np.float32)
        n = np.zeros(len(KERNEL_CLASSES), np.int32)
        _check(self.L.freekv_step_graph_profile(self.h, _np_ptr(ms), _np_ptr(n)))
        return {c: (float(ms[i]), int(n[i])) for i, c in enumerate(KERNEL_CLASSES)}

    def synchronize(self):
        _check(self.L.freekv_synchronize(self.h))

    def profile_begin(self, max_launches=200000):
        _check(self.L.freekv_profile_begin(self.h, max_launches))

    def profile_end(self):
        ms = np.zeros(len(KERNEL_CLASSES), np.float32)
        n = np.zeros(len(KERNEL_CLASSES), np.int32)
        _check(self.L.freekv_profile_end(self.h, _np_ptr(ms), _np_ptr(n)))
        return {c: (float(ms[i]), int(n[i])) for i, c in enumerate(KERNEL_CLASSES)}

    def debug_trace(self):
        """[12][4096][8] uint64 %globaltimer stamps (ns) of the kernels since the last call."""
        out = np.zeros((12, 4096, 8), np.uint64)
        _check(self.L.freekv_debug_trace(self.h, _np_ptr(out), out.size))
        return out

    # -- inspection (blocking) -------------------------------------------------
    def get_selection(self, layer):
        pages = np.empty((self.U, self.K), np.int32)
        front = np.empty(self.U, np.int32)
        flags = np.empty(self.U, np.uint8)
        cbar = np.empty(self.U, np.float32)
        _check(self.L.freekv_get_selection(self.h, layer, _np_ptr(pages), _np_ptr(front), _np_ptr(flags),
                                           _np_ptr(cbar)))
        return {"pages": pages, "frontier": front, "flags": flags, "cbar": cbar}

    def get_resident(self, layer):
        pages = np.empty((self.U, self.K), np.int32)
        front = np.empty(self.U, np.int32)
        _check(self.L.freekv_get_resident(self.h, layer, _np_ptr(pages), _np_ptr(front)))
        return pages, front

    def get_fetch(self, layer):
        n = np.empty(self.U, np.int32)
        pages = np.empty((self.U, self.K), np.int32)
        _check(self.L.freekv_get_fetch(self.h, layer, _np_ptr(n), _np_ptr(pages)))
        return n, pages

    # -- multi-GPU: the library's own NCCL communicator and per-layer all-gather ---------------
    @staticmethod
    def comm_unique_id() -> bytes:
        """Rank 0: a fresh NCCL unique id (128 bytes) to broadcast to the other ranks."""
        L = load_library()
        buf = (ctypes.c_uint8 * 128)()
        _check(L.freekv_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
        return bytes(buf)

    def comm_init(self, uid: bytes, n_ranks: int, rank: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(self.L.freekv_comm_init(self.h, ctypes.cast(buf, ctypes.c_void_p), n_ranks, rank))

    def set_gather_output(self, gather_all):
        """gather_all: device fp32 [n_layers][n_ranks][nb][n_qo][d] (or None)."""
        self._gather = gather_all
        _check(self.L.freekv_set_gather_output(self.h, _ptr(gather_all)))

    def get_step_stats(self, layer):
        """Recall accounting of the layer's last step (freekv_get_step_stats)."""
        st = _StepStats()
        _check(self.L.freekv_get_step_stats(self.h, layer, ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in _StepStats._fields_}

    def get_summaries(self, layer, unit, page_begin, page_end):
        out = np.empty((page_end - page_begin, 2, self.cfg.head_dim), np.uint16)
        _check(self.L.freekv_get_summaries(self.h, layer, unit, page_begin, page_end, _np_ptr(out)))
        return out

    def context(self, layer) -> int:
        c = ctypes.c_int32()
        _check(self.L.freekv_get_context(self.h, layer, ctypes.byref(c)))
        return c.value

    def close(self):
        if getattr(self, "h", None):
            self.L.freekv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
