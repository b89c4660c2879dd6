"""CPU oracle of FreeKV's per-layer decode-step KV-retrieval path (arXiv 2505.13109).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  It shares no code with ``paper_2505_13109_b200`` and never imports it.

The arithmetic lives in ``freekv_oracle.c`` (plain C, one function per paper
step, CFR of DESIGN.md §3).  This file is the ctypes binding plus the decode
state machine O-1..O-7 of DESIGN.md §3 written step by step
in the paper's order:

  O-1 append       P:317, P:231         (page leaves the window -> summary)
  O-2 correction   P:247-250 (§3.3)     (group-mean cosine < tau)
  O-3 selection    P:231-234, P:257     (for every unit, every step)
  O-4 pages used   P:223, P:255-256     (flagged: S_i; others: resident)
  O-5 attention    P:95-97, P:100       (fp64 over sink + pages + local)
  O-6 advance      P:225                (resident := S_i, q_prev := q_i)
  O-7 layer 0 dense when first_layer_dense

Parity status: every function is pinned by tests/test_oracle_pins.py (see the
table in DESIGN.md §3); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "freekv_oracle.c")

MODE_SPECULATIVE, MODE_ALWAYS, MODE_NEVER = 0, 1, 2

_u16p = ctypes.POINTER(ctypes.c_uint16)
_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build(force: bool = False) -> str:
    """Compile the oracle with the CFR-0 flags (gcc, no fast-math, no contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "freekv_oracle.h"))
    ):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _SO, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.fko_bf16_to_f32.restype = ctypes.c_float
        L.fko_bf16_to_f32.argtypes = [ctypes.c_uint16]
        L.fko_f32_to_bf16.restype = ctypes.c_uint16
        L.fko_f32_to_bf16.argtypes = [ctypes.c_float]
        L.fko_page_summary.argtypes = [_u16p, ctypes.c_int, ctypes.c_int, _u16p, _u16p]
        L.fko_page_bound.restype = ctypes.c_float
        L.fko_page_bound.argtypes = [_u16p, _u16p, _u16p, ctypes.c_int]
        L.fko_score_scale.restype = ctypes.c_float
        L.fko_score_scale.argtypes = [ctypes.c_int]
        L.fko_cexp2.restype = ctypes.c_float
        L.fko_cexp2.argtypes = [ctypes.c_float]
        L.fko_tree_sum.restype = ctypes.c_float
        L.fko_tree_sum.argtypes = [_f32p, ctypes.c_int]
        L.fko_pool_means.argtypes = [_f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _f32p]
        L.fko_topk.restype = ctypes.c_int
        L.fko_topk.argtypes = [_f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i32p]
        L.fko_select_unit.restype = ctypes.c_int
        L.fko_select_unit.argtypes = [_u16p, _u16p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, _i32p, _f32p]
        L.fko_cosine.restype = ctypes.c_float
        L.fko_cosine.argtypes = [_u16p, _u16p, ctypes.c_int]
        L.fko_pool_correct.restype = ctypes.c_int
        L.fko_pool_correct.argtypes = [_f32p, ctypes.c_int, ctypes.c_float, ctypes.c_int, _f32p]
        L.fko_correct_unit.restype = ctypes.c_int
        L.fko_correct_unit.argtypes = [_u16p, _u16p, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                       ctypes.c_int, ctypes.c_int, _f32p]
        L.fko_attn_unit.argtypes = [_u16p, _u16p, _u16p, ctypes.c_int, ctypes.c_int, _i32p,
                                    ctypes.c_int, _f64p]
        L.fko_select_batch.argtypes = [ctypes.c_int, _u16p, ctypes.POINTER(_u16p), ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, _i32p, ctypes.c_int, _i32p]
        L.fko_attn_batch.argtypes = [ctypes.c_int, _u16p, ctypes.POINTER(_u16p), ctypes.POINTER(_u16p),
                                     ctypes.c_int, ctypes.c_int, ctypes.POINTER(_i32p), _i32p, _f64p]
        L.fko_num_threads.restype = ctypes.c_int
        L.fko_select_unit_pool.restype = ctypes.c_int
        L.fko_select_unit_pool.argtypes = [_u16p, _u16p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, _i32p, _f32p]
        L.fko_pool_correct_v.restype = ctypes.c_int
        L.fko_pool_correct_v.argtypes = [_f32p, ctypes.c_int, ctypes.c_float, ctypes.c_int, ctypes.c_int, _f32p]
        _lib = L
    return _lib


def _p(a: np.ndarray, t):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


def _u16(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint16))


# ---------------------------------------------------------------- bf16 helpers
def bf16_to_f32(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.uint16)
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bits (test input construction only)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = x.view(np.uint32).astype(np.uint64)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)


# ------------------------------------------------------------ single functions
def page_summary(keys) -> tuple[np.ndarray, np.ndarray]:
    keys = _u16(keys)
    n_tok, d = keys.shape
    mn = np.empty(d, np.uint16)
    mx = np.empty(d, np.uint16)
    lib().fko_page_summary(_p(keys, _u16p), n_tok, d, _p(mn, _u16p), _p(mx, _u16p))
    return mn, mx


def page_bound(q, mn, mx) -> float:
    q, mn, mx = _u16(q), _u16(mn), _u16(mx)
    return lib().fko_page_bound(_p(q, _u16p), _p(mn, _u16p), _p(mx, _u16p), q.shape[0])


def score_scale(d: int) -> np.float32:
    return np.float32(lib().fko_score_scale(d))


def cexp2(x: float) -> np.float32:
    return np.float32(lib().fko_cexp2(float(x)))


def tree_sum(a) -> np.float32:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    return np.float32(lib().fko_tree_sum(_p(a, _f32p), a.shape[0]))


def pool_means(s, j_begin: int, j_end: int) -> np.ndarray:
    s = np.ascontiguousarray(np.asarray(s, dtype=np.float32))
    G, ld = s.shape
    pooled = np.zeros(ld, np.float32)
    lib().fko_pool_means(_p(s, _f32p), G, ld, j_begin, j_end, _p(pooled, _f32p))
    return pooled


def topk(pooled, j_begin: int, j_end: int, K: int) -> np.ndarray:
    pooled = np.ascontiguousarray(np.asarray(pooled, dtype=np.float32))
    sel = np.empty(K, np.int32)
    lib().fko_topk(_p(pooled, _f32p), j_begin, j_end, K, _p(sel, _i32p))
    return sel


def select_unit(q, summ, n_sink: int, n_off: int, K: int, want_pooled: bool = False):
    """q: [G][d] bf16 bits; summ: [>=n_off][2][d] bf16 bits (min, max)."""
    q = _u16(q)
    summ = _u16(summ)
    G, d = q.shape
    sel = np.empty(K, np.int32)
    pooled = np.zeros(max(n_off, 1), np.float32)
    lib().fko_select_unit(_p(q, _u16p), _p(summ, _u16p), G, d, n_sink, n_off, K,
                          _p(sel, _i32p), _p(pooled, _f32p))
    return (sel, pooled) if want_pooled else sel


# group-consistency variants (tab:abl-g-cons)
POOL_MEAN_S, POOL_MAX_S, POOL_MEAN_QK, POOL_MAX_QK, POOL_MEAN_Q, POOL_MAX_Q = range(6)
POOL_NAMES = ["MeanS", "MaxS", "MeanQK", "MaxQK", "MeanQ", "MaxQ"]


def select_unit_pool(q, summ, n_sink: int, n_off: int, K: int, pool: int, want_pooled: bool = False):
    """select_unit with the group pooling `pool` (POOL_*)."""
    q = _u16(q)
    summ = _u16(summ)
    G, d = q.shape
    sel = np.empty(K, np.int32)
    pooled = np.zeros(max(n_off, 1), np.float32)
    lib().fko_select_unit_pool(_p(q, _u16p), _p(summ, _u16p), G, d, n_sink, n_off, K, pool,
                               _p(sel, _i32p), _p(pooled, _f32p))
    return (sel, pooled) if want_pooled else sel


def pool_correct_v(C, tau: float, mode: int, cpool: int) -> tuple[int, np.float32]:
    """Correction pooling: cpool 0 mean (FreeKV), 1 max pooling of the need to correct (R-11)."""
    C = np.ascontiguousarray(np.asarray(C, dtype=np.float32))
    cbar = ctypes.c_float()
    f = lib().fko_pool_correct_v(_p(C, _f32p), C.shape[0], tau, mode, cpool, ctypes.byref(cbar))
    return f, np.float32(cbar.value)


def cosine(a, b) -> np.float32:
    a, b = _u16(a), _u16(b)
    return np.float32(lib().fko_cosine(_p(a, _u16p), _p(b, _u16p), a.shape[0]))


def pool_correct(C, tau: float, mode: int = MODE_SPECULATIVE) -> tuple[int, np.float32]:
    C = np.ascontiguousarray(np.asarray(C, dtype=np.float32))
    cbar = ctypes.c_float()
    f = lib().fko_pool_correct(_p(C, _f32p), C.shape[0], tau, mode, ctypes.byref(cbar))
    return f, np.float32(cbar.value)


def correct_unit(q, q_prev, tau: float, mode: int, bootstrap: bool) -> tuple[int, np.float32]:
    q, q_prev = _u16(q), _u16(q_prev)
    G, d = q.shape
    cbar = ctypes.c_float()
    f = lib().fko_correct_unit(_p(q, _u16p), _p(q_prev, _u16p), G, d, tau, mode,
                               int(bootstrap), ctypes.byref(cbar))
    return f, np.float32(cbar.value)


def attn_unit(q, Kt, Vt, toks) -> np.ndarray:
    q, Kt, Vt = _u16(q), _u16(Kt), _u16(Vt)
    toks = np.ascontiguousarray(np.asarray(toks, dtype=np.int32))
    G, d = q.shape
    out = np.zeros((G, d), np.float64)
    lib().fko_attn_unit(_p(q, _u16p), _p(Kt, _u16p), _p(Vt, _u16p), G, d, _p(toks, _i32p),
                        toks.shape[0], _p(out, _f64p))
    return out


def num_threads() -> int:
    return lib().fko_num_threads()


# -------------------------------------------------------------- state machine
@dataclass
class OracleConfig:
    n_layers: int
    batch: int
    n_qo: int
    n_kv: int
    head_dim: int
    page_size: int
    budget_tokens: int
    sink_tokens: int
    window_tokens: int
    max_ctx_tokens: int
    tau: float = 0.8
    mode: int = MODE_SPECULATIVE
    first_layer_dense: bool = False
    pool: int = 0       # POOL_* (f3); 0 = MeanS, FreeKV's choice
    corr_pool: int = 0  # 0 = mean over the group (FreeKV), 1 = max pooling of the need to correct

    @property
    def G(self) -> int:
        return self.n_qo // self.n_kv

    @property
    def K(self) -> int:  # A-6: B counts sink + window + selected
        return (self.budget_tokens - self.sink_tokens - self.window_tokens) // self.page_size

    @property
    def n_sink(self) -> int:
        return self.sink_tokens // self.page_size

    @property
    def n_win(self) -> int:
        return self.window_tokens // self.page_size


class OracleEngine:
    """Decode state machine O-1..O-7 over host arrays (one entry per layer)."""

    def __init__(self, cfg: OracleConfig):
        self.cfg = cfg
        U = cfg.batch * cfg.n_kv
        self.U = U
        L, d = cfg.max_ctx_tokens, cfg.head_dim
        self.Kc = [np.zeros((U, L, d), np.uint16) for _ in range(cfg.n_layers)]
        self.Vc = [np.zeros((U, L, d), np.uint16) for _ in range(cfg.n_layers)]
        n_page_max = L // cfg.page_size + 1
        self.summ = [np.zeros((U, n_page_max, 2, d), np.uint16) for _ in range(cfg.n_layers)]
        self.Lc = [0] * cfg.n_layers
        self.n_off = [[cfg.n_sink] * U for _ in range(cfg.n_layers)]
        self.R = [[None] * U for _ in range(cfg.n_layers)]      # resident page list (None = none yet)
        self.fR = [[0] * U for _ in range(cfg.n_layers)]
        self.q_prev = [np.zeros((cfg.batch, cfg.n_qo, d), np.uint16) for _ in range(cfg.n_layers)]

    # O-1 -----------------------------------------------------------------
    def append(self, layer: int, k_new, v_new):
        """k_new/v_new: [batch][n_new][n_kv][d] bf16 bits (NHD)."""
        cfg = self.cfg
        k_new, v_new = _u16(k_new), _u16(v_new)
        nb, n_new, n_kv, d = k_new.shape
        L0 = self.Lc[layer]
        if L0 + n_new > cfg.max_ctx_tokens:
            raise ValueError("context exceeds max_ctx_tokens")
        for b in range(nb):
            for m in range(n_kv):
                u = b * n_kv + m
                self.Kc[layer][u, L0:L0 + n_new] = k_new[b, :, m]
                self.Vc[layer][u, L0:L0 + n_new] = v_new[b, :, m]
        Lc = L0 + n_new
        self.Lc[layer] = Lc
        p = cfg.page_size
        n_pc = Lc // p
        new_off = max(cfg.n_sink, n_pc - cfg.n_win)
        for u in range(self.U):
            old = self.n_off[layer][u]
            for j in range(old, new_off):  # page j leaves the window
                mn, mx = page_summary(self.Kc[layer][u, j * p:(j + 1) * p])
                self.summ[layer][u, j, 0] = mn
                self.summ[layer][u, j, 1] = mx
            self.n_off[layer][u] = max(old, new_off)
        if n_new > 1:  # bulk append restarts speculation (reading R-9)
            self.R[layer] = [None] * self.U

    def token_set(self, layer: int, u: int, sel, f: int) -> np.ndarray:
        """A-9: T = [0, min(S, Lc)) U pages(sel) U [f*p, Lc)."""
        cfg = self.cfg
        p, Lc = cfg.page_size, self.Lc[layer]
        parts = [np.arange(0, min(cfg.sink_tokens, Lc))]
        for j in sel:
            if j >= 0:
                parts.append(np.arange(j * p, (j + 1) * p))
        parts.append(np.arange(min(f * p, Lc), Lc))
        return np.concatenate(parts).astype(np.int32)

    # O-2..O-6 --------------------------------------------------------------
    def step(self, layer: int, q, k_new, v_new, select_only: bool = False):
        """One decode step of one layer.  q: [batch][n_qo][d] bf16 bits."""
        cfg = self.cfg
        self.append(layer, k_new, v_new)
        q = _u16(q)
        G, d, n_kv = cfg.G, cfg.head_dim, cfg.n_kv
        U = self.U
        flags = np.zeros(U, np.uint8)
        cbar = np.zeros(U, np.float32)
        for u in range(U):
            b, m = divmod(u, n_kv)
            qg = q[b, m * G:(m + 1) * G]
            qp = self.q_prev[layer][b, m * G:(m + 1) * G]
            if cfg.corr_pool == 0:
                f, c = correct_unit(qg, qp, cfg.tau, cfg.mode, self.R[layer][u] is None)
            else:
                C = [cosine(qg[g], qp[g]) for g in range(G)]
                f, c = pool_correct_v(C, cfg.tau, cfg.mode, cfg.corr_pool)
                if self.R[layer][u] is None:
                    f = 1  # A-12
            flags[u], cbar[u] = f, c
        # O-3: selection with q_i for every unit
        qs = np.ascontiguousarray(q.reshape(U, G, d))
        summ_ptrs = (_u16p * U)(*[self.summ[layer][u].ctypes.data_as(_u16p) for u in range(U)])
        n_off = np.array(self.n_off[layer], np.int32)
        sel = np.empty((U, cfg.K), np.int32)
        if cfg.pool == POOL_MEAN_S:
            lib().fko_select_batch(U, _p(qs, _u16p), summ_ptrs, G, d, cfg.n_sink, _p(n_off, _i32p),
                                   cfg.K, _p(sel, _i32p))
        else:
            for u in range(U):
                sel[u] = select_unit_pool(qs[u], self.summ[layer][u], cfg.n_sink, int(n_off[u]), cfg.K, cfg.pool)
        # O-4: pages used by this step's attention
        used_sel, used_f, fetch_sync, fetch_bg = [], [], [], []
        for u in range(U):
            Si = [int(j) for j in sel[u] if j >= 0]
            R = self.R[layer][u]
            Rset = set(R) if R is not None else set()
            fetch = [j for j in Si if j not in Rset]
            if flags[u]:
                used_sel.append(Si)
                used_f.append(int(n_off[u]))
                fetch_sync.append(fetch)
                fetch_bg.append([])
            else:
                used_sel.append(list(R))
                used_f.append(self.fR[layer][u])
                fetch_sync.append([])
                fetch_bg.append(fetch)
        out = None
        if not select_only:
            dense = cfg.first_layer_dense and layer == 0
            toks = [np.arange(self.Lc[layer], dtype=np.int32) if dense
                    else self.token_set(layer, u, used_sel[u], used_f[u]) for u in range(U)]
            out = self.attention(layer, qs, toks).reshape(cfg.batch, cfg.n_qo, d)
        # O-6: advance
        for u in range(U):
            self.R[layer][u] = [int(j) for j in sel[u] if j >= 0]
            self.fR[layer][u] = int(n_off[u])
        self.q_prev[layer] = q.copy()
        return {
            "Lc": self.Lc[layer], "flags": flags, "cbar": cbar, "sel": sel, "frontier": n_off.copy(),
            "used_sel": used_sel, "used_f": used_f,
            "fetch_sync": fetch_sync, "fetch_bg": fetch_bg, "out": out,
        }

    def attention(self, layer: int, qs: np.ndarray, toks) -> np.ndarray:
        cfg = self.cfg
        U, G, d = self.U, cfg.G, cfg.head_dim
        toks = [np.ascontiguousarray(t, dtype=np.int32) for t in toks]
        out = np.zeros((U, G, d), np.float64)
        kp = (_u16p * U)(*[self.Kc[layer][u].ctypes.data_as(_u16p) for u in range(U)])
        vp = (_u16p * U)(*[self.Vc[layer][u].ctypes.data_as(_u16p) for u in range(U)])
        tp = (_i32p * U)(*[t.ctypes.data_as(_i32p) for t in toks])
        nt = np.array([t.shape[0] for t in toks], np.int32)
        lib().fko_attn_batch(U, _p(qs, _u16p), kp, vp, G, d, tp, _p(nt, _i32p), _p(out, _f64p))
        return out
