"""Seeded synthetic inputs for FreeKV's decode path (DESIGN.md §6 input recipe).

This module is shared by the oracle side (tests, bench cpu_baseline) and the
CUDA side (tests, bench).  It holds NONE of the method's arithmetic: it only
draws random bf16 tensors with the structure of the paper's workloads.

  GEN-S (keys/values): per (layer, unit) a unit "topic" u_m (unit-norm
        Gaussian); keys k_t = z_t + alpha * w_page(t) * u_m with z ~ N(0, I_d),
        w = 0 for cold pages and w = 0.5 + Exp(1) (heavy-tailed importance) for
        hot pages; values v ~ N(0, I_d).  At prefill 1.5*K random candidate
        pages are hot; every later page is hot with probability p_hot.  This
        mimics the vertical attention lines of P:184 (fig:algo-ob2) so
        selections stay stable across steps (delta recall).
  GEN-Q (queries): q_{h,i} = beta * u_{m(h)} + e_{h,i},
        e_{h,i} = rho * e_{h,i-1} + sqrt(1 - rho^2) * xi,  xi ~ N(0, I_d).
        beta = 6, rho = 0.872 give mean adjacent cosine ~0.89 (Table
        tab:q-sim-all 0.82-0.92) and ~0.8 changed pages per unit per step at
        K = 32 (measured).  With probability `event_rate` per
        (step, b, kv-head) the unit's heads redraw e with rho = 0
        (cosine ~0.22 < tau): a controlled correction rate (Table
        tab:corr-rate 0.04-0.52).
Everything is rounded once to bf16 (round-to-nearest-even by torch).
"""
from __future__ import annotations

import math

import torch

SEED0 = 250513109
ALPHA = 8.0   # hot-page key shift along the unit topic (x heavy-tailed weight 0.5 + Exp(1))
BETA = 6.0    # persistent query component along the topic
RHO = 0.872   # AR(1) coefficient of the query innovation: mean adjacent cosine (36 + 128 rho)/164 = 0.90


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return g


def topics(batch: int, n_kv: int, d: int, seed: int, layer: int, device="cpu") -> torch.Tensor:
    g = _gen(seed * 1000003 + layer * 7919 + 1, device)
    u = torch.randn(batch, n_kv, d, generator=g, device=device, dtype=torch.float32)
    return u / u.norm(dim=-1, keepdim=True)


def gen_prefill(batch, n_kv, d, page, L0, n_sink_pages, K, seed, layer, device="cpu",
                alpha: float = ALPHA, hot_factor: float = 1.5):
    """Prefill K/V, NHD [batch][L0][n_kv][d] bf16, with hot_factor*K hot candidate pages per unit.

    Hot page j gets strength alpha * w_j with w_j = 0.5 + Exp(1): a heavy-tailed
    page importance, so the top of the ranking is stable step to step and the
    churn is concentrated at the selection boundary."""
    g = _gen(seed * 1000003 + layer * 7919 + 2, device)
    u = topics(batch, n_kv, d, seed, layer, device)
    k = torch.randn(batch, L0, n_kv, d, generator=g, device=device, dtype=torch.float32)
    v = torch.randn(batch, L0, n_kv, d, generator=g, device=device, dtype=torch.float32)
    n_pages = L0 // page
    n_cand = max(0, n_pages - n_sink_pages)
    n_hot = min(n_cand, int(math.ceil(hot_factor * K)))
    if n_hot > 0:
        hot = torch.zeros(batch, n_kv, n_pages, device=device, dtype=torch.float32)
        scores = torch.rand(batch, n_kv, n_cand, generator=g, device=device)
        idx = scores.topk(n_hot, dim=-1).indices + n_sink_pages
        w = 0.5 + torch.empty(batch, n_kv, n_hot, device=device).exponential_(1.0, generator=g)
        hot.scatter_(2, idx, w)
        hot_tok = hot.repeat_interleave(page, dim=2)                     # [b][kv][n_pages*page]
        hot_tok = torch.nn.functional.pad(hot_tok, (0, L0 - hot_tok.shape[2]))
        k = k + alpha * hot_tok.permute(0, 2, 1).unsqueeze(-1) * u.unsqueeze(1)
    return k.to(torch.bfloat16), v.to(torch.bfloat16)


def gen_decode_kv(batch, n_kv, d, page, t, seed, layer, device="cpu", alpha: float = ALPHA,
                  p_hot: float = 0.05):
    """k/v of the token at position t, NHD [batch][1][n_kv][d] bf16."""
    g = _gen(seed * 1000003 + layer * 7919 + 3 + 104729 * t, device)
    u = topics(batch, n_kv, d, seed, layer, device)
    k = torch.randn(batch, 1, n_kv, d, generator=g, device=device, dtype=torch.float32)
    v = torch.randn(batch, 1, n_kv, d, generator=g, device=device, dtype=torch.float32)
    gp = _gen(seed * 1000003 + layer * 7919 + 5 + 104729 * (t // page), device)
    hot = (torch.rand(batch, n_kv, generator=gp, device=device) < p_hot).float()
    hot = hot * (0.5 + torch.empty(batch, n_kv, device=device).exponential_(1.0, generator=gp))
    k = k + alpha * (hot.unsqueeze(-1) * u).unsqueeze(1)
    return k.to(torch.bfloat16), v.to(torch.bfloat16)


class QueryProcess:
    """GEN-Q for one layer: call next() once per decode step."""

    def __init__(self, batch, n_qo, n_kv, d, seed, layer, device="cpu", beta: float = BETA,
                 rho: float = RHO, event_rate: float = 0.05):
        self.batch, self.n_qo, self.n_kv, self.d = batch, n_qo, n_kv, d
        self.G = n_qo // n_kv
        self.beta, self.rho, self.event_rate = beta, rho, event_rate
        self.device = device
        self.g = _gen(seed * 1000003 + layer * 7919 + 4, device)
        self.u = topics(batch, n_kv, d, seed, layer, device)
        self.e = torch.randn(batch, n_qo, d, generator=self.g, device=device)
        self.step = 0

    def next(self):
        """Returns (q [batch][n_qo][d] bf16, events [batch][n_kv] bool)."""
        xi = torch.randn(self.batch, self.n_qo, self.d, generator=self.g, device=self.device)
        ev = torch.rand(self.batch, self.n_kv, generator=self.g, device=self.device) < self.event_rate
        if self.step == 0:
            ev = torch.zeros_like(ev)
        rho = torch.full((self.batch, self.n_kv), self.rho, device=self.device)
        rho = torch.where(ev, torch.zeros_like(rho), rho).repeat_interleave(self.G, dim=1).unsqueeze(-1)
        self.e = rho * self.e + torch.sqrt(1 - rho * rho) * xi
        q = self.beta * self.u.repeat_interleave(self.G, dim=1) + self.e
        self.step += 1
        return q.to(torch.bfloat16), ev


def bf16_bits(t: torch.Tensor):
    """bf16 tensor -> numpy uint16 bit patterns (CPU copy)."""
    return t.detach().to("cpu").contiguous().view(torch.int16).numpy().view("uint16")


def from_bits(a, device="cpu") -> torch.Tensor:
    import numpy as np
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(device)
