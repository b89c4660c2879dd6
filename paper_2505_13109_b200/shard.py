"""Multi-GPU partition of the FreeKV decode path.

Units (batch row, KV head) are independent in every stage (per-head softmax,
group pooling inside a GQA group, per-unit top-K, correction and recall), so
the path shards by KV head -- a group never straddles GPUs -- and, when there
are more GPUs than KV heads, by batch.  The only exchange is gathering the
per-head attention outputs (one all-gather per layer over NCCL/NVLink).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    kv_begin: int
    kv_end: int
    batch_begin: int
    batch_end: int

    @property
    def n_kv(self) -> int:
        return self.kv_end - self.kv_begin

    @property
    def batch(self) -> int:
        return self.batch_end - self.batch_begin


def shard_for(n_kv: int, batch: int, world: int, rank: int) -> Shard:
    """Contiguous KV-head blocks for world <= n_kv; one KV head x a batch chunk otherwise."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if world <= n_kv:
        if n_kv % world:
            raise ValueError("world size must divide n_kv")
        per = n_kv // world
        return Shard(rank * per, (rank + 1) * per, 0, batch)
    if world % n_kv or batch % (world // n_kv):
        raise ValueError("world must be a multiple of n_kv that divides batch * n_kv")
    chunks = world // n_kv
    m, c = divmod(rank, chunks)
    per_b = batch // chunks
    return Shard(m, m + 1, c * per_b, (c + 1) * per_b)


def assemble(gathered, shards, n_qo: int, n_kv: int, batch: int):
    """Place every rank's [batch_loc][n_qo_loc][d] output block into the global
    [batch][n_qo][d] tensor (the all-gather is a pure copy)."""
    import torch
    G = n_qo // n_kv
    d = gathered[0].shape[-1]
    out = torch.empty(batch, n_qo, d, dtype=gathered[0].dtype, device=gathered[0].device)
    for blk, s in zip(gathered, shards):
        out[s.batch_begin:s.batch_end, s.kv_begin * G:s.kv_end * G] = blk
    return out
