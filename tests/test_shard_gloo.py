"""Multi-process (gloo, world_size 2 and 4) checks of the multi-GPU partition and
the per-layer output all-gather of SURVEY.md §8(e), on CPU.  Each rank fills its
shard's outputs with a value that encodes (b, head, channel); after the gather
every rank must hold exactly the global tensor (the gather is a pure copy)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_13109_b200.shard import assemble, shard_for


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_kv, n_qo, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = 8
    G = n_qo // n_kv
    shards = [shard_for(n_kv, batch, world, r) for r in range(world)]
    me = shards[rank]
    b = torch.arange(me.batch_begin, me.batch_end).view(-1, 1, 1).float()
    h = torch.arange(me.kv_begin * G, me.kv_end * G).view(1, -1, 1).float()
    c = torch.arange(d).view(1, 1, -1).float()
    local = (b * 10000 + h * 100 + c).contiguous()
    gathered = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(gathered, local)
    out = assemble(gathered, shards, n_qo, n_kv, batch)
    bb = torch.arange(batch).view(-1, 1, 1).float()
    hh = torch.arange(n_qo).view(1, -1, 1).float()
    ref = bb * 10000 + hh * 100 + c
    q.put((rank, bool(torch.equal(out, ref))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_kv,n_qo,batch", [(2, 8, 32, 8), (4, 8, 64, 16), (2, 1, 4, 4)])
def test_shard_and_gather(world, n_kv, n_qo, batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_kv, n_qo, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_shard_partition_covers_units_once():
    for n_kv, batch in [(8, 8), (4, 4), (8, 16)]:
        for world in (1, 2, 4, 8):
            if world > n_kv and (world % n_kv or batch % (world // n_kv)):
                continue
            seen = set()
            for r in range(world):
                s = shard_for(n_kv, batch, world, r)
                for b in range(s.batch_begin, s.batch_end):
                    for m in range(s.kv_begin, s.kv_end):
                        assert (b, m) not in seen
                        seen.add((b, m))
            assert len(seen) == n_kv * batch
