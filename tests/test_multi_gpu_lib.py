"""World-size-2 decode through the library's own NCCL communicator: each rank
holds one kv-head shard of the same model, the per-layer all-gather runs inside the library
(eagerly and in the step graph), and rank 0 checks the gathered outputs and every rank its
selections against the CPU oracle of the full configuration.  Needs two GPUs (one process per
GPU); skipped otherwise -- the partition / gather host logic is covered on CPU by
test_shard_gloo.py."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, graph, q):
    try:
        import torch.distributed as dist

        import paper_2505_13109_b200 as P
        import synth
        from oracle import oracle as O
        from paper_2505_13109_b200.shard import assemble, shard_for
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        nb, n_qo, n_kv, d, p, L0, n_layers, steps = 2, 8, 2, 128, 32, 1500, 2, 3
        G = n_qo // n_kv
        sh = shard_for(n_kv, nb, world, rank)
        kw = dict(n_layers=n_layers, head_dim=d, page_size=p, budget_tokens=256, sink_tokens=64, window_tokens=64,
                  max_ctx_tokens=L0 + steps + 4)
        fkv = P.FreeKV(P.FreeKVConfig(batch=sh.batch, n_qo=sh.n_kv * G, n_kv=sh.n_kv, **kw))
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid.copy_(torch.tensor(list(P.FreeKV.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        fkv.comm_init(bytes(uid.tolist()), world, rank)
        gat = torch.empty(n_layers, world, sh.batch, sh.n_kv * G, d, dtype=torch.float32, device=fkv.device)
        fkv.set_gather_output(gat)
        eng = O.OracleEngine(O.OracleConfig(batch=nb, n_qo=n_qo, n_kv=n_kv, **kw))
        seed = 77
        for l in range(n_layers):
            k, v = synth.gen_prefill(nb, n_kv, d, p, L0, 2, eng.cfg.K, seed, l)
            eng.append(l, synth.bf16_bits(k), synth.bf16_bits(v))
            fkv.append_kv(l, k[sh.batch_begin:sh.batch_end, :, sh.kv_begin:sh.kv_end].contiguous().to(fkv.device),
                          v[sh.batch_begin:sh.batch_end, :, sh.kv_begin:sh.kv_end].contiguous().to(fkv.device))
        fkv.synchronize()
        qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, l, event_rate=0.3) for l in range(n_layers)]
        qb = torch.empty(n_layers, sh.batch, sh.n_kv * G, d, dtype=torch.bfloat16, device=fkv.device)
        kb = torch.empty(n_layers, sh.batch, 1, sh.n_kv, d, dtype=torch.bfloat16, device=fkv.device)
        vb = torch.empty_like(kb)
        ob = torch.empty(n_layers, sh.batch, sh.n_kv * G, d, dtype=torch.float32, device=fkv.device)
        captured = False
        worst = 0.0
        for i in range(steps):
            refs = []
            for l in range(n_layers):
                qf, _ = qps[l].next()
                kf, vf = synth.gen_decode_kv(nb, n_kv, d, p, L0 + i, seed, l)
                refs.append(eng.step(l, synth.bf16_bits(qf), synth.bf16_bits(kf), synth.bf16_bits(vf)))
                qb[l] = qf[sh.batch_begin:sh.batch_end, sh.kv_begin * G:sh.kv_end * G].to(fkv.device)
                kb[l] = kf[sh.batch_begin:sh.batch_end, :, sh.kv_begin:sh.kv_end].to(fkv.device)
                vb[l] = vf[sh.batch_begin:sh.batch_end, :, sh.kv_begin:sh.kv_end].to(fkv.device)
            torch.cuda.synchronize()
            if graph:
                if not captured:
                    fkv.step_graph_capture(qb, kb, vb, ob)
                    captured = True
                fkv.step_graph_launch()
            else:
                for l in range(n_layers):
                    fkv.decode_step(l, qb[l], kb[l], vb[l], ob[l])
            fkv.synchronize()
            shards = [shard_for(n_kv, nb, world, r) for r in range(world)]
            for l in range(n_layers):
                full = assemble([gat[l, r].cpu() for r in range(world)], shards, n_qo, n_kv, nb).double().numpy()
                ref = refs[l]["out"]
                num = np.abs(full - ref).max(axis=-1)
                den = np.maximum(np.abs(ref).max(axis=-1), 1e-6)
                worst = max(worst, float((num / den).max()))
                sel = fkv.get_selection(l)
                units = [b * n_kv + m for b in range(sh.batch_begin, sh.batch_end) for m in range(sh.kv_begin, sh.kv_end)]
                assert np.array_equal(sel["pages"], refs[l]["sel"][units]), (rank, i, l)
                assert np.array_equal(sel["flags"], refs[l]["flags"][units]), (rank, i, l)
        assert worst <= 2e-3, worst
        fkv.close()
        dist.destroy_process_group()
        q.put((rank, "ok", worst))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, "fail", traceback.format_exc()))


@pytest.mark.parametrize("graph", [False, True])
def test_world2_through_library(graph):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one process per GPU)")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, graph, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r, st, info in res:
        assert st == "ok", (r, info)
