"""Small decode runs for compute-sanitizer (memcheck / racecheck / synccheck): every default kernel
of the serial step (score grid with the append / correction CTAs, select, attention with the
cluster merge and commit, background recall), eagerly and through the step graph, plus the
primitive API (append, select_pages, recall_pages, sparse_decode_attn, summarize_pages).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py c1|c2s
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_2505_13109_b200 as P
import synth

CFG = {"c1": dict(nb=1, n_qo=32, n_kv=8, ctx=4096, budget=512, sink=128, window=128, layers=1),
       "c2s": dict(nb=2, n_qo=32, n_kv=8, ctx=8192, budget=2048, sink=512, window=512, layers=2)}
c = CFG[sys.argv[1] if len(sys.argv) > 1 else "c1"]
nb, n_qo, n_kv, d, p, L = c["nb"], c["n_qo"], c["n_kv"], 128, 32, c["layers"]
steps = 3
cfg = P.FreeKVConfig(n_layers=L, batch=nb, n_qo=n_qo, n_kv=n_kv, head_dim=d, page_size=p,
                     budget_tokens=c["budget"], sink_tokens=c["sink"], window_tokens=c["window"],
                     max_ctx_tokens=c["ctx"] + 4 * steps + 8)
fkv = P.FreeKV(cfg)
dev = fkv.device
seed = 99
for l in range(L):
    k, v = synth.gen_prefill(nb, n_kv, d, p, c["ctx"], c["sink"] // p, fkv.K, seed, l, device=dev)
    fkv.append_kv(l, k, v)
fkv.synchronize()
qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, l, device=dev, event_rate=0.3) for l in range(L)]
out = torch.empty(nb, n_qo, d, dtype=torch.float32, device=dev)
t = c["ctx"]
for i in range(steps):  # eager decode steps
    for l in range(L):
        q, _ = qps[l].next()
        kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, t, seed, l, device=dev)
        torch.cuda.synchronize()
        fkv.decode_step(l, q, kn, vn, out)
    t += 1
fkv.synchronize()
qb = torch.empty(L, nb, n_qo, d, dtype=torch.bfloat16, device=dev)
kb = torch.empty(L, nb, 1, n_kv, d, dtype=torch.bfloat16, device=dev)
vb = torch.empty_like(kb)
ob = torch.empty(L, nb, n_qo, d, dtype=torch.float32, device=dev)
for l in range(L):
    q, _ = qps[l].next()
    kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, t, seed, l, device=dev)
    qb[l], kb[l], vb[l] = q, kn, vn
torch.cuda.synchronize()
fkv.step_graph_capture(qb, kb, vb, ob)
for i in range(steps):  # step graph replays
    fkv.step_graph_launch()
    fkv.synchronize()
t += steps
# primitive API on layer 0
q, _ = qps[0].next()
kn, vn = synth.gen_decode_kv(nb, n_kv, d, p, t, seed, 0, device=dev)
torch.cuda.synchronize()
fkv.append_kv(0, kn, vn)
fkv.select_pages(0, q)
fkv.recall_pages(0)
fkv.sparse_decode_attn(0, q, out)
fkv.summarize_pages(0, c["sink"] // p, (t - c["window"]) // p)
fkv.synchronize()
fkv.close()
print("sanitize run ok", sys.argv[1:])
