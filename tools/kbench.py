"""Kernel micro-bench at c2 (Llama-3.1-8B shape, 32K ctx, batch 8) with few layers:
per-kernel device time from the library's event profiler.  Used for fast
build -> measure iterations and as the ncu target."""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_13109_b200 as P
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--n_qo", type=int, default=32)
ap.add_argument("--n_kv", type=int, default=8)
ap.add_argument("--event_rate", type=float, default=0.05)
ap.add_argument("--tau", type=float, default=0.8)
ap.add_argument("--mode", type=int, default=0, help="0 speculative, 1 always correct, 2 never correct")
ap.add_argument("--pool", type=int, default=0, help="FREEKV_POOL_* group pooling (f3)")
ap.add_argument("--corr_pool", type=int, default=0)
ap.add_argument("--no-profile", action="store_true")
ap.add_argument("--graph", action="store_true", help="whole-step graph replay with in-graph event profiling")
a = ap.parse_args()
dev = torch.device("cuda", 0)
nb, nq, nk, d, p = a.batch, a.n_qo, a.n_kv, 128, 32
G = nq // nk
cfg = P.FreeKVConfig(n_layers=a.layers, batch=nb, n_qo=nq, n_kv=nk, max_ctx_tokens=a.ctx + a.warmup + a.steps + 2,
                     tau=a.tau, mode=a.mode, pool=a.pool, corr_pool=a.corr_pool)
fkv = P.FreeKV(cfg)
s = fkv.stream
seed = synth.SEED0 + 2
with torch.cuda.stream(s):
    for l in range(a.layers):
        k, v = synth.gen_prefill(nb, nk, d, p, a.ctx, 16, cfg.K, seed, l, device=dev)
        fkv.append_kv(l, k, v)
        del k, v
    qps = [synth.QueryProcess(nb, nq, nk, d, seed, l, device=dev, event_rate=a.event_rate) for l in range(a.layers)]
    T = a.warmup + a.steps
    Q = torch.empty(T, a.layers, nb, nq, d, dtype=torch.bfloat16, device=dev)
    Kn = torch.empty(T, a.layers, nb, 1, nk, d, dtype=torch.bfloat16, device=dev)
    Vn = torch.empty_like(Kn)
    for i in range(T):
        for l in range(a.layers):
            q, _ = qps[l].next()
            kn, vn = synth.gen_decode_kv(nb, nk, d, p, a.ctx + i, seed, l, device=dev)
            Q[i, l], Kn[i, l], Vn[i, l] = q, kn, vn
out = torch.empty(nb, nq, d, dtype=torch.float32, device=dev)
s.synchronize()
for i in range(a.warmup):
    for l in range(a.layers):
        fkv.decode_step(l, Q[i, l], Kn[i, l], Vn[i, l], out)
fkv.synchronize()
if a.graph:
    qb, kb, vb = torch.empty_like(Q[0]), torch.empty_like(Kn[0]), torch.empty_like(Vn[0])
    ob = torch.empty(a.layers, nb, nq, d, dtype=torch.float32, device=dev)
    fkv.step_graph_capture(qb, kb, vb, ob, profile=not a.no_profile)
    acc = {}
    tot = 0.0
    for i in range(a.warmup, T):
        with torch.cuda.stream(s):
            qb.copy_(Q[i]); kb.copy_(Kn[i]); vb.copy_(Vn[i])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fkv.step_graph_launch()
        e1.record(s)
        fkv.synchronize()
        tot += e0.elapsed_time(e1)
        if not a.no_profile:
            for k, (t, n) in fkv.step_graph_profile().items():
                x = acc.setdefault(k, [0.0, 0])
                x[0] += t
                x[1] += n
    res = {"us_per_layer_graph_synced": tot * 1e3 / (a.steps * a.layers)}
    res["kernels_us_in_graph"] = {k: round(v[0] / max(v[1], 1) * 1e3, 2) for k, v in acc.items()}
    print(json.dumps(res))
    sys.exit(0)
if not a.no_profile:
    fkv.profile_begin(a.steps * a.layers * 8 + 16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for i in range(a.warmup, T):
    for l in range(a.layers):
        fkv.decode_step(l, Q[i, l], Kn[i, l], Vn[i, l], out)
e1.record(s)
fkv.synchronize()
res = {"us_per_layer": e0.elapsed_time(e1) * 1e3 / (a.steps * a.layers)}
if not a.no_profile:
    prof = fkv.profile_end()
    res["kernels_us"] = {k: round(v[0] / max(v[1], 1) * 1e3, 2) for k, v in prof.items()}
print(json.dumps(res))
