"""In-kernel %globaltimer timeline of one decode step of one layer (FREEKV_TRACE=1)."""
import json, os, sys
os.environ["FREEKV_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2505_13109_b200 as P
import synth

CFG = {"c2": (8, 32, 8, 128, 32, 32768), "c3": (4, 28, 4, 128, 32, 131072)}
nb, nq, nk, d, p, ctx = CFG[os.environ.get("FKV_TRACE_CFG", "c2")]
L = int(os.environ.get("FKV_TRACE_LAYERS", "2"))
cfg = P.FreeKVConfig(n_layers=L, batch=nb, n_qo=nq, n_kv=nk, max_ctx_tokens=ctx + 64)
fkv = P.FreeKV(cfg)
dev = fkv.device
seed = synth.SEED0 + 2
for l in range(L):
    k, v = synth.gen_prefill(nb, nk, d, p, ctx, 16, cfg.K, seed, l, device=dev)
    torch.cuda.synchronize()
    fkv.append_kv(l, k, v)
fkv.synchronize()
qps = [synth.QueryProcess(nb, nq, nk, d, seed, l, device=dev, event_rate=float(os.environ.get("FKV_EVENT_RATE", "0.05")))
       for l in range(L)]
out = torch.empty(nb, nq, d, dtype=torch.float32, device=dev)
GRAPH = "--graph" in sys.argv
if GRAPH:
    qb = torch.empty(L, nb, nq, d, dtype=torch.bfloat16, device=dev)
    kb = torch.empty(L, nb, 1, nk, d, dtype=torch.bfloat16, device=dev)
    vb = torch.empty_like(kb)
    ob = torch.empty(L, nb, nq, d, dtype=torch.float32, device=dev)
names = {0: "score", 1: "select", 2: "recall_sync", 3: "recall_bg", 4: "attn", 5: "attn_phase1", 6: "attn_phase2",
         7: "merge", 8: "pre", 9: "rank_phases", 10: "finalize_bg", 11: "radix_passes"}
res = {}
def steps():
    for i in range(12):
        if GRAPH:
            for l in range(L):
                q, _ = qps[l].next()
                kn, vn = synth.gen_decode_kv(nb, nk, d, p, ctx + i, seed, l, device=dev)
                qb[l], kb[l], vb[l] = q, kn, vn
            torch.cuda.synchronize()
            if i == 0:
                fkv.step_graph_capture(qb, kb, vb, ob)
            fkv.step_graph_launch()
            fkv.synchronize()
            yield i, L - 1  # the trace holds the last layer of the step
        else:
            for l in range(L):
                q, _ = qps[l].next()
                kn, vn = synth.gen_decode_kv(nb, nk, d, p, ctx + i, seed, l, device=dev)
                torch.cuda.synchronize()
                fkv.decode_step(l, q, kn, vn, out)
                fkv.synchronize()
                yield i, l


for i, l in steps():
        tr = fkv.debug_trace().astype(np.int64)
        if i < 8:
            continue
        t0 = tr[tr > 0].min()
        step = {}
        for c, nm in names.items():
            a = tr[c]
            ents = a[a[:, 0] > 0]
            if len(ents) == 0:
                continue
            rel = np.where(ents > 0, ents - t0, -1) / 1000.0  # us
            last = np.max(np.where(ents > 0, ents, 0), axis=1)
            step[nm] = {"n": int(len(ents)), "first_start_us": round(float(rel[:, 0].min()), 2),
                        "last_start_us": round(float(rel[:, 0].max()), 2),
                        "end_us": round(float((last.max() - t0) / 1000.0), 2),
                        "median_stamps_rel_start_us": [round(float(np.median(np.where(ents[:, j] > 0, ents[:, j] - ents[:, 0], np.nan)[~np.isnan(np.where(ents[:, j] > 0, ents[:, j] - ents[:, 0], np.nan))]) / 1000.0), 2) if (ents[:, j] > 0).any() else None for j in range(1, 8)],
                        "max_span_us": round(float((last - ents[:, 0]).max() / 1000.0), 2)}
        res[f"step{i}_layer{l}"] = step
        if i == 9 and "--dump" in sys.argv:  # raw stamps of this step for offline analysis
            sel = fkv.get_selection(l)
            np.savez(os.path.join(ROOT, "gpurun_out", "trace_raw.npz"), tr=tr, t0=t0, flags=sel["flags"])
print(json.dumps(res, indent=1))
