"""Timeline of the clustered attention kernel launched alone (sparse_decode_attn after select_pages,
L2 flushed), FREEKV_TRACE=1: per-warp start, page list loaded, first slab, end of its pages; per-unit
merge start / end (us relative to the first warp start)."""
import json, os, sys
os.environ["FREEKV_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2505_13109_b200 as P
import synth
CFG = {"c2": dict(nb=8, nq=32, nk=8, ctx=32768), "c3": dict(nb=4, nq=28, nk=4, ctx=131072)}
c = CFG[sys.argv[1] if len(sys.argv) > 1 else "c2"]
nb, nq, nk, d, p = c["nb"], c["nq"], c["nk"], 128, 32
cfg = P.FreeKVConfig(n_layers=1, batch=nb, n_qo=nq, n_kv=nk, max_ctx_tokens=c["ctx"] + 64)
fkv = P.FreeKV(cfg)
dev = fkv.device
s = fkv.stream
seed = synth.SEED0 + 2
k, v = synth.gen_prefill(nb, nk, d, p, c["ctx"], 16, cfg.K, seed, 0, device=dev)
torch.cuda.synchronize()
fkv.append_kv(0, k, v)
fkv.synchronize()
del k, v
qp = synth.QueryProcess(nb, nq, nk, d, seed, 0, device=dev, event_rate=0.05)
out = torch.empty(nb, nq, d, dtype=torch.float32, device=dev)
for i in range(4):
    q, _ = qp.next()
    kn, vn = synth.gen_decode_kv(nb, nk, d, p, c["ctx"] + i, seed, 0, device=dev)
    torch.cuda.synchronize()
    fkv.decode_step(0, q, kn, vn, out)
    fkv.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fkv.select_pages(0, q)
fkv.synchronize()
for rep in range(3):
    flush.fill_(1)
    torch.cuda.synchronize()
    fkv.debug_trace()
    fkv.sparse_decode_attn(0, q, out)
    fkv.synchronize()
    tr = fkv.debug_trace().astype(np.int64)
    a = tr[4]
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    rel = lambda x: np.round((x - t0) / 1e3, 2)
    mg = tr[7]
    mg = mg[mg[:, 0] > 0]
    res = {"warps": len(a), "start": [float(rel(np.percentile(a[:, 0], q_))) for q_ in (0, 50, 100)],
           "list_loaded": float(np.median(a[:, 1] - a[:, 0]) / 1e3),
           "first_slab": float(np.median(a[:, 2] - a[:, 0]) / 1e3),
           "end_attend": [float(rel(np.percentile(a[:, 3], q_))) for q_ in (0, 50, 100)],
           "merge_start": [float(rel(np.percentile(mg[:, 0], q_))) for q_ in (0, 50, 100)],
           "merge_end": [float(rel(np.percentile(mg[:, 1], q_))) for q_ in (0, 50, 100)]}
    # per SM: number of attention CTAs (warps / 4) and the mean end time of its warps
    sm = a[:, 7]
    per = {}
    for smv in np.unique(sm):
        sel = sm == smv
        per[int(smv)] = (int(sel.sum()) // 4, float(np.mean(a[sel, 3] - t0) / 1e3))
    by = {}
    for ctas, e in per.values():
        by.setdefault(ctas, []).append(e)
    res["end_by_ctas_per_sm"] = {k: (len(v), round(float(np.mean(v)), 2)) for k, v in sorted(by.items())}
    res["sms_used"] = len(per)
    print(json.dumps(res))
