"""Phase timeline of the fused layer kernel (FREEKV_TRACE=1), one layer in isolation at a BASELINE
config shape: per CTA stamps 0 start, 1 after the correction check + append, 2 after the scoring,
3 after the ranking, 4 after the delta, 5 after the attention + merge, 6 end; medians split by
corrected / not corrected units (relative to stamp 1 of the same CTA)."""
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
seed = synth.SEED0 + 2
k, v = synth.gen_prefill(nb, nk, d, p, c["ctx"], 16, cfg.K, seed, 0, device=dev)
torch.cuda.synchronize()
fkv.append_kv(0, k, v)
fkv.synchronize()
del k, v
qp = synth.QueryProcess(nb, nq, nk, d, seed, 0, device=dev, event_rate=0.2)
out = torch.empty(nb, nq, d, dtype=torch.float32, device=dev)
C = None
for i in range(10):
    q, _ = qp.next()
    kn, vn = synth.gen_decode_kv(nb, nk, d, p, c["ctx"] + i, seed, 0, device=dev)
    torch.cuda.synchronize()
    fkv.debug_trace()
    fkv.decode_step(0, q, kn, vn, out)
    fkv.synchronize()
    trall = fkv.debug_trace().astype(np.int64)
    tr = trall[4]
    rk = trall[9]
    fl = fkv.get_selection(0)["flags"].astype(bool)
    if i < 6:
        continue
    ent = tr[tr[:, 0] > 0]
    n = len(ent)
    C = n // fkv.U
    t0 = ent[:, 0].min()
    res = {"ctas": n, "ctas_per_unit": C, "corrected_units": int(fl.sum()), "start_spread_us": round((ent[:, 0].max() - t0) / 1e3, 2),
           "end_us": round((ent[:, 6].max() - t0) / 1e3, 2)}
    for name, sel in (("not_corrected", ~fl), ("corrected", fl)):
        rows = ent[np.repeat(sel, C)[:n]]
        if len(rows) == 0:
            continue
        ph = {}
        for j in range(2, 7):
            ok = rows[:, j] > 0
            if ok.any():
                ph[f"s{j}"] = round(float(np.median(rows[ok, j] - rows[ok, 1])) / 1e3, 2)
        ph["s1_from_start"] = round(float(np.median(rows[:, 1] - rows[:, 0])) / 1e3, 2)
        rr = rk[:n][np.repeat(sel, C)[:n]]
        rr = rr[rr[:, 0] > 0]
        if len(rr):
            ph["rank_phases_us"] = [round(float(np.median(rr[:, j] - rr[:, j - 1])) / 1e3, 2) for j in range(1, 8)]
        res[name] = ph
    print(json.dumps(res))
