"""Is the select kernel slow because its code is cold?  Time score + select (eager, CUDA
events around each kernel) right after streaming 256 MB through L2 (cold code and data)
and again immediately after (warm)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_13109_b200 as P
import synth

dev = torch.device("cuda", 0)
nb, nq, nk, d, p, ctx = 8, 32, 8, 128, 32, 32768
cfg = P.FreeKVConfig(n_layers=1, batch=nb, n_qo=nq, n_kv=nk, max_ctx_tokens=ctx + 64)
fkv = P.FreeKV(cfg)
s = fkv.stream
seed = synth.SEED0 + 2
with torch.cuda.stream(s):
    k, v = synth.gen_prefill(nb, nk, d, p, ctx, 16, cfg.K, seed, 0, device=dev)
    fkv.append_kv(0, k, v)
    del k, v
qp = synth.QueryProcess(nb, nq, nk, d, seed, 0, device=dev, event_rate=0.05)
q, _ = qp.next()
junk = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fkv.synchronize()
res = {}
for trial in range(6):
    for label in ("cold", "warm"):
        with torch.cuda.stream(s):
            if label == "cold":
                junk.fill_(trial)  # evict L2
            torch.cuda._sleep(2_000_000)
        fkv.profile_begin(16)
        fkv.select_pages(0, q)
        prof = fkv.profile_end()
        for kname in ("score", "select_finalize"):
            res.setdefault(f"{label}_{kname}", []).append(round(prof[kname][0] * 1e3, 2))
print(json.dumps(res))
