"""Isolated kernel timing (one layer): score + select via select_pages and the attention via
sparse_decode_attn, each launch preceded by an L2 flush, device time from the library's event
profiler / CUDA events.  Fast A/B tool for kernel variants (FREEKV_LIB_SUFFIX=_X).

    python tools/iso_bench.py --config c2|c3 [--reps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_2505_13109_b200 as P
import synth

CFG = {"c2": dict(nb=8, nq=32, nk=8, ctx=32768), "c3": dict(nb=4, nq=28, nk=4, ctx=131072),
       "c5s": dict(nb=16, nq=8, nk=1, ctx=131072), "c1": dict(nb=1, nq=32, nk=8, ctx=4096)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--trace", action="store_true", help="in-kernel %globaltimer phases (FREEKV_TRACE=1)")
a = ap.parse_args()
if a.trace:
    os.environ["FREEKV_TRACE"] = "1"
import numpy as np
c = CFG[a.config]
nb, nq, nk, d, p = c["nb"], c["nq"], c["nk"], 128, 32
sink = 128 if a.config == "c1" else 512
budget = 512 if a.config == "c1" else 2048
cfg = P.FreeKVConfig(n_layers=1, batch=nb, n_qo=nq, n_kv=nk, max_ctx_tokens=c["ctx"] + a.steps + 8,
                     budget_tokens=budget, sink_tokens=sink, window_tokens=sink)
fkv = P.FreeKV(cfg)
dev = fkv.device
s = fkv.stream
seed = synth.SEED0 + 2
with torch.cuda.stream(s):
    k, v = synth.gen_prefill(nb, nk, d, p, c["ctx"], sink // p, cfg.K, seed, 0, device=dev)
    fkv.append_kv(0, k, v)
    del k, v
qp = synth.QueryProcess(nb, nq, nk, d, seed, 0, device=dev, event_rate=0.05)
out = torch.empty(nb, nq, d, dtype=torch.float32, device=dev)
for i in range(a.steps):
    q, _ = qp.next()
    kn, vn = synth.gen_decode_kv(nb, nk, d, p, c["ctx"] + i, seed, 0, device=dev)
    s.wait_stream(torch.cuda.current_stream())
    fkv.decode_step(0, q, kn, vn, out)
fkv.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_r = torch.ones(64 << 20, dtype=torch.float32, device=dev)
acc = torch.empty((), dtype=torch.float32, device=dev)
fkv.profile_begin(4 * a.reps + 8)
with torch.cuda.stream(s):
    torch.cuda._sleep(2_000_000)
    for _ in range(a.reps):
        flush.fill_(1)
        torch.sum(flush_r, dim=0, out=acc)
        fkv.select_pages(0, q, stream=s)
prof = fkv.profile_end()
phases = {}
if a.trace:
    # one more select_pages after a flush, alone; per-CTA stamps of the score (class 0) and select (1)
    fkv.debug_trace()
    with torch.cuda.stream(s):
        flush.fill_(1)
        torch.sum(flush_r, dim=0, out=acc)
        fkv.select_pages(0, q, stream=s)
    tr = fkv.debug_trace().astype(np.int64)
    for cls, nm in ((0, "score"), (1, "select")):
        e = tr[cls]
        e = e[e[:, 0] > 0]
        if len(e) == 0:
            continue
        t0 = e[:, 0].min()
        ph = {"ctas": int(len(e)), "start_spread_us": round(float((e[:, 0].max() - t0) / 1e3), 2)}
        for j in range(1, 8):
            ok = e[:, j] > 0
            if ok.any():
                ph[f"med_stamp{j}_us"] = round(float(np.median(e[ok, j] - e[ok, 0]) / 1e3), 2)
                ph[f"max_stamp{j}_us"] = round(float(np.max(e[ok, j] - t0) / 1e3), 2)
        if cls == 0 and False:  # FKV_SC_CLK builds: SM cycles between stamps 1 and 2
            ok = (e[:, 5] > 0) & (e[:, 2] > e[:, 1])
            ph["sm_mhz_in_loop"] = round(float(np.median(e[ok, 5] / ((e[ok, 2] - e[ok, 1]) / 1e3))), 1)
        phases[nm] = ph
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
with torch.cuda.stream(s):
    torch.cuda._sleep(2_000_000)
    for ea, eb in evs:
        flush.fill_(1)
        torch.sum(flush_r, dim=0, out=acc)
        ea.record(s)
        fkv.sparse_decode_attn(0, q, out, stream=s)
        eb.record(s)
s.synchronize()
att = sorted(ea.elapsed_time(eb) * 1e3 for ea, eb in evs)
res = {k: round(v[0] / v[1] * 1e3, 2) for k, v in prof.items() if v[1]}
res["attn_us_median"] = round(att[len(att) // 2], 2)
if phases:
    res["phases"] = phases
res["lib"] = os.environ.get("FREEKV_LIB_SUFFIX", "")
res["config"] = a.config
print(json.dumps(res))
