"""Model stand-in decode loop: the FreeKV path inside a decode step with
real-shape projections and FFN.

Each layer of the step runs, on the path's compute stream,
  RMSNorm -> QKV projection -> FreeKV decode step (append, correction, select, attention,
  background recall) -> O projection + residual -> RMSNorm -> gate/up -> SiLU*up -> down + residual
with random bf16 weights of the model's shape (cuBLAS GEMMs through torch; there are no trained
weights, so accuracy is out of scope).  The projections' q/k/v values are merged into the
synthetic GEN-Q / GEN-S inputs by a dependent elementwise op (q_in = q_syn + 0 * q_proj), so
every data dependency of a real layer is kept while the correction rate stays the workload's
(random weights would make consecutive queries uncorrelated: every unit corrected every step).
The projection and FFN segments of each layer are CUDA graphs (host launch cost out of the
way); the FreeKV step is its C-ABI call.  This is the paper's overlap window: the
background recall of layer l runs during the GEMMs of layers l..l+k.

Three variants, device time with CUDA events on the compute stream, L2 not flushed (weights
of 32 layers, 14 GB, stream through it every step):
  gemm   -- the stand-in layers without the FreeKV step (attention output left constant)
  model  -- the full stand-in decode step
  path   -- the FreeKV steps alone (same eager per-layer calls)
exposed = (model - gemm) per layer is what the path adds to a real decode step.

usage: python tools/model_standin.py [--config c2] [--steps 32] [--warmup 4]   (one JSON line)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MODEL = {  # hidden, ffn (the attention shape comes from the bench config)
    "c1": dict(hidden=4096, ffn=14336, name="llama3.1-8b"),
    "c2": dict(hidden=4096, ffn=14336, name="llama3.1-8b"),
    "c3": dict(hidden=3584, ffn=18944, name="qwen2.5-7b"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--warmup", type=int, default=4)
    args = ap.parse_args()
    import torch
    import torch.nn.functional as F

    import bench
    import paper_2505_13109_b200 as P
    import synth

    c = bench.CONFIGS[args.config]
    m = MODEL[args.config]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n_kv, n_qo, nb, d, L, p = c["n_kv"], c["n_qo"], c["batch"], 128, c["n_layers"], 32
    H, FF = m["hidden"], m["ffn"]
    seed = synth.SEED0 + 1 + list(bench.CONFIGS).index(args.config)
    n_dec = 2 * (args.warmup + args.steps)  # decode steps the handle advances (path + model variants)
    stream = torch.cuda.Stream(dev, priority=-1)
    cfg, fkv = bench.build_handle(P, c, n_kv, n_qo, c["ctx"] + n_dec + 1, stream)
    with torch.cuda.stream(stream):
        for layer in range(L):
            k, v = synth.gen_prefill(nb, n_kv, d, p, c["ctx"], c["sink"] // p, cfg.K, seed, layer, device=dev)
            fkv.append_kv(layer, k, v)
            del k, v
    # step inputs (GEN-Q queries, GEN-S new tokens), generated outside the timed regions
    qps = [synth.QueryProcess(nb, n_qo, n_kv, d, seed, layer, device=dev, event_rate=c["event_rate"])
           for layer in range(L)]
    Qs = torch.empty(n_dec, L, nb, n_qo, d, dtype=torch.bfloat16, device=dev)
    Ks = torch.empty(n_dec, L, nb, 1, n_kv, d, dtype=torch.bfloat16, device=dev)
    Vs = torch.empty_like(Ks)
    with torch.cuda.stream(stream):
        for i in range(n_dec):
            for layer in range(L):
                Qs[i, layer] = qps[layer].next()[0]
                Ks[i, layer], Vs[i, layer] = synth.gen_decode_kv(nb, n_kv, d, p, c["ctx"] + i, seed, layer, device=dev)
    # random weights of the model's shape (bf16), scaled to keep activations O(1)
    gen = torch.Generator(device=dev).manual_seed(seed)

    def w(i, o):
        return (torch.randn(i, o, generator=gen, device=dev, dtype=torch.float32) * (i ** -0.5)).to(torch.bfloat16)

    qkv_n = (n_qo + 2 * n_kv) * d
    Wqkv = [w(H, qkv_n) for _ in range(L)]
    Wo = [w(n_qo * d, H) for _ in range(L)]
    Wgu = [w(H, 2 * FF) for _ in range(L)]
    Wd = [w(FF, H) for _ in range(L)]
    ln1 = torch.ones(H, dtype=torch.bfloat16, device=dev)
    ln2 = torch.ones(H, dtype=torch.bfloat16, device=dev)
    weight_bytes = sum(t.numel() * 2 for t in Wqkv + Wo + Wgu + Wd)
    # static buffers of the captured segments
    x = torch.randn(nb, H, device=dev).to(torch.bfloat16)
    x0 = x.clone()
    q_src = torch.empty(L, nb, n_qo, d, dtype=torch.bfloat16, device=dev)
    k_src = torch.empty(L, nb, 1, n_kv, d, dtype=torch.bfloat16, device=dev)
    v_src = torch.empty_like(k_src)
    q_in, k_in, v_in = torch.empty_like(q_src), torch.empty_like(k_src), torch.empty_like(v_src)
    out = torch.zeros(L, nb, n_qo, d, dtype=torch.float32, device=dev)
    zero = torch.zeros((), dtype=torch.bfloat16, device=dev)

    def seg1(l):  # RMSNorm -> QKV projection -> path inputs (dependent on the projection)
        h = F.rms_norm(x, (H,), ln1, 1e-5)
        qkv = h @ Wqkv[l]
        torch.addcmul(q_src[l], qkv[:, :n_qo * d].view(nb, n_qo, d), zero, out=q_in[l])
        torch.addcmul(k_src[l], qkv[:, n_qo * d:(n_qo + n_kv) * d].view(nb, 1, n_kv, d), zero, out=k_in[l])
        torch.addcmul(v_src[l], qkv[:, (n_qo + n_kv) * d:].view(nb, 1, n_kv, d), zero, out=v_in[l])

    def seg2(l):  # O projection + residual, FFN + residual
        o = out[l].view(nb, n_qo * d).to(torch.bfloat16)
        x.add_(o @ Wo[l])
        h = F.rms_norm(x, (H,), ln2, 1e-5)
        gu = h @ Wgu[l]
        x.add_((F.silu(gu[:, :FF]) * gu[:, FF:]) @ Wd[l])

    g1, g2 = [], []
    with torch.cuda.stream(stream):
        for l in range(L):  # warm the kernels (cuBLAS handles, workspaces) before capture
            seg1(l)
            seg2(l)
    stream.synchronize()
    for l in range(L):
        for seg, gl in ((seg1, g1), (seg2, g2)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                seg(l)
            gl.append(g)
    torch.cuda.synchronize()

    state = {"i": 0}

    def stage(i):
        with torch.cuda.stream(stream):
            q_src.copy_(Qs[i], non_blocking=True)
            k_src.copy_(Ks[i], non_blocking=True)
            v_src.copy_(Vs[i], non_blocking=True)

    def step_model(with_path):
        i = state["i"]
        stage(i)
        with torch.cuda.stream(stream):
            for l in range(L):
                g1[l].replay()
                if with_path:
                    fkv.decode_step(l, q_in[l], k_in[l], v_in[l], out[l])
                g2[l].replay()
        if with_path:
            state["i"] += 1

    def step_path():
        i = state["i"]
        for l in range(L):
            fkv.decode_step(l, Qs[i, l], Ks[i, l], Vs[i, l], out[l])
        state["i"] += 1

    def timed(fn, n, warm):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n  # ms per step

    t0 = time.time()
    ms_path = timed(step_path, args.steps, args.warmup)
    ms_gemm = timed(lambda: step_model(False), args.steps, args.warmup)
    ms_model = timed(lambda: step_model(True), args.steps, args.warmup)
    finite = bool(torch.isfinite(x).all().item()) and bool(torch.isfinite(out).all().item())
    line = {
        "metric": "model stand-in decode step (f4)", "config": {"workload": c["workload"], "model": m["name"],
                                                                 "hidden": H, "ffn": FF, "layers": L, "batch": nb,
                                                                 "weights": "random bf16", "weight_bytes": weight_bytes},
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": {"model": round(ms_model, 4), "gemm_only": round(ms_gemm, 4), "path_only": round(ms_path, 4)},
        "tokens_per_s": {"model": round(nb / (ms_model / 1e3), 2), "gemm_only": round(nb / (ms_gemm / 1e3), 2)},
        "us_per_layer": {"model": round(ms_model / L * 1e3, 2), "gemm_only": round(ms_gemm / L * 1e3, 2),
                         "path_only": round(ms_path / L * 1e3, 2),
                         "path_exposed": round((ms_model - ms_gemm) / L * 1e3, 2)},
        "gemm_weight_stream_gbs": round(weight_bytes / (ms_gemm / 1e3) / 1e9, 1),
        "finite": finite, "wall_s": round(time.time() - t0, 1),
        "note": "projections' values merged into GEN-Q/GEN-S inputs (q_in = q_syn + 0*q_proj); eager per-layer "
                "FreeKV calls between captured projection/FFN segments; device time, CUDA events",
    }
    del x0
    print(json.dumps(line))


if __name__ == "__main__":
    main()
