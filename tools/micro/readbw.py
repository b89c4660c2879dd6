"""HBM read bandwidth reference points (CUDA events, best of N): a plain reduction over a large
buffer (read-only stream) and over 67 MB / 33 MB (one layer's attention / score traffic at c2),
L2 flushed before each rep."""
import json
import torch

dev = "cuda"
big = torch.ones(1 << 30, dtype=torch.bfloat16, device=dev)  # 2 GiB
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
for name, n in (("sum_2GiB", 1 << 30), ("sum_67MB", 67616768 // 2), ("sum_33MB", 32702464 // 2)):
    x = big[:n]
    best = 1e9
    for _ in range(10):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.sum(x, dtype=torch.float32)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3)
    res[name] = {"us": round(best, 2), "gbs": round(n * 2 / best / 1e3, 1)}
print(json.dumps(res))
