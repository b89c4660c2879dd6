"""Device-side cost of back-to-back dependent tiny kernels on this GPU (graph-replayed)."""
import torch, json
x = torch.zeros(1, device="cuda")
y = torch.zeros(1 << 20, device="cuda")
s = torch.cuda.Stream()
res = {}
for name, fn in [("tiny_1cta", lambda: x.add_(1)), ("fill_4MiB", lambda: y.add_(1))]:
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(100): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10): g.replay()
    e1.record(s); torch.cuda.synchronize()
    res[name + "_us_per_kernel_graph"] = e0.elapsed_time(e1) * 1e3 / 1000
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(1000): fn()
    e1.record(s); torch.cuda.synchronize()
    res[name + "_us_per_kernel_eager"] = e0.elapsed_time(e1) * 1e3 / 1000
print(json.dumps(res))
