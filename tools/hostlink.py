"""P0 box facts: pinned host<->device copy peaks. Writes JSON to stdout."""
import json, os, subprocess, sys, time
import torch

def best_copy(dst, src, reps=10):
    s = torch.cuda.current_stream()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s); dst.copy_(src, non_blocking=True); b.record(s); b.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return src.numel() * src.element_size() / best / 1e9

def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

def main():
    n = 1 << 30
    t0 = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    t_pin = time.time() - t0
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h.fill_(1)
    out = {
        "h2d_gbs_1gib": best_copy(d, h),
        "d2h_gbs_1gib": best_copy(h, d),
        "pin_1gib_s": t_pin,
        "nproc": os.cpu_count(),
        "gpu": torch.cuda.get_device_name(0),
    }
    for sz in [16 << 10, 256 << 10, 1 << 20, 16 << 20]:
        out[f"h2d_gbs_{sz>>10}KiB"] = best_copy(d[:sz], h[:sz], reps=50)
    print(json.dumps(out))
    print(sh("free -g; lscpu | head -30; nvidia-smi topo -m; nvidia-smi -q | grep -iE 'pcie|link' | head -20; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c"))

if __name__ == "__main__":
    main()
