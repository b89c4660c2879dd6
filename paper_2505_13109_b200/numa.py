"""NUMA-local pinned host shards (each GPU's host pool on its own NUMA node).

cudaHostAlloc'd pages are placed by the kernel's default local-allocation policy on the node of
the CPU that first touches them (the allocating thread).  Binding the process to the CPUs of the
GPU's NUMA node before the pool is allocated therefore pins it node-locally; the binding is kept
for the host-side work (the per-step input staging) as well.
"""
from __future__ import annotations

import os


def _pci_bus_id(device_index: int) -> str | None:
    try:
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(device_index)
        bid = N.nvmlDeviceGetPciInfo(h).busId
        bid = bid.decode() if isinstance(bid, bytes) else bid
        # NVML: "00000000:1B:00.0" -> sysfs "0000:1b:00.0"
        dom, rest = bid.split(":", 1)
        return f"{int(dom, 16):04x}:{rest.lower()}"
    except Exception:  # noqa: BLE001
        return None


def _parse_cpulist(s: str) -> list[int]:
    cpus = []
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.extend(range(int(a), int(b) + 1))
        else:
            cpus.append(int(part))
    return cpus


def bind_to_gpu_node(device_index: int) -> dict:
    """Bind this process to the CPUs of the GPU's NUMA node; returns what was done (for the
    bench line).  No-op (reported) where sysfs / NVML give no node."""
    bus = _pci_bus_id(device_index)
    if not bus:
        return {"node": None, "note": "no PCI bus id (NVML unavailable)"}
    base = f"/sys/bus/pci/devices/{bus}"
    try:
        node = int(open(f"{base}/numa_node").read().strip())
    except Exception:  # noqa: BLE001
        return {"node": None, "note": f"no numa_node for {bus}"}
    if node < 0:
        return {"node": None, "note": f"{bus}: single NUMA domain (numa_node = -1)"}
    try:
        cpus = _parse_cpulist(open(f"/sys/devices/system/node/node{node}/cpulist").read())
        allowed = os.sched_getaffinity(0)
        cpus = [c for c in cpus if c in allowed]
        if cpus:
            os.sched_setaffinity(0, cpus)
        return {"node": node, "cpus": len(cpus), "pci": bus}
    except Exception as e:  # noqa: BLE001
        return {"node": node, "note": f"affinity not set: {e}"}
