"""Pinned H2D bandwidth of a 512 MB buffer, with and without the process
pinned to the GPU's local CPUs (NUMA placement of the page-locked memory)."""
import os
import sys
import time

import torch

pr = torch.cuda.get_device_properties(0)
bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
path = f"/sys/bus/pci/devices/{bus}/local_cpulist"
local = open(path).read().strip() if os.path.exists(path) else None
print("gpu", bus, "local cpus", local, "numa", open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip()
      if os.path.exists(f"/sys/bus/pci/devices/{bus}/numa_node") else "?")


def cpus(spec):
    out = set()
    for part in spec.split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out


def bw(tag):
    x = torch.empty(128 << 20, dtype=torch.float32).pin_memory()
    x.fill_(1.0)
    d = torch.empty_like(x, device="cuda")
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(x, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{tag}: {x.numel() * 4 / dt / 1e9:.1f} GB/s")


bw("default affinity")
if local:
    os.sched_setaffinity(0, cpus(local))
    bw("gpu-local affinity")
