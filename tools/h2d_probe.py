#!/usr/bin/env python
"""PCIe / host-memory probe for the e2e arm: pinned H2D and D2H bandwidth (torch), repeated,
with the process's CPU affinity and the GPU's local CPU list, to explain e2e variance."""
import json
import os
import time

import torch


def gpu_local_cpus(dev=0):
    try:
        bus = torch.cuda.get_device_properties(dev).pci_bus_id
    except Exception:
        return None
    try:
        import subprocess
        out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                             capture_output=True, text=True).stdout.strip().splitlines()
        bus = out[dev].strip().lower()
        bus = bus[4:] if len(bus.split(":")[0]) == 8 else bus
        path = f"/sys/bus/pci/devices/{bus}/local_cpulist"
        return open(path).read().strip()
    except Exception as e:
        return f"unknown ({e})"


def bw(n_bytes=1 << 30, reps=5, direction="h2d"):
    h = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n_bytes, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        if direction == "h2d":
            d.copy_(h, non_blocking=True)
        else:
            h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        out.append(n_bytes / (time.perf_counter() - t0) / 1e9)
    return out


def main():
    res = {"affinity": sorted(os.sched_getaffinity(0))[:64], "n_cpus": os.cpu_count(),
           "gpu_local_cpulist": gpu_local_cpus()}
    res["h2d_gbs"] = bw()
    res["d2h_gbs"] = bw(direction="d2h")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
