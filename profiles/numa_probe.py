"""PCIe copy bandwidth from pinned host memory by NUMA placement (the e2e path's floor).

    python profiles/numa_probe.py

For the CPU set NVML reports as local to GPU 0, the remaining CPUs, and no restriction: pin the
process there, allocate and first-touch 400 MB of pinned host memory (its pages land on that
node), then time H2D, D2H and both directions at once.
"""
import os
import sys

import torch

try:
    import pynvml
except ImportError:  # pragma: no cover
    pynvml = None


def local_cpus(index=0):
    if pynvml is None:
        return None
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(index)
    n = os.cpu_count()
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
    cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
    return [c for c in cpus if c < n]


def bw(nbytes=400 << 20, reps=5):
    host_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    host_in.fill_(1)  # first touch from this (pinned) thread
    host_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    host_out.fill_(0)
    dev_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dev_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    res = {}
    for mode in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        e[0].record(s1)
        s2.wait_event(e[0])
        for _ in range(reps):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    dev_a.copy_(host_in, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    host_out.copy_(dev_b, non_blocking=True)
        e[1].record(s1)
        e[2].record(s2)
        torch.cuda.synchronize()
        ms = max(e[0].elapsed_time(e[1]), e[0].elapsed_time(e[2]))
        res[mode] = nbytes * reps / (ms * 1e-3) / 1e9
    return res


if __name__ == "__main__":
    n = os.cpu_count()
    loc = local_cpus()
    print(f"cpus {n}; NVML local to GPU 0: {loc}", flush=True)
    sets = [("all", list(range(n)))]
    if loc and len(loc) < n:
        sets += [("gpu-local", loc), ("remote", [c for c in range(n) if c not in loc])]
    for name, cpus in sets:
        os.sched_setaffinity(0, cpus)
        r = bw()
        print(f"{name:10s} H2D {r['h2d']:.1f} GB/s  D2H {r['d2h']:.1f} GB/s  both {r['both']:.1f} GB/s (each way)", flush=True)
    sys.exit(0)
