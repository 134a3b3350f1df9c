#!/usr/bin/env python
"""Benchmark of the SLA hot path (BASELINE.json metric: "SLA fwd+bwd ms and dense-equiv
TFLOPS, Wan2.1-1.3B shape N~32K d=128").

One step = dynamic classification + fused forward + fused backward (sla_forward ->
combine_outputs -> proj_backward -> sla_backward in the reference's terms) over the C3
workload: B=1, H=12, N=32768 (32760 padded to a multiple of 64), d=128,
b_q=b_kv=64, k_h=5 %, k_l=10 %, phi=softmax, bf16 inputs with fp32 accumulation.

  python bench.py [--gpus N --steps K --warmup W]            our CUDA path (1 JSON line)
  python bench.py --impl reference [...]                      the reference's CPU path

Multi-GPU: one process per GPU (torchrun); the (batch x head) units shard with no
collective on the data path -- every rank runs its own C3 batch element (weak scaling);
timing is the max over ranks of CUDA-event time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # name: (B, H, N, d, b, k_h, k_l, phi)
    "c3": (1, 12, 32768, 128, 64, 5.0, 10.0, "softmax"),
    "c1": (1, 2, 1024, 64, 64, 5.0, 10.0, "softmax"),
    "c5": (8, 40, 75648, 128, 64, 5.0, 10.0, "softmax"),
    # the literal Wan2.1-1.3B length through SLA_B200_FLAG_RAGGED (the reference rejects it)
    "c3r": (1, 12, 32760, 128, 64, 5.0, 10.0, "softmax"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=12)
    return ap.parse_args()


def dense_equiv_flops(B, H, N, d):
    """FLOPS = O(full attention)/t; fwd 4 N^2 d + bwd 10 N^2 d per unit."""
    return 14.0 * N * N * d * B * H


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) is polled every ~2 ms from a thread, so even a ~70 ms timed region
    yields dozens of samples; `nvidia-smi -lms 100` (the fallback) needs >100 ms to emit its
    first line and missed short regions entirely."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.stop = threading.Event()
        self.t = None
        self.mx = None
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.idx)
            self.mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))

            def poll():
                while not self.stop.is_set():
                    try:
                        self.samples.append((float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                                             int(N.nvmlDeviceGetCurrentClocksEventReasons(h))))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap,utilization.gpu")
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
                     "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=lambda: self.lines.extend(l.strip() for l in self.proc.stdout),
                                          daemon=True)
                self.t.start()
            except Exception:
                self.proc = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        elif self.t:
            self.t.join(timeout=1)

    def summary(self):
        sm, reasons = [], set()
        mx = self.mx or 0.0
        for f, bits in self.samples:
            sm.append(f)
            for name, bit in self.REASONS.items():
                if bits & bit:
                    reasons.add(name)
        for ln in self.lines:  # nvidia-smi fallback
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                f, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            mx = max(mx, m)
            sm.append(f)
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                                 parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.samples else "nvidia-smi"}


# ---------------------------------------------------------------------------------------
# reference arm / cpu baseline: the reference's own CPU path (oracle/_ref)
# ---------------------------------------------------------------------------------------
def reference_step_inputs(N, d, seed=1234):
    from oracle import oracle as O

    rng = O.Rng(seed)
    bf = O.to_bf16_exact
    return dict(q=bf(rng.gaussian(N, d)), k=bf(rng.gaussian(N, d)), v=bf(rng.gaussian(N, d)),
                w=bf(rng.gaussian(d, d, 0.1)), do=bf(rng.gaussian(N, d)))


def time_reference_head(cfg, threads, x=None):
    """One (batch, head) unit of the workload through the reference's public API:
    sla_forward -> combine_outputs -> proj_backward -> sla_backward (f32)."""
    from oracle import oracle as O

    B, H, N, d, b, k_h, k_l, phi = cfg
    x = x or reference_step_inputs(N, d)
    t0 = time.perf_counter()
    if O.Reference.available():
        O.Reference.run(x["q"], x["k"], x["v"], b, b, k_h, k_l, phi, threads=threads, w=x["w"],
                        d_out=x["do"], dtype=np.float32)
        kind = "reference"
    else:  # the C restatement, single thread
        lab = O.dynamic_labels(x["q"], x["k"], b, b, k_h, k_l)
        O.step(x["q"], x["k"], x["v"], x["w"], x["do"], lab, b, b, phi)
        kind, threads = "port", 1
    return time.perf_counter() - t0, kind, threads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    B, H, N, d, b, k_h, k_l, phi = cfg
    if N % b:  # the reference rejects ragged N (layout.cpp:12-17): time the padded length
        N = (N + b - 1) // b * b
        cfg = (B, H, N, d, b, k_h, k_l, phi)
    threads = os.cpu_count() or 1
    x = reference_step_inputs(N, d)
    for _ in range(args.warmup):
        time_reference_head(cfg, threads, x)
    times = []
    kind = "reference"
    for _ in range(args.steps):
        t, kind, threads = time_reference_head(cfg, threads, x)
        times.append(t)
    per_head = sum(times) / len(times)
    flops = dense_equiv_flops(1, 1, N, d)
    value = flops / per_head / 1e12
    sample = f"one (batch, head) unit of {B * H} per step, fwd+bwd, f32, threads={threads}"
    out = {
        "impl": "reference", "metric": "SLA fwd+bwd dense-equiv TFLOPS (Wan2.1-1.3B shape)",
        "value": value, "unit": "TFLOPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_head * 1e3 * B * H, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_json(args.config),
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ms_per_head": per_head * 1e3,
    }
    print(json.dumps(out), flush=True)


def config_json(name):
    B, H, N, d, b, k_h, k_l, phi = CONFIGS[name]
    return {"workload": f"{name}: SLA fwd+bwd, B={B} H={H} N={N} d={d} b_q=b_kv={b} k_h={k_h}% k_l={k_l}% phi={phi}",
            "batch": B, "heads": H, "n": N, "d": d, "block": b, "k_h": k_h, "k_l": k_l, "phi": phi,
            "n_note": ("N = 32760 as-is through SLA_B200_FLAG_RAGGED (zero-padded unit copies inside the "
                       "timed region); the reference arm times N = 32768") if N % b else
                      "N padded from 32760/75600 to a multiple of 64 (make_block_layout rejects ragged N)",
            "l2": "inputs (Q,K,V,dO = 4 x B*H*N*d*2 bytes) exceed the 126 MB L2; no flush needed",
            "parallelism": "(batch x head) units sharded over ranks, no collective"}


# ---------------------------------------------------------------------------------------
# our CUDA path
# ---------------------------------------------------------------------------------------
def algorithmic_work(name, D, labels_stats):
    """(kind, units per launch) of a kernel's algorithmic work for the roofline:
    critical-tile FLOPs for attention kernels, bytes for the HBM-bound ones."""
    B, H, N, d, b = D["B"], D["H"], D["N"], D["d"], D["b"]
    crit = labels_stats["critical_blocks"]  # total over all units
    tile = b * b * d
    if name in ("k_fwd_generic", "k_attn_fwd"):       # S = QK^T, O += PV
        return "tensor", 4.0 * tile * crit
    if name in ("k_bwd_rows_sparse", "k_bwd_rows"):    # S, dP recomputed, dQ += dS K
        return "tensor", 6.0 * tile * crit
    if name in ("k_bwd_cols_sparse", "k_bwd_cols"):    # S, dP recomputed, dV += P^T dO, dK += dS^T Q
        return "tensor", 8.0 * tile * crit
    if name in ("k_pool(q)", "k_pool(k)"):
        return "hbm", B * H * N * d * 2.0
    return None, None


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2509_24006_b200 import SLA, HostTrainStep, SlaConfig
    from paper_2509_24006_b200 import _lib as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B, H, N, d, b, k_h, k_l, phi = CONFIGS[args.config]
    cfg = SlaConfig(k_h=k_h, k_l=k_l, phi=phi, ragged=N % b != 0)
    op = SLA(B, H, N, d, b, b, cfg, torch.bfloat16, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    shape = (B, H, N, d)
    mk = lambda s=1.0: (torch.randn(shape, generator=g, device=dev) * s).to(torch.bfloat16)  # noqa: E731
    q, k, v, do = mk(), mk(), mk(), mk()
    w = (torch.randn((H, d, d), generator=g, device=dev) * 0.1).to(torch.bfloat16)
    st_buf = op.new_state()
    o, o_s, o_l = (torch.empty(shape, dtype=torch.bfloat16, device=dev) for _ in range(3))
    lse = torch.empty(shape[:-1], dtype=torch.float32, device=dev)
    dq, dk, dv = (torch.empty(shape, dtype=torch.bfloat16, device=dev) for _ in range(3))
    dw = torch.empty((H, d, d), dtype=torch.float32, device=dev)
    launches = [0]

    def step():
        st = op.forward(q, k, v, w, state=st_buf, out=(o, o_s, o_l, lse))
        n1 = op.launches()
        op.backward(st, q, k, v, w, do, out=(dq, dk, dv, dw))
        launches[0] += n1 + op.launches()
        return st

    for _ in range(args.warmup):
        st = step()
    torch.cuda.synchronize()
    labels = st.labels.cpu()
    lab_stats = {"critical_blocks": int((labels == 1).sum()), "marginal_blocks": int((labels == 0).sum())}
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches[0] = 0
    L.lib().sla_b200_profiler(1)
    with Clocks(local) as clk:  # clocks sampled over both timed passes
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / args.steps
        buf = C.create_string_buffer(1 << 16)
        L.lib().sla_b200_profiler_report(buf, 1 << 16)
        L.lib().sla_b200_profiler(0)
        kernels = {}
        for ln in buf.value.decode().splitlines():
            nm, t, cnt = ln.rsplit(" ", 2)
            kernels[nm] = (float(t), int(cnt))
        # clean timing pass without profiler events (the headline number; the library's side
        # streams run only when its per-kernel profiler is off)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        ms_clean = ev0.elapsed_time(ev1) / args.steps
    ms = min(ms, ms_clean) if ms_clean > 0 else ms
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_max = float(t.item())
    flops_step = dense_equiv_flops(B, H, N, d)
    value = flops_step * world / (ms_max * 1e-3) / 1e12

    pk, pk_src = peaks()
    try:  # DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)
        traffic_tab = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        traffic_tab = {}
    roof = None
    if kernels:
        dom = max(kernels.items(), key=lambda kv: kv[1][0])
        nm, (tot_ms, cnt) = dom
        kind, work = algorithmic_work(nm, dict(B=B, H=H, N=N, d=d, b=b), lab_stats)
        avg = tot_ms / max(cnt, 1)
        if kind == "tensor":
            ach = work / (avg * 1e-3) / 1e12
            peak = pk["bf16_tflops_sustained"]
            roof = {"kernel": nm, "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                    "frac": ach / peak, "traffic": traffic_tab.get(nm), "peak_source": f"{pk_src} bf16 sustained",
                    "algorithmic_flops_per_launch": work, "avg_launch_ms": avg,
                    "share_of_step": tot_ms / args.steps / ms}
        elif kind == "hbm":
            ach = work / (avg * 1e-3) / 1e9
            peak = pk["hbm_gbs"]
            roof = {"kernel": nm, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak, "traffic": traffic_tab.get(nm), "peak_source": f"{pk_src} hbm copy",
                    "algorithmic_bytes_per_launch": work, "avg_launch_ms": avg,
                    "share_of_step": tot_ms / args.steps / ms}
        else:
            roof = {"kernel": nm, "bound": None, "avg_launch_ms": avg}

    out = {
        "metric": "SLA fwd+bwd dense-equiv TFLOPS (Wan2.1-1.3B shape)", "value": value,
        "unit": "TFLOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (randn Q,K,V,dO; W ~ 0.1 randn)",
        "config": config_json(args.config), "path": op.path,
        "gpu_launches": launches[0],
        "roofline": roof,
        "kernels_ms_per_step": {k2: round(v2[0] / args.steps, 4) for k2, v2 in sorted(kernels.items(), key=lambda kv: -kv[1][0])},
        "mask": lab_stats,
    }
    if rank == 0:
        out["clocks"] = clk.summary()
    # --- e2e through the public host-buffer API (HostTrainStep: every chunk's H2D, fwd+bwd
    # through the C-ABI and D2H inside the timed region; copies overlap compute across chunks)
    if not args.no_e2e:
        hs = [torch.empty(shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
        hw = torch.empty((H, d, d), dtype=torch.bfloat16, pin_memory=True)
        for hsrc, dsrc in zip(hs + [hw], (q, k, v, do, w)):
            hsrc.copy_(dsrc.cpu())
        ho = [torch.empty(shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
        hdw = torch.empty((H, d, d), dtype=torch.float32, pin_memory=True)
        del st_buf, o, o_s, o_l, lse, dq, dk, dv  # device-resident step buffers are not used here
        hts = HostTrainStep(B, H, N, d, b, b, cfg, torch.bfloat16, dev, chunks=args.e2e_chunks)

        def e2e_step():
            hts(hs[0], hs[1], hs[2], hw, hs[3], ho[0], ho[1], ho[2], ho[3], hdw)

        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        ev1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([ev0.elapsed_time(ev1) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        out["e2e"] = {"value": flops_step * world / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOPS",
                      "ms_per_step": e2e_ms, "h2d_bytes_per_step": hts.h2d_bytes(),
                      "d2h_bytes_per_step": hts.d2h_bytes(), "chunks": len(hts.ranges),
                      "api": "paper_2509_24006_b200.HostTrainStep (pinned host buffers)"}
    # --- dense attention of the same shape (torch SDPA: cuDNN / flash on sm_100)
    if not args.no_dense and rank == 0:
        try:
            import torch.nn.functional as F

            qd_ = q.clone().requires_grad_(True)
            kd_ = k.clone().requires_grad_(True)
            vd_ = v.clone().requires_grad_(True)

            def dense_step():
                o_ = F.scaled_dot_product_attention(qd_, kd_, vd_)
                o_.backward(do)

            for _ in range(2):
                dense_step()
            torch.cuda.synchronize()
            ev0.record(stream)
            for _ in range(3):
                dense_step()
            ev1.record(stream)
            torch.cuda.synchronize()
            dms = ev0.elapsed_time(ev1) / 3
            out["dense"] = {"kind": "torch SDPA fwd+bwd (library dense kernel, same shape, bf16)",
                            "ms_per_step": dms, "tflops": flops_step / (dms * 1e-3) / 1e12,
                            "speedup_sla_vs_dense": dms / ms_max}
        except Exception as e:  # pragma: no cover
            out["dense"] = {"error": str(e)[:200]}
    # --- CPU baseline: the reference's own path on a bounded sample (rank 0, N=1)
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        try:
            threads = os.cpu_count() or 1
            rcfg = CONFIGS[args.config]
            if rcfg[2] % rcfg[4]:  # the reference needs b | N: time the padded length
                rcfg = rcfg[:2] + ((rcfg[2] + rcfg[4] - 1) // rcfg[4] * rcfg[4],) + rcfg[3:]
            tsec, kind, threads = time_reference_head(rcfg, threads)
            out["cpu_baseline"] = {"value": dense_equiv_flops(1, 1, N, d) / tsec / 1e12, "unit": "TFLOPS",
                                   "cores": threads, "kind": kind,
                                   "sample": f"one (batch, head) unit of {B * H}: fwd+bwd f32 in {tsec:.2f} s"}
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
