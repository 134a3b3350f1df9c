#!/usr/bin/env python
"""Benchmark of the SLA hot path (BASELINE.json metric: "SLA fwd+bwd ms and dense-equiv
TFLOPS, Wan2.1-1.3B shape N~32K d=128").

One step = dynamic classification + fused forward + fused backward (sla_forward ->
combine_outputs -> proj_backward -> sla_backward in the reference's terms) over the C3
workload: B=1, H=12, N=32768 (32760 padded to a multiple of 64), d=128,
b_q=b_kv=64, k_h=5 %, k_l=10 %, phi=softmax, bf16 inputs with fp32 accumulation.

  python bench.py [--gpus N --steps K --warmup W]            our CUDA path (1 JSON line)
  python bench.py --impl reference [...]                      the reference's CPU path

Multi-GPU (paper_2509_24006_b200/runner.py): one process per GPU.  `--gpus N` without a
torchrun environment re-launches itself under torch.distributed.run with N ranks.  The B*H
(batch, head) units of ONE global problem are partitioned over ranks with
shard.partition_units; the data path has no collective, the step ends with the one real
exchange (the per-head dW all-reduce when a head's batch is split), and a validation gather of
per-unit checksums runs after the timed region.
  c3 (default): weak scaling -- the global problem is B = N batch elements of the C3 shape
                (12 heads each), so every rank owns 12 units at any N.
  c5:           strong scaling -- the fixed B=8 x H=40 problem (configs[4]) split over N ranks.
Timing is the max over ranks of CUDA-event time.
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


SCALING = {"c3": "weak", "c1": "weak", "c3r": "weak", "c5": "strong"}


def global_batch(name, world):
    """Batch of the global problem: weak-scaling configs grow it with the world size."""
    B = CONFIGS[name][0]
    return B * world if SCALING[name] == "weak" else B


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
    ap.add_argument("--no-sustained", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the eager step instead of its CUDA-graph replay")
    ap.add_argument("--e2e-chunks", type=int, default=12)
    ap.add_argument("--e2e-slots", type=int, default=3)
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
def reference_unit_inputs(N, d, unit, seed=1234):
    """bf16-exact SplitMix64 inputs of one (batch, head) unit (rng.hpp:22-57), f32 storage."""
    from oracle import oracle as O

    rng = O.Rng(seed + 7919 * unit)
    bf = lambda a: O.to_bf16_exact(a).astype(np.float32)  # noqa: E731
    return dict(q=bf(rng.gaussian(N, d)), k=bf(rng.gaussian(N, d)), v=bf(rng.gaussian(N, d)),
                w=bf(rng.gaussian(d, d, 0.1)), do=bf(rng.gaussian(N, d)))


def time_reference_unit(cfg, threads, x):
    """One (batch, head) unit through the reference's public API:
    sla_forward -> combine_outputs -> proj_backward -> sla_backward (f32, `threads`)."""
    from oracle import oracle as O

    B, H, N, d, b, k_h, k_l, phi = cfg
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


def reference_cfg(name):
    cfg = CONFIGS[name]
    B, H, N, d, b, k_h, k_l, phi = cfg
    if N % b:  # the reference rejects ragged N (layout.cpp:12-17): time the padded length
        N = (N + b - 1) // b * b
    return (B, H, N, d, b, k_h, k_l, phi)


# units of one reference step that are actually run (~2 s per C3 unit on 16 cores): the 12 units
# of one C3 batch element (all of them at N = 1; weak scaling grows the global batch with N, and
# the step time is scaled by units / 12), or 2 units of c5 (~11 s each) scaled to its 320
REF_UNITS = {"c5": 2}
REF_UNITS_DEFAULT = 12


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = reference_cfg(args.config)
    B, H, N, d, b, k_h, k_l, phi = cfg
    world = max(1, int(os.environ.get("WORLD_SIZE", "1")))
    units_total = global_batch(args.config, world) * H
    run_units = min(units_total, REF_UNITS.get(args.config, REF_UNITS_DEFAULT))
    threads = os.cpu_count() or 1
    xs = [reference_unit_inputs(N, d, u) for u in range(run_units)]
    for i in range(args.warmup):  # a CPU path has nothing to warm beyond its pages: one unit each
        time_reference_unit(cfg, threads, xs[i % run_units])
    kind = "reference"
    steps = []
    for _ in range(args.steps):
        t = 0.0
        for x in xs:
            dt, kind, threads = time_reference_unit(cfg, threads, x)
            t += dt
        steps.append(t * units_total / run_units)
    step_s = sum(steps) / len(steps)
    flops = dense_equiv_flops(1, units_total, N, d)
    value = flops / step_s / 1e12
    sample = (f"every step runs all {units_total} (batch, head) units, fwd+bwd, f32, threads={threads}"
              if run_units == units_total else
              f"every step runs {run_units} of the {units_total} (batch, head) units (fwd+bwd, f32, "
              f"threads={threads}) and scales the time by {units_total}/{run_units}")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": SCALING[args.config], "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_json(args.config, world),
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ms_per_unit": step_s * 1e3 / units_total,
        "warmup_note": "warm-up steps run one unit each",
    }
    print(json.dumps(out), flush=True)


METRIC = "SLA fwd+bwd dense-equiv TFLOPS (Wan2.1-1.3B shape)"


def config_json(name, world=1):
    B, H, N, d, b, k_h, k_l, phi = CONFIGS[name]
    Bg = global_batch(name, world)
    return {"workload": f"{name}: SLA fwd+bwd, B={Bg} H={H} N={N} d={d} b_q=b_kv={b} k_h={k_h}% k_l={k_l}% phi={phi}",
            "batch": Bg, "heads": H, "n": N, "d": d, "block": b, "k_h": k_h, "k_l": k_l, "phi": phi,
            "units": Bg * H, "units_per_rank": -(-Bg * H // world),
            "n_note": ("N = 32760 as-is through SLA_B200_FLAG_RAGGED (read and written in place, TMA zero "
                       "fill past N); the reference arm times N = 32768") if N % b else
                      "N padded from 32760/75600 to a multiple of 64 (make_block_layout rejects ragged N)",
            "l2": "inputs (Q,K,V,dO = 4 x B*H*N*d*2 bytes) exceed the 126 MB L2; no flush needed",
            "parallelism": (f"{Bg * H} (batch x head) units partitioned over {world} rank(s) "
                            f"(shard.partition_units), no data-path collective; dW all-reduce at step end"
                            + (" when world > 1" if world == 1 else "")),
            "scaling_rule": ("weak: the global batch is 1 x world (12 units per rank)" if SCALING[name] == "weak"
                             else "strong: fixed B x H units split over the ranks")}


# ---------------------------------------------------------------------------------------
# roofline bookkeeping
# ---------------------------------------------------------------------------------------
def kernel_work(name, D, crit):
    """Algorithmic work of one step's launches of a kernel: (bound, amount)
    with amount in FLOPs for tensor-bound kernels and bytes for HBM-bound ones.  D: U (units of
    this rank), N, d, T.  crit: critical blocks over all units."""
    U, N, d, T = D["U"], D["N"], D["d"], D["T"]
    tile = 64 * 64 * d
    nd2 = U * N * d * 2  # one [U, N, d] bf16 tensor
    h2 = U * T * d * d * 2  # one [U, T, d, d] bf16 summary tensor
    m0 = U * T * ((T + 7) // 8 * 8) * 2
    return {
        "k_attn_fwd": ("tensor", 4.0 * tile * crit),   # S = QK^T, O += PV
        "k_bwd_rows": ("tensor", 6.0 * tile * crit),   # S, dP recomputed, dQ += dS K
        "k_bwd_cols": ("tensor", 8.0 * tile * crit),   # S, dP recomputed, dV += P^T dO, dK += dS^T Q
        "gemm_aggregate": ("tensor", 2.0 * U * T * T * d * d),
        "gemm_aggregate_t": ("tensor", 2.0 * U * T * T * d * d),
        "gemm_dw": ("tensor", 2.0 * U * N * d * d),
        # HBM: bytes read + written
        "k_pool": ("hbm", 2.0 * nd2 + 2 * U * T * d * 8),                      # Q, K -> pooled f64
        "k_scores": ("hbm", 2.0 * U * T * d * 8 + U * T * T * 8),              # pooled -> f64 scores
        "k_classify": ("hbm", U * T * T * 8 + U * T * T + m0 + U * T * 4 * 2),  # scores -> labels, M0, counts
        "k_phi_kz": ("hbm", 2.0 * nd2 + U * T * 3 * d * 2),                    # K -> phi(K), z parts
        "gemm_summaries": ("hbm", 2.0 * nd2 + h2),                             # phi(K), V -> h
        "k_bwd_lin": ("hbm", 5.0 * nd2 + 2 * h2 + U * N * 4),                  # Q dO O^s O^l H -> dH dQ^phi D^s
    }.get(name, (None, None))


def roofline_table(kernels, steps, D, crit, pk, peak_key):
    rows = []
    for nm, (tot_ms, cnt) in sorted(kernels.items(), key=lambda kv: -kv[1][0]):
        kind, work = kernel_work(nm, D, crit)
        ms = tot_ms / steps
        row = {"kernel": nm, "ms_per_step": round(ms, 4), "launches_per_step": cnt / steps}
        if kind == "tensor":
            ach = work / (ms * 1e-3) / 1e12
            row.update(bound="tensor", achieved=round(ach, 1), unit="TFLOP/s", peak=pk[peak_key],
                       frac=round(ach / pk[peak_key], 3))
        elif kind == "hbm":
            ach = work / (ms * 1e-3) / 1e9
            row.update(bound="hbm", achieved=round(ach, 1), unit="GB/s", peak=pk["hbm_gbs"],
                       frac=round(ach / pk["hbm_gbs"], 3))
        rows.append(row)
    return rows


# ---------------------------------------------------------------------------------------
# our CUDA path
# ---------------------------------------------------------------------------------------
def relaunch_under_torchrun(args):
    """`--gpus N` outside torchrun: one process per GPU via torch.distributed.run."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def dense_comparators(units_q, units_k, units_v, units_do, stream, flops_per_unit, n_units, cfg_tuple, dev):
    """Dense attention of the same shape: torch SDPA (library kernel, name recorded) and this
    repo's own tcgen05 kernels with every block critical (k_h = 100 %: a FlashAttention loop)."""
    import torch
    import torch.nn.functional as F

    out = {}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    qd_, kd_, vd_ = (t.clone().requires_grad_(True) for t in (units_q, units_k, units_v))

    def dense_step():
        o_ = F.scaled_dot_product_attention(qd_, kd_, vd_)
        o_.backward(units_do)

    try:
        for _ in range(2):
            dense_step()
        torch.cuda.synchronize()
        names = []
        try:
            from torch.profiler import ProfilerActivity, profile

            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                dense_step()
                torch.cuda.synchronize()
            ka = sorted(prof.key_averages(), key=lambda e: -getattr(e, "device_time_total", 0))
            names = [e.key for e in ka[:4]]
        except Exception as e:  # pragma: no cover
            names = [f"profiler unavailable: {str(e)[:80]}"]
        ev0.record(stream)
        for _ in range(3):
            dense_step()
        ev1.record(stream)
        torch.cuda.synchronize()
        dms = ev0.elapsed_time(ev1) / 3
        out["sdpa"] = {"kind": "torch SDPA fwd+bwd (library dense kernel, same shape, bf16)",
                       "kernels": names, "ms_per_step": dms * n_units / units_q.shape[1],
                       "tflops": flops_per_unit * units_q.shape[1] / (dms * 1e-3) / 1e12}
    except Exception as e:  # pragma: no cover
        out["sdpa"] = {"error": str(e)[:200]}
    del qd_, kd_, vd_
    try:  # the repo's own dense kernel: the same fused tcgen05 kernels with an all-critical mask
        from paper_2509_24006_b200 import SLA, SlaConfig

        B_, H_, N_, d_, b_, _, _, phi_ = cfg_tuple
        cnt = units_q.shape[1]
        op = SLA(1, cnt, N_, d_, b_, b_, SlaConfig(k_h=100.0, k_l=0.0, phi=phi_), torch.bfloat16, dev)
        w = torch.zeros((cnt, d_, d_), dtype=torch.bfloat16, device=dev)
        st_buf = op.new_state()

        def rd_step():
            st = op.forward(units_q, units_k, units_v, w, state=st_buf)
            op.backward(st, units_q, units_k, units_v, w, units_do)

        rd_step()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(2):
            rd_step()
        ev1.record(stream)
        torch.cuda.synchronize()
        rms = ev0.elapsed_time(ev1) / 2
        out["repo_dense"] = {"kind": "this repo's tcgen05 attention kernels, all blocks critical (k_h = 100 %)",
                             "ms_per_step": rms * n_units / cnt,
                             "tflops": flops_per_unit * cnt / (rms * 1e-3) / 1e12}
        del op, st_buf
    except Exception as e:  # pragma: no cover
        out["repo_dense"] = {"error": str(e)[:200]}
    return out


E2E_MAX_UNITS = 24  # pinned host footprint: 8 [N, d] bf16 tensors per unit
E2E_PASSES = 3  # e2e timed passes of K steps each; the median pass is reported


def run_ours(args):
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    import torch
    import torch.distributed as dist

    from paper_2509_24006_b200 import HostTrainStep, SlaConfig
    from paper_2509_24006_b200 import _lib as L
    from paper_2509_24006_b200.runner import CudaUnits, ShardedStep

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU over NCCL; with more ranks than GPUs (a multi-rank smoke run on a
    # one-GPU box) ranks share devices and the collectives go over gloo
    shared = world > torch.cuda.device_count()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    B, H, N, d, b, k_h, k_l, phi = CONFIGS[args.config]
    Bg = global_batch(args.config, world)
    cfg = SlaConfig(k_h=k_h, k_l=k_l, phi=phi, ragged=N % b != 0)
    runner = ShardedStep(Bg, H, d, world, rank)
    comp = CudaUnits(runner.shard, H, N, d, b, cfg, dev)
    runner.attach(comp)
    # every step runs on one side stream: eager steps and the graph capture below then share the
    # operator's per-stream workspace (a capture on another stream would allocate a second one --
    # 52 GB at c5)
    torch.cuda.synchronize()
    torch.cuda.set_stream(torch.cuda.Stream(dev))
    U = runner.shard.count

    for _ in range(args.warmup):
        runner.step()
    torch.cuda.synchronize()
    labels = comp.last_state.labels
    crit = int((labels == 1).sum())
    lab_stats = {"critical_blocks": crit, "marginal_blocks": int((labels == 0).sum())}
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # The rank's fwd+bwd (every kernel of the step, side-stream fork / join included) captured
    # once into a CUDA graph and replayed per step; the dW reduction (a collective when world > 1)
    # stays eager.  Eager launching leaves the device idle between dependent kernels on some hosts
    # (profiles/host_probe.py: 2.93-3.04 eager vs 2.71 ms graph on one box, with the host only
    # 0.2-0.5 ms per step into the enqueue).
    graph = None
    graph_launches = 0
    if not args.no_graph:
        n0 = comp.launches
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=torch.cuda.current_stream()):
            comp.step()
        graph_launches = comp.launches - n0
        graph.replay()
        runner.reduce_dw()
        torch.cuda.synchronize()

    def step_once():
        if graph is not None:
            graph.replay()
            comp.launches += graph_launches
            runner.reduce_dw()
        else:
            runner.step()

    def timed(n, eager=False):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(n):
            if eager:
                runner.step()
            else:
                step_once()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / n

    with Clocks(local) as clk:  # clocks sampled over both timed passes
        # clean pass without profiler events first: the headline number (the library's side
        # streams run only when its per-kernel profiler is off)
        comp.launches = 0
        ms_clean = timed(args.steps)
        launches = comp.launches // args.steps
        ms_eager = timed(args.steps, eager=True) if graph is not None else ms_clean
        # then the per-kernel breakdown pass (CUDA events after every launch), after the board
        # has idled back to the power state the first pass started from (a second pass run
        # back to back measured 0.15-0.3 ms per step slower at the same SM clock)
        time.sleep(3.0)
        L.lib().sla_b200_profiler(1)
        ms_prof = timed(args.steps, eager=True)  # per-launch events need the eager step
        buf = C.create_string_buffer(1 << 16)
        L.lib().sla_b200_profiler_report(buf, 1 << 16)
        L.lib().sla_b200_profiler(0)
        kernels = {}
        for ln in buf.value.decode().splitlines():
            nm, t, cnt = ln.rsplit(" ", 2)
            kernels[nm] = (float(t), int(cnt))
    ms = ms_clean
    coll_dev = torch.device("cpu") if shared else dev  # gloo reduces host tensors

    def max_over_ranks(x):
        t = torch.tensor([x], device=coll_dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_max = max_over_ranks(ms)
    flops_unit = dense_equiv_flops(1, 1, N, d)
    value = flops_unit * runner.n_units / (ms_max * 1e-3) / 1e12

    # ---- roofline: the dominant kernel and every kernel with a stated algorithmic work
    pk, pk_src = peaks()
    cl = clk.summary()
    at_max = cl["sm_mhz"] is not None and cl["sm_max_mhz"] and cl["sm_mhz"] >= 0.97 * cl["sm_max_mhz"]
    peak_key = "bf16_tflops" if at_max else "bf16_tflops_sustained"
    peak_note = (f"{pk_src} bf16 {'burst' if at_max else 'sustained'}: median SM clock {cl['sm_mhz']} MHz "
                 f"{'at' if at_max else 'below'} max {cl['sm_max_mhz']} MHz over the timed region")
    try:  # DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)
        traffic_tab = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        traffic_tab = {}
    D = dict(U=U, N=N if N % b == 0 else (N + b - 1) // b * b, d=d, T=-(-N // b))
    table = roofline_table(kernels, args.steps, D, crit, pk, peak_key)
    roof = None
    if table:
        dom = table[0]
        nm = dom["kernel"]
        tot_ms, cnt = kernels[nm]
        roof = {"kernel": nm, "bound": dom.get("bound"), "achieved": dom.get("achieved"), "peak": dom.get("peak"),
                "unit": dom.get("unit"), "frac": dom.get("frac"), "traffic": traffic_tab.get(nm),
                "peak_source": peak_note if dom.get("bound") == "tensor" else f"{pk_src} hbm copy",
                "algorithmic_per_launch": kernel_work(nm, D, crit)[1] / max(1, cnt / args.steps),
                "avg_launch_ms": tot_ms / cnt, "share_of_step": tot_ms / args.steps / ms_prof}
        att = [r for r in table if r["kernel"] in ("k_attn_fwd", "k_bwd_rows", "k_bwd_cols")]
        if att:
            w_sum = sum(kernel_work(r["kernel"], D, crit)[1] for r in att)
            t_sum = sum(r["ms_per_step"] for r in att)
            roof["critical_tiles_combined"] = {"achieved": round(w_sum / (t_sum * 1e-3) / 1e12, 1),
                                               "frac": round(w_sum / (t_sum * 1e-3) / 1e12 / pk[peak_key], 3)}

    out = {
        "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": SCALING[args.config], "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (randn Q,K,V,dO per unit seed; W ~ 0.1 randn per head)",
        "config": config_json(args.config, world), "path": comp.op.path,
        "gpu_launches": launches * args.steps, "gpu_launches_per_step": launches,
        "roofline": roof, "kernels": table, "mask": lab_stats,
        "ms_per_step_profiled": ms_prof,
        "launch": ("CUDA graph: the rank's fwd+bwd captured once, replayed per step (dW reduction eager)"
                   if graph is not None else "eager"),
        "ms_per_step_eager": max_over_ranks(ms_eager),
    }
    if rank == 0:
        out["clocks"] = cl
    # ---- sustained: ~2 s of back-to-back steps (the board settles under its power cap; the
    # headline above is the short clean pass), with its own clock samples
    if not args.no_sustained:
        n_sus = min(max(args.steps, int(2000.0 / max(ms_clean, 1e-3))), 2000)
        time.sleep(1.0)
        with Clocks(local) as clk2:
            ms_sus = max_over_ranks(timed(n_sus))
        if rank == 0:
            c2 = clk2.summary()
            out["sustained"] = {"ms_per_step": ms_sus, "steps": n_sus, "seconds": round(ms_sus * n_sus / 1e3, 2),
                                "value": flops_unit * runner.n_units / (ms_sus * 1e-3) / 1e12,
                                "sm_mhz": c2.get("sm_mhz"), "reasons": c2.get("reasons")}
    # ---- validation gather (after the timed region): per-unit checksums to rank 0 over NCCL
    sums = runner.gather_checksums(device=coll_dev)
    if rank == 0 and sums is not None:
        s = sums.double().cpu()
        out["validation"] = {"units": int(s.shape[0]), "checksum_first_unit": [float(x) for x in s[0]],
                             "checksum_all": [float(x) for x in s.sum(0)]}
        if s.shape[0] <= 64:  # per unit: sum and sum |x| of o, dq, dk, dv
            out["validation"]["checksums"] = s.tolist()
    # ---- dense attention of the same shape (rank 0): torch SDPA and the repo's own kernels
    if not args.no_dense and rank == 0:
        nd = min(U, 12)
        out["dense"] = dense_comparators(comp.q[:, :nd], comp.k[:, :nd], comp.v[:, :nd], comp.do[:, :nd], stream,
                                         flops_unit, U, CONFIGS[args.config], dev)
        if "ms_per_step" in out["dense"].get("sdpa", {}):
            out["dense"]["speedup_sla_vs_sdpa"] = out["dense"]["sdpa"]["ms_per_step"] / ms
        if "ms_per_step" in out["dense"].get("repo_dense", {}):
            out["dense"]["speedup_sla_vs_repo_dense"] = out["dense"]["repo_dense"]["ms_per_step"] / ms
    # ---- e2e through the public host-buffer API (HostTrainStep: every chunk's H2D, fwd+bwd
    # through the C-ABI and D2H inside the timed region; copies overlap compute across chunks)
    if not args.no_e2e:
        ne = min(U, E2E_MAX_UNITS)
        shape = (1, ne, N, d)
        hs = [torch.empty(shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
        hw = torch.empty((ne, d, d), dtype=torch.bfloat16, pin_memory=True)
        for hsrc, dsrc in zip(hs + [hw], (comp.q[:, :ne], comp.k[:, :ne], comp.v[:, :ne], comp.do[:, :ne],
                                          comp.w[:ne])):
            hsrc.copy_(dsrc.cpu())
        ho = [torch.empty(shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
        hdw = torch.empty((ne, d, d), dtype=torch.float32, pin_memory=True)
        runner.compute = None
        graph = None  # the captured step's buffers and private pool go with it
        del comp
        torch.cuda.empty_cache()
        # pipelined: step k+1's uploads overlap step k's last downloads (every step still copies
        # its own inputs in and its outputs out inside the timed region; finish() orders the
        # timing stream after the last step)
        hts = HostTrainStep(1, ne, N, d, b, b, cfg, torch.bfloat16, dev, chunks=min(args.e2e_chunks, ne),
                            slots=args.e2e_slots, pipelined=True)

        def e2e_step():
            hts(hs[0], hs[1], hs[2], hw, hs[3], ho[0], ho[1], ho[2], ho[3], hdw)

        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        hts.finish()
        torch.cuda.synchronize()
        # three passes of K steps (PCIe throughput drifts between runs on one box); the median pass
        # is the value, every pass is listed
        passes = []
        for _ in range(E2E_PASSES):
            if world > 1:
                dist.barrier()
            ev0.record(stream)
            for _ in range(args.steps):
                e2e_step()
            hts.finish()
            ev1.record(stream)
            torch.cuda.synchronize()
            passes.append(max_over_ranks(ev0.elapsed_time(ev1) / args.steps))
        e2e_ms = sorted(passes)[len(passes) // 2]
        out["e2e"] = {"value": flops_unit * ne * world / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOPS",
                      "ms_per_step": e2e_ms * U / ne, "passes_ms_per_step": [round(x * U / ne, 4) for x in passes],
                      "h2d_bytes_per_step": hts.h2d_bytes() * U // ne,
                      "d2h_bytes_per_step": hts.d2h_bytes() * U // ne, "chunks": len(hts.ranges),
                      "api": "paper_2509_24006_b200.HostTrainStep (pinned host buffers, pipelined: step k+1's "
                             "H2D overlaps step k's D2H)",
                      "sample": ("all units of the rank" if ne == U else
                                 f"{ne} of the rank's {U} units per step (pinned host footprint); "
                                 f"time and bytes scaled by {U}/{ne}")}
    # ---- CPU baseline: the reference's own path on a bounded sample (rank 0, N=1)
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        try:
            threads = os.cpu_count() or 1
            rcfg = reference_cfg(args.config)
            tsec, kind, threads = time_reference_unit(rcfg, threads, reference_unit_inputs(rcfg[2], d, 0))
            out["cpu_baseline"] = {"value": dense_equiv_flops(1, 1, rcfg[2], d) / tsec / 1e12, "unit": "TFLOPS",
                                   "cores": threads, "kind": kind,
                                   "sample": f"one (batch, head) unit of {runner.n_units}: fwd+bwd f32 in {tsec:.2f} s"}
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
