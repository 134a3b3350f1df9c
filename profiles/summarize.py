"""Turn the outputs of profiles/collect.sh into the tracked summaries under profiles/.

    python profiles/summarize.py gpurun_out r01

writes profiles/<tag>_launches.md (per-kernel share of the ncu launch list),
profiles/<tag>_ncu_kernels.md (one `--set full` capture per kernel: duration, DRAM bytes,
L2 bytes into the SMs, tensor-pipe activity, occupancy) and profiles/traffic.json (DRAM bytes per
launch by bench.py kernel name, read by bench.py's roofline `traffic` field), and copies the
bench line to profiles/<tag>_bench.json.  Needs `ncu` (present in this image) to read the report.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))

# ncu kernel (template instance) -> bench.py / profiler name
GEMM_NAMES = {  # template arguments BM, BN, A_MN, B_MN, OutT (the trailing MC / P2 flags dropped)
    "k_gemm<128, 128, 1, 1, __nv_bfloat16>": "gemm_summaries",
    "k_gemm<128, 256, 0, 1, __nv_bfloat16>": "gemm_aggregate",
    "k_gemm<128, 256, 1, 1, __nv_bfloat16>": "gemm_aggregate_t",
    "k_gemm<128, 128, 1, 1, float>": "gemm_dw / gemm_aggregate_dz",
    "k_gemm<128, 128, 0, 1, float>": "gemm_aggregate_z",
}


def short(name: str) -> str:
    m = re.search(r"(k_gemm<[^>]*>)", name)
    if m:
        key = re.sub(r"(, [01])+>$", ">", m.group(1))  # the multicast / CTA-pair flags dropped
        return GEMM_NAMES.get(key, m.group(1))
    m = re.search(r"(k_aggregate_vec)<(\d)>", name)
    if m:
        return "k_aggregate_z" if m.group(2) == "0" else "k_aggregate_dz"
    m = re.search(r"\b(k_[A-Za-z0-9_]+)", name)
    if not m:
        return name[:40]
    # kernels whose bench.py / profiler name differs from the symbol (variants of one stage)
    return {"k_bwd_cols2": "k_bwd_cols", "k_attn_fwd_pp": "k_attn_fwd"}.get(m.group(1), m.group(1))


def launches(path: str):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        k = short(d["Kernel Name"])
        tot[k] += v
        cnt[k] += 1
    return tot, cnt


def full(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1024, "byte/block": 1,
             "ms": 1, "us": 1e-3, "ns": 1e-6, "msecond": 1, "usecond": 1e-3, "nsecond": 1e-6}
    out = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        k = short(d["Kernel Name"])

        def f(m):  # value in base units (bytes, ms, %)
            try:
                return float(d.get(m, "").replace(",", "")) * scale.get(units.get(m, ""), 1)
            except ValueError:
                return None

        out[k] = {
            "duration_ms": f("gpu__time_duration.sum"),
            "dram_read": f("dram__bytes_read.sum"),
            "dram_write": f("dram__bytes_write.sum"),
            "l2_to_sm_bytes": f("l1tex__m_xbar2l1tex_read_bytes.sum"),
            "tensor_active_pct": f("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
            "utc_bf16_pct": f("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"),
            "lts_pct": f("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "regs": f("launch__registers_per_thread"),
            "smem_dyn": f("launch__shared_mem_per_block_dynamic"),
        }
    return out


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
    tot, cnt = launches(os.path.join(src, "launches.csv"))
    all_ns = sum(tot.values())
    with open(os.path.join(HERE, f"{tag}_launches.md"), "w") as fh:
        fh.write(f"# ncu launch list, {tag}\n\n`profiles/collect.sh` step 1: `ncu --metrics gpu__time_duration.sum "
                 "--clock-control none --csv python bench.py --steps 2 --warmup 1 --no-dense --no-e2e "
                 "--no-cpu-baseline`\n\nCold-cache, serialised per-launch device times summed over the 3 "
                 "executed steps (1 warm-up + 2 timed) plus bench.py's profiler pass and clean pass; compare "
                 "SHARES with bench.py's live `kernels_ms_per_step`, not absolutes.  Non-`k_`/`gemm_` rows are "
                 "torch's input initialisation.\n\n| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            fh.write(f"| {k} | {cnt[k]} | {v / 1e6:.3f} | {100 * v / all_ns:.1f}% |\n")
    fk = full(os.path.join(src, "full.ncu-rep"))
    with open(os.path.join(HERE, f"{tag}_ncu_kernels.md"), "w") as fh:
        fh.write(f"# `ncu --set full` per kernel, {tag}\n\n`profiles/collect.sh` step 2: one capture of each "
                 "kernel of a C3 fwd+bwd step (B=1, H=12, N=32768, d=128, k_h=5%, k_l=10%, softmax phi) "
                 "with `--clock-control none`.\n\n- DRAM = dram__bytes_read.sum + dram__bytes_write.sum; "
                 "L2->SM = l1tex__m_xbar2l1tex_read_bytes.sum (TMA / load bytes delivered to the SMs)\n"
                 "- tensor% = sm__pipe_tensor_cycles_active_realtime (pct of peak, elapsed); "
                 "UTC bf16% = tcgen05 bf16 ops vs peak\n\n"
                 "| kernel | ms | DRAM MB | DRAM TB/s | L2->SM MB | L2->SM TB/s | tensor % | UTC bf16 % | LTS % | occ % | regs | dyn smem KB |\n"
                 "|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for k, m in sorted(fk.items(), key=lambda kv: -(kv[1]["duration_ms"] or 0)):
            ms = m["duration_ms"] or 0
            dram = (m["dram_read"] or 0) + (m["dram_write"] or 0)
            l2 = m["l2_to_sm_bytes"] or 0
            g = lambda x: "-" if x is None else f"{x:.1f}"  # noqa: E731
            fh.write(f"| {k} | {ms:.3f} | {dram / 1e6:.0f} | {dram / (ms * 1e-3) / 1e12 if ms else 0:.2f} | "
                     f"{l2 / 1e6:.0f} | {l2 / (ms * 1e-3) / 1e12 if ms else 0:.2f} | {g(m['tensor_active_pct'])} | "
                     f"{g(m['utc_bf16_pct'])} | {g(m['lts_pct'])} | {g(m['occupancy_pct'])} | "
                     f"{g(m['regs'])} | {(m['smem_dyn'] or 0) / 1024:.0f} |\n")
    traffic = {k: (m["dram_read"] or 0) + (m["dram_write"] or 0) for k, m in fk.items()}
    json.dump(traffic, open(os.path.join(HERE, "traffic.json"), "w"), indent=1, sort_keys=True)
    bench = os.path.join(src, "bench.json")
    if os.path.exists(bench):
        line = open(bench).read().strip().splitlines()[-1]
        json.dump(json.loads(line), open(os.path.join(HERE, f"{tag}_bench.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
