#!/usr/bin/env bash
# Profile collection for profiles/ (run on the GPU box from the repo root, e.g. via gpurun).
# 1. launch list of the bench command (cold-cache, serialised per-launch times)
# 2. one `--set full` capture of every distinct kernel of a C3 fwd+bwd step (second step)
# 3. the bench line itself (never taken under a profiler)
set -u
out=${1:-gpurun_out}
mkdir -p "$out"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" \
    python bench.py --steps 2 --warmup 1 --no-dense --no-e2e --no-cpu-baseline --no-sustained > "$out/launches_bench.log" 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:k_bwd_cols|k_bwd_rows|k_attn_fwd|k_bwd_lin|k_gemm|k_classify|k_scores|k_aggregate_vec|k_phi_kz|k_pool" \
    -s 14 -c 14 -o "$out/full" python profiles/prof_step.py 2 > "$out/full.log" 2>&1
python bench.py --steps 20 --warmup 5 > "$out/bench.json" 2> "$out/bench.err"
