#!/usr/bin/env bash
# Build-flag variants of libsla_b200.so timed by bench.py (per-kernel ms/step); GPU box only.
# usage: profiles/variants.sh "-DFLAG=1" "-DFLAG=2" ...
set -u
for v in "$@"; do
  make -s -C paper_2509_24006_b200/csrc clean >/dev/null
  make -s -j32 -C paper_2509_24006_b200/csrc EXTRA_NVFLAGS="$v" >/dev/null 2>&1 || { echo "$v: build failed"; continue; }
  python bench.py --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; r=json.loads(sys.stdin.readline()); k={x['kernel']: x['ms_per_step'] for x in r['kernels']}
print('$v'.ljust(28), 'step %.3f ms' % r['ms_per_step'], ' '.join('%s=%.3f' % (n, k[n]) for n in ('k_bwd_cols','k_bwd_rows','k_attn_fwd','k_bwd_lin','gemm_aggregate','gemm_aggregate_t','k_classify','k_scores','gemm_aggregate_z','gemm_aggregate_dz','k_pool','k_phi_kz','gemm_summaries','k_build_csc') if n in k))"
done
