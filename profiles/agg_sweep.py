"""Aggregation regime sweep (the reference's direct / complement /
Four-Russians strategies, aggregation.cpp:40-156): is there a marginal fraction at which a
gather of the marginal summaries h_j would beat the tensor-core GEMM H = M0 h?

    python profiles/agg_sweep.py [out.md]

At the C5 unit shape (N = 75648, T = 1182, d = 128, 4 heads) and at C3 (N = 32768, T = 512,
12 heads), k_h = 5 %, k_l in {0, 10, 45, 90, 94} (marginal fraction 95 % .. 1 %), the library's
per-kernel profiler times the aggregation GEMMs (gemm_aggregate: H = M0 h; gemm_aggregate_t:
dH_agg = M0^T dH) and the whole fwd+bwd step.  Beside them: the HBM floor of a gather
aggregation, which must stream every marginal block's h_j (d^2 bf16) once per (row, marginal
block) pair -- marginal blocks x d^2 x 2 bytes per direction -- at the measured HBM copy peak.
"""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_24006_b200 import SLA, SlaConfig  # noqa: E402
from paper_2509_24006_b200 import _lib as L  # noqa: E402


def run(H, N, d, kl, steps=3):
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v, do = (torch.randn((1, H, N, d), generator=g, device="cuda").bfloat16() for _ in range(4))
    w = (torch.randn((H, d, d), generator=g, device="cuda") * 0.1).bfloat16()
    op = SLA(1, H, N, d, 64, 64, SlaConfig(k_h=5.0, k_l=kl, phi="softmax"), torch.bfloat16)
    st = op.forward(q, k, v, w)
    op.backward(st, q, k, v, w, do)
    marg = int((st.labels == 0).sum().item())
    torch.cuda.synchronize()
    L.lib().sla_b200_profiler(1)
    for _ in range(steps):
        st = op.forward(q, k, v, w)
        op.backward(st, q, k, v, w, do)
    torch.cuda.synchronize()
    buf = C.create_string_buffer(1 << 16)
    L.lib().sla_b200_profiler_report(buf, 1 << 16)
    L.lib().sla_b200_profiler(0)
    ker = {}
    for ln in buf.value.decode().splitlines():
        nm, t, _ = ln.rsplit(" ", 2)
        ker[nm] = float(t) / steps
    del q, k, v, do, st, op
    torch.cuda.empty_cache()
    return marg, ker


def main(out=None):
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    lines = ["| shape | k_l % | marginal blocks | marginal fraction | gemm_aggregate ms | gemm_aggregate_t ms | "
             "gather floor ms (fwd + bwd) | step ms |", "|---|---|---|---|---|---|---|---|"]
    for name, H, N in (("C5 unit x4", 4, 75648), ("C3", 12, 32768)):
        d = 128
        T = N // 64
        for kl in (0.0, 10.0, 45.0, 90.0, 94.0):
            marg, ker = run(H, N, d, kl)
            gather_ms = 2 * marg * d * d * 2 / (hbm * 1e9) * 1e3  # H_i and dH_agg_j: each h read once per pair
            step = sum(ker.values())
            lines.append(f"| {name} | {kl:g} | {marg} | {marg / (H * T * T):.3f} | {ker.get('gemm_aggregate', 0):.4f} | "
                         f"{ker.get('gemm_aggregate_t', 0):.4f} | {gather_ms:.4f} | {step:.3f} |")
            print(lines[-1], flush=True)
    text = "\n".join(lines) + "\n"
    print(text)
    if out:
        open(out, "w").write(text)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
