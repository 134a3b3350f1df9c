"""BASELINE.json configs[3]: sparsity sweep k_h in {2.5, 5, 10, 20}% at N in {8K, 32K, 75K}, d = 128,
SLA fwd+bwd through the library against torch SDPA (cuDNN / flash, the library dense kernel) of the
same shape, plus the configs[4] shape (B=8, H=40, N=75648) for SLA alone.

    python profiles/sweep.py [out.md]

Every number is a device time from CUDA events around `iters` (10) back-to-back steps after warm-up,
inputs resident (> L2 for every N here).  Critical-tile TFLOP/s counts 14 * 64 * 64 * d per
critical tile (fwd 4 + bwd 10 block matmul-equivalents); dense-equivalent counts 14 N^2 d.
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24006_b200 import SLA, SlaConfig  # noqa: E402


def timed(fn, iters, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def sla_case(B, H, N, d, kh, kl=10.0, iters=5):
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v, do = (torch.randn((B, H, N, d), generator=g, device="cuda").bfloat16() for _ in range(4))
    w = (torch.randn((H, d, d), generator=g, device="cuda") * 0.1).bfloat16()
    op = SLA(B, H, N, d, 64, 64, SlaConfig(k_h=kh, k_l=kl, phi="softmax"), torch.bfloat16)
    st = op.forward(q, k, v, w)
    crit = int((st.labels == 1).sum().item())

    def step():
        s = op.forward(q, k, v, w)
        op.backward(s, q, k, v, w, do)

    ms = timed(step, iters)
    del q, k, v, do, st, op
    torch.cuda.empty_cache()
    return ms, crit


def dense_case(B, H, N, d, iters=5):
    g = torch.Generator(device="cuda").manual_seed(2)
    q, k, v = (torch.randn((B, H, N, d), generator=g, device="cuda").bfloat16().requires_grad_(True)
               for _ in range(3))
    do = torch.randn((B, H, N, d), generator=g, device="cuda").bfloat16()

    def step():
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v)
        o.backward(do)

    ms = timed(step, iters, warm=3)
    del q, k, v, do
    torch.cuda.empty_cache()
    return ms


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep.md"
    rows = []
    d = 128
    for N, B, H in ((8192, 1, 12), (32768, 1, 12), (75648, 1, 4)):
        # SLA first, the (power-hungry) dense run after: a dense run right before the first SLA
        # case left it up to 25 % slow on some boxes
        time.sleep(3)  # let the board power average settle after the previous dense run
        cases = [(kh, *sla_case(B, H, N, d, kh, iters=10)) for kh in (2.5, 5.0, 10.0, 20.0)]
        dense = dense_case(B, H, N, d)
        for kh, ms, crit in cases:
            dense_eq = 14.0 * N * N * d * B * H / (ms * 1e-3) / 1e12
            tile_tf = 14.0 * 64 * 64 * d * crit / (ms * 1e-3) / 1e12
            rows.append((N, B * H, kh, ms, dense, dense / ms, dense_eq, tile_tf))
            print(rows[-1], flush=True)
    ms5, crit5 = sla_case(8, 40, 75648, d, 5.0, iters=2)
    with open(out, "w") as f:
        f.write("| N | units | k_h % | SLA fwd+bwd ms | torch SDPA fwd+bwd ms | speed-up | dense-equiv TFLOPS | critical-tile TFLOP/s |\n")
        f.write("|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write("| %d | %d | %.1f | %.3f | %.3f | %.2fx | %.0f | %.0f |\n" % r)
        f.write("\nconfigs[4] shape B=8 H=40 N=75648 d=128 k_h=5%%: SLA fwd+bwd %.2f ms per step "
                "(%d critical tiles, %.0f critical-tile TFLOP/s, %.0f dense-equiv TFLOPS)\n"
                % (ms5, crit5, 14.0 * 64 * 64 * d * crit5 / (ms5 * 1e-3) / 1e12,
                   14.0 * 75648 ** 2 * d * 320 / (ms5 * 1e-3) / 1e12))
    print(open(out).read())


if __name__ == "__main__":
    main()
