"""One small fwd+bwd through the C-ABI, for compute-sanitizer (tests/test_gpu_sanitizer.py):
N = 1024, d in {64, 128}, dynamic mask, both phi kinds that exercise every kernel branch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

from paper_2509_24006_b200 import SLA, SlaConfig  # noqa: E402


def main(d: int, generic: bool) -> None:
    n, heads = 1024, 2
    g = torch.Generator(device="cuda").manual_seed(5)
    shape = (1, heads, n, d)
    q, k, v, do, dol = (torch.randn(shape, generator=g, device="cuda").to(torch.bfloat16) for _ in range(5))
    w = (torch.randn((heads, d, d), generator=g, device="cuda") * 0.1).to(torch.bfloat16)
    for phi in ("softmax", "elu1"):
        op = SLA(1, heads, n, d, 64, 64, SlaConfig(k_h=10.0, k_l=20.0, phi=phi, force_generic=generic),
                 torch.bfloat16)
        st = op.forward(q, k, v, w)
        op.backward(st, q, k, v, w, do, parts=True)
        op.backward(st, q, k, v, None, do, d_out_linear=dol)
    torch.cuda.synchronize()
    print("sanitize step ok")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 128, len(sys.argv) > 2 and sys.argv[2] == "generic")
