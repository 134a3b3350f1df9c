"""Where the e2e step loses time against the PCIe floor (both directions at once).

    python profiles/e2e_gap.py

A: the e2e step's copy pattern alone (per step 48 H2D + 48 D2H copies of one head's [N, d] bf16
   tensor, on two streams, no compute);
B: the same copies while the C3 fwd+bwd step runs back to back on a third stream (the SLA
   kernels' HBM and SM traffic beside the DMA engines);
C: the compute alone.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24006_b200 import SLA, SlaConfig  # noqa: E402

H, N, d, STEPS = 12, 32768, 128, 10
nb = N * d * 2
host_in = [torch.empty(nb, dtype=torch.uint8, pin_memory=True).fill_(1) for _ in range(4 * H)]
host_out = [torch.empty(nb, dtype=torch.uint8, pin_memory=True).fill_(0) for _ in range(4 * H)]
dev_in = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(4 * H)]
dev_out = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(4 * H)]
s_in, s_out, s_c = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
op = SLA(1, H, N, d, 64, 64, SlaConfig(k_h=5, k_l=10, phi="softmax"), torch.bfloat16)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn((1, H, N, d), generator=g, device="cuda").bfloat16() for _ in range(4))
w = (torch.randn((H, d, d), generator=g, device="cuda") * 0.1).bfloat16()


def step():
    st = op.forward(q, k, v, w)
    op.backward(st, q, k, v, w, do)


def run(copies, compute, steps=STEPS):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    cur = torch.cuda.current_stream()
    e[0].record(cur)
    for s in (s_in, s_out, s_c):
        s.wait_event(e[0])
    for _ in range(steps):
        if copies:
            with torch.cuda.stream(s_in):
                for a, b in zip(dev_in, host_in):
                    a.copy_(b, non_blocking=True)
            with torch.cuda.stream(s_out):
                for a, b in zip(host_out, dev_out):
                    a.copy_(b, non_blocking=True)
        if compute:
            with torch.cuda.stream(s_c):
                step()
    for i, s in enumerate((s_in, s_out, s_c)):
        e[i + 1].record(s)
    torch.cuda.synchronize()
    return max(e[0].elapsed_time(x) for x in e[1:]) / steps


step()
run(True, True, 2)
a = run(True, False)
b = run(True, True)
c = run(False, True)
print(f"A copies alone {a:.2f} ms/step; B copies + compute {b:.2f}; C compute alone {c:.2f}")
