"""Per-chunk timeline of one pipelined HostTrainStep call in the steady state (C3, 12 one-head
chunks, 12 slots so every chunk keeps its own events): when each chunk's H2D, compute and D2H end,
relative to the end of the previous call's last D2H.

    python profiles/e2e_timeline.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24006_b200 import HostTrainStep, SlaConfig  # noqa: E402

H, N, d = 12, 32768, 128
shape = (1, H, N, d)
hs = [torch.randn(shape).bfloat16().pin_memory() for _ in range(4)]
hw = (torch.randn(H, d, d) * 0.1).bfloat16().pin_memory()
ho = [torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
hdw = torch.empty((H, d, d), dtype=torch.float32).pin_memory()
hts = HostTrainStep(1, H, N, d, 64, 64, SlaConfig(k_h=5, k_l=10, phi="softmax"), torch.bfloat16, "cuda",
                    chunks=12, slots=int(sys.argv[1]) if len(sys.argv) > 1 else 12, pipelined=True)
T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for nm in ("ev_in", "ev_c", "ev_out"):
    setattr(hts, nm, [T() for _ in range(hts.nslots)])
hts.ev_dwout = [T(), T()]
f = lambda: hts(hs[0], hs[1], hs[2], hw, hs[3], ho[0], ho[1], ho[2], ho[3], hdw)  # noqa: E731
for _ in range(4):
    f()
ref = [e for e in hts.ev_out]
rows = []
prev_dw = hts.ev_dwout[1]  # the last call's dW D2H (calls alternate parity; 4 calls done -> parity 1)
for call in range(3):
    f()
    torch.cuda.synchronize()
    base = prev_dw
    S = hts.nslots  # with fewer slots than chunks only the call's last S chunks keep their events
    t = [(base.elapsed_time(hts.ev_in[i % S]), base.elapsed_time(hts.ev_c[i % S]), base.elapsed_time(hts.ev_out[i % S]))
         for i in range(12 - min(S, 12), 12)]
    dw = base.elapsed_time(hts.ev_dwout[(hts.calls - 1) & 1])
    prev_dw = hts.ev_dwout[(hts.calls - 1) & 1]
    print(f"call {call}: dW D2H done at {dw:.2f} ms after the previous call's")
    for i, (a, b, c) in zip(range(12 - len(t), 12), t):
        print(f"  chunk {i:2d}: H2D end {a:7.2f}  compute end {b:7.2f}  D2H end {c:7.2f}")
