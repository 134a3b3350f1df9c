"""Timeline of k_attn_fwd_pp CTA 7 (build with EXTRA_NVFLAGS=-DSLAB_TIMELINE), C3 shape."""
import sys, os, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SLA_B200_FWD_PAIR"] = "2"
from paper_2509_24006_b200 import SLA, SlaConfig, _lib
B, H, n, d = 1, 12, 32768, 128
op = SLA(B, H, n, d, 64, 64, SlaConfig(k_h=5, k_l=10, phi="softmax"), torch.bfloat16)
g = torch.Generator(device='cuda').manual_seed(0); shape = (B, H, n, d)
q, k, v = (torch.randn(shape, generator=g, device='cuda').bfloat16() for _ in range(3))
w = (torch.randn((H, d, d), generator=g, device='cuda') * 0.1).bfloat16()
for _ in range(3): st = op.forward(q, k, v, w)
torch.cuda.synchronize()
buf = (C.c_longlong * 256)(); assert _lib.lib().sla_b200_diag_fpp_timeline(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).copy(); t0 = t[255]
rel = lambda s: int(t[s] - t0) if t[s] else -1
print("  g   Sissue  Sseen  Pstored PVissue")
for i in range(32): print(f" {i:2d} {rel(32+i):8d} {rel(96+i):8d} {rel(i):8d} {rel(64+i):8d}")
print("softmax steps g=4..7 (S loaded, own max, partner max, exps, P buffer free, vote, stored, fenced):")
for gg in range(4): print("  ", [rel(128 + 8 * gg + k) for k in range(8)])
print("epilogue start/done per block:", [(rel(192+i), rel(224+i)) for i in range(4)])
print("ring item issue:", [rel(160+i) for i in range(32)])
