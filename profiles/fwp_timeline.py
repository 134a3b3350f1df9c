"""Timeline of k_attn_fwd_pair (build with EXTRA_NVFLAGS=-DSLAB_TIMELINE): per-CTA phases of every
CTA and the event clocks of CTA (100, 6), C3 shape."""
import sys, os, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24006_b200 import SLA, SlaConfig, _lib
B, H, n, d = 1, 12, 32768, 128
op = SLA(B, H, n, d, 64, 64, SlaConfig(k_h=5, k_l=10, phi="softmax"), torch.bfloat16)
g = torch.Generator(device='cuda').manual_seed(0); shape = (B, H, n, d)
q, k, v, do = (torch.randn(shape, generator=g, device='cuda').bfloat16() for _ in range(4))
w = (torch.randn((H, d, d), generator=g, device='cuda') * 0.1).bfloat16()
for _ in range(3):
    st = op.forward(q, k, v, w)
torch.cuda.synchronize()
L = _lib.lib()
lab = st.labels.cpu().numpy().reshape(B * H, 512, 512)
buf = (C.c_ulonglong * (8192 * 4))()
assert L.sla_b200_diag_fwp_prof(buf) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 4)[:512 * 12].copy()
sm = (a[:, 3] >> 56).astype(int); a[:, 3] &= (1 << 56) - 1
a = a.astype(np.int64)
cnt = (lab == 1).sum(axis=2).reshape(-1); npairs = (cnt + 1) // 2
pro, loop, epi, tot = a[:, 1] - a[:, 0], a[:, 2] - a[:, 1], a[:, 3] - a[:, 2], a[:, 3] - a[:, 0]
print(f"CTAs {len(a)} mean cycles: prologue {pro.mean():.0f} loop {loop.mean():.0f} epilogue {epi.mean():.0f} total {tot.mean():.0f}")
print(f"pairs/CTA {npairs.mean():.2f}; loop cycles/pair {loop.sum() / max(1, npairs.sum()):.0f}")
span = 0; busy = 0; conc = []
for s in np.unique(sm):
    idx = np.where(sm == s)[0]
    t0, t1 = a[idx, 0].min(), a[idx, 3].max(); span += t1 - t0; busy += tot[idx].sum()
print(f"SMs {len(np.unique(sm))}; mean resident CTAs per SM {busy / span:.2f}")
buf = (C.c_longlong * 256)()
assert L.sla_b200_diag_fwp_timeline(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).copy(); t0 = t[255]
rel = lambda s: int(t[s] - t0) if t[s] else -1
print("CTA (100, 6): x_full", rel(248), "o_ready", rel(250), "proj issue", rel(249), "proj done", rel(251), "stored", rel(252))
cols = [("Ka", 0), ("Kb", 16), ("Va", 32), ("Vb", 48), ("S", 64), ("PV", 80), ("Sseen", 96), ("PVdone", 112), ("Pst", 128)]
print("  p " + "".join(f"{c:>8}" for c, _ in cols))
for i in range(16):
    print(f" {i:2d} " + "".join(f"{rel(o + i):8d}" for _, o in cols))
