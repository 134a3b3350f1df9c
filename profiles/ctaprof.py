"""Per-CTA phase profile of k_bwd_rows / k_bwd_cols (build with EXTRA_NVFLAGS=-DSLAB_TIMELINE)."""
import sys, os, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24006_b200 import SLA, SlaConfig, _lib
B,H,n,d = 1,12,32768,128
op = SLA(B,H,n,d,64,64,SlaConfig(k_h=5,k_l=10,phi="softmax"),torch.bfloat16)
g = torch.Generator(device='cuda').manual_seed(0); shape=(B,H,n,d)
q,k,v,do = (torch.randn(shape,generator=g,device='cuda').bfloat16() for _ in range(4))
w = (torch.randn((H,d,d),generator=g,device='cuda')*0.1).bfloat16()
for _ in range(3):
    st = op.forward(q,k,v,w); gr = op.backward(st,q,k,v,w,do)
torch.cuda.synchronize()
L = _lib.diag_lib()
lab = st.labels.cpu().numpy().reshape(B*H, 512, 512)
cols_v2 = os.environ.get("SLA_B200_COLS", "2") == "2"  # the default columns kernel (attn_bwd_cols2.cu)
cols_prof = L.sla_b200_diag_cols2_ctaprof if cols_v2 else L.sla_b200_diag_cols_ctaprof
cols_tl = L.sla_b200_diag_cols2_timeline if cols_v2 else L.sla_b200_diag_cols_timeline
for name, fn in (("rows", L.sla_b200_diag_rows_ctaprof), ("cols", cols_prof)):
    buf = (C.c_ulonglong * (8192*4))()
    assert fn(buf) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 4)[:512*12].copy()
    sm = (a[:,3] >> 56).astype(int); a[:,3] &= (1<<56)-1
    a = a.astype(np.int64)
    if name == "rows": cnt = (lab == 1).sum(axis=2).reshape(-1)
    else: cnt = (lab == 1).sum(axis=1).reshape(-1)
    npairs = (cnt + 1)//2
    pro, loop, epi = a[:,1]-a[:,0], a[:,2]-a[:,1], a[:,3]-a[:,2]
    tot = a[:,3]-a[:,0]
    print(f"== {name}: CTAs {len(a)}  mean cycles: prologue {pro.mean():.0f}  loop {loop.mean():.0f}  epilogue {epi.mean():.0f}  total {tot.mean():.0f}")
    print(f"   pairs/CTA mean {npairs.mean():.2f}  loop cycles/pair {loop.sum()/max(1,npairs.sum()):.0f}")
    for pct in (10,50,90,99): print(f"   p{pct}: pro {np.percentile(pro,pct):.0f} loop {np.percentile(loop,pct):.0f} epi {np.percentile(epi,pct):.0f}")
    gaps=[]; busy=0; span=0
    for s in np.unique(sm):
        idx = np.where(sm==s)[0]; o = idx[np.argsort(a[idx,0])]
        gaps += list(a[o[1:],0]-a[o[:-1],3]); busy += tot[o].sum(); span += a[o[-1],3]-a[o[0],0]
    gaps=np.array(gaps); print(f"   inter-CTA gap on an SM: mean {gaps.mean():.0f} p50 {np.median(gaps):.0f}; SM busy frac {busy/span:.3f}; SMs {len(np.unique(sm))}")

# single-CTA (blockIdx 100, unit 6) event timelines (ts_mark slots, clock64)
for name, fn, cols in (("rows", L.sla_b200_diag_bwd_timeline, [("ldK", 0), ("ldV", 112), ("Kin", 80), ("Vin", 96), ("sdp", 16), ("sdp_r", 208), ("got", 32), ("ldw", 240), ("math", 128), ("empty", 144), ("dS", 48), ("acc", 64), ("acc_r", 224)]),
                       ("cols", cols_tl, [("ld", 0), ("in", 80), ("sdp", 16), ("got", 32), ("math", 128), ("empty", 144), ("PdS", 48), ("acc", 96), ("adone", 64)])):
    buf = (C.c_longlong * 256)()
    assert fn(buf) == 0
    t = np.frombuffer(buf, dtype=np.int64).copy(); t0 = t[127]
    rel = lambda s: (t[s] - t0) if t[s] else -1
    print(f"== {name} CTA timeline (cycles from entry); marks 118-126:", [rel(s) for s in range(118, 127)])
    print("   t  " + "  ".join(f"{c:>6}" for c, _ in cols))
    for i in range(16):
        print(f"  {i:2d}  " + "  ".join(f"{rel(o + i) if o != 112 or i < 8 else -1:6d}" for _, o in cols))

buf = (C.c_longlong * 256)(); L.sla_b200_diag_bwd_timeline(buf)
t = np.frombuffer(buf, dtype=np.int64).copy(); t0 = t[127]
print("rows per-warp (warps 2..9) got / dS-arrive for t=4..7, cycles from entry:")
for i in range(4):
    print(f"  t={4+i} got ", [int(t[192 + 8*i + w] - t0) for w in range(8)])
    print(f"       done", [int(t[160 + 8*i + w] - t0) for w in range(8)])

lat_k = [t[80 + i] - t[i] for i in range(3, 12)]; lat_v = [t[96 + i] - t[112 + i] for i in range(3, 8)]
print(f"rows TMA latency (t>=3): K pair {np.mean(lat_k):.0f} cyc, V pair {np.mean(lat_v):.0f} cyc; loop/pair {(t[64+11]-t[64+3])/8:.0f}")

# forward CTA (100, 6) timeline (attn_fwd.cu fts marks)
buf = (C.c_longlong * 128)(); L.sla_b200_diag_fwd_timeline(buf)
t = np.frombuffer(buf, dtype=np.int64).copy(); t0 = t[127]
rel = lambda s: int(t[s] - t0) if t[s] else -1
print("fwd marks 96-105:", [rel(s) for s in range(96, 106)])
print("   t   ldK     S   got     P")
for i in range(24):
    print(f"  {i:2d} " + " ".join(f"{rel(o + i):6d}" for o in (0, 24, 48, 72)))
