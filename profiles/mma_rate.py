"""tcgen05 MMA cost per shape on one SM (csrc/diag.cu sla_b200_diag_mma_rate); output in profiles/r01_mma_rate.txt."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_24006_b200 import _lib as L
lib = L.diag_lib(); torch.zeros(1, device='cuda')
out = C.c_longlong()
for (m, n, am, bm) in [(64,64,0,0),(64,128,0,0),(64,256,0,0),(128,64,0,0),(128,128,0,0),(128,256,0,0),
                       (128,64,1,1),(128,128,1,1),(64,128,0,1),(128,64,0,1),(64,64,0,1),
                       (128,64,2,0),(128,128,2,0),(128,256,2,0),(64,64,2,0),(64,128,2,0),(128,64,2,1),(128,128,2,1),
                       (128,64,3,0),(128,64,4,0),(128,64,6,0),(64,64,4,0),(128,128,4,0)]:
    res = []
    for reps in (16, 256):
        lib.sla_b200_diag_mma_rate(m, n, am, bm, reps, C.byref(out)); lib.sla_b200_diag_mma_rate(m, n, am, bm, reps, C.byref(out))
        res.append(out.value)
    per = (res[1]-res[0])/240
    print(f"M={m} N={n} a_mn={am} b_mn={bm}: 16 MMAs {res[0]} cyc, 256 MMAs {res[1]} cyc, marginal {per:.1f} cyc/MMA, "
          f"{2*m*n*16/per:.0f} flop/cyc, smem {((m*32 if am != 2 else 0)+n*32)/per:.0f} B/cyc" + (" (A in TMEM)" if am == 2 else "") + (f" ({am-2} accumulators round-robin)" if am >= 3 else ""))
