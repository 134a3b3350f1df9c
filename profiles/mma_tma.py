import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_24006_b200 import _lib as L
lib = L.diag_lib()
rows = 16 * 1024 * 1024 // 256
buf = torch.randn(rows, 128, device='cuda').bfloat16()
ctas = 148
for (m, n) in [(128, 64), (64, 64), (128, 128), (128, 256)]:
    for tma in (0, 1):
        out = (C.c_longlong * (2 * ctas))()
        reps = 2048
        for _ in range(2):
            lib.sla_b200_diag_mma_tma(C.c_void_p(buf.data_ptr()), rows, ctas, m, n, reps, tma, out)
        cyc = sorted(out[0::2]); med = cyc[len(cyc)//2]
        loads = sorted(out[1::2]); lm = loads[len(loads)//2]
        print(f"M={m} N={n} tma={tma}: {med/reps:.1f} cyc/MMA, TMA {lm*16384/med:.1f} B/cyc during the MMA stream")
