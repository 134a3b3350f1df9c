"""TMA latency under the backward kernels' other activity (csrc/diag.cu sla_b200_diag_contention)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_24006_b200 import _lib as L
lib = L.diag_lib()
rows = 16 * 1024 * 1024 // 256
buf = torch.randn(rows, 128, device='cuda').bfloat16()
names = {0: "TMA alone", 1: "+ MMA stream", 2: "+ softmax warps (fence)", 3: "+ MMA + softmax warps (fence)",
         6: "+ softmax warps (no fence)", 7: "+ MMA + softmax warps (no fence)",
         9: "+ MMA stream (pipe kept full)", 25: "+ MN-major MMA stream (pipe kept full)",
         11: "+ MMA (full) + softmax warps (fence)", 27: "+ MN-major MMA (full) + softmax (fence)"}
for mode in (0, 1, 9, 25, 11, 27):
    ctas, iters = 148, 64
    out = (C.c_longlong * (2 * ctas))()
    for _ in range(2):
        assert lib.sla_b200_diag_contention(C.c_void_p(buf.data_ptr()), rows, ctas, iters, mode, out) == 0
    cyc = sorted(out[:2 * ctas]); med = cyc[len(cyc)//2]
    print(f"mode {mode} {names[mode]:36s}: {med/iters:.0f} cyc per 32 KB item (2 producers)")
