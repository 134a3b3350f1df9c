"""TMA issue-to-complete latency per ring item (csrc/diag.cu sla_b200_diag_tma_lat), 148 CTAs."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_24006_b200 import _lib as L
lib = L.diag_lib()
for mb in [int(a) for a in sys.argv[1:]] or (16, 400):
    rows = mb * 1024 * 1024 // 256
    buf = torch.randn(rows, 128, device='cuda').bfloat16()
    for boxes, prod in ([(4,2)] if len(sys.argv) > 1 else [(2,1),(4,1),(8,1),(4,2),(4,4),(8,2),(2,4)]):
        ctas, iters = 148, 64
        out = (C.c_longlong * (8 * ctas))()
        for _ in range(2):
            assert lib.sla_b200_diag_tma_lat(C.c_void_p(buf.data_ptr()), rows, ctas, boxes, iters, prod, out) == 0
        cyc = sorted(out[8*c + p] for c in range(ctas) for p in range(prod)); med = cyc[len(cyc)//2]
        lat = med / iters; kb = boxes * 8
        print(f"buf {mb} MB, item {kb} KB, producers {prod}: {lat:.0f} cyc/item, {kb*1024*prod/lat:.1f} B/cyc/SM")
