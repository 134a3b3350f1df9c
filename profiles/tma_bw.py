import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_24006_b200 import _lib as L
lib = L.diag_lib()
mb = 16
rows = mb * 1024 * 1024 // 256
buf = torch.randn(rows, 128, device='cuda').bfloat16()
for ctas, slots, prod in [(148,4,1),(148,4,2),(148,8,2),(148,8,4),(148,12,4),(148,12,3),(148,12,6),(296,4,1),(296,4,2),(296,6,3),(444,4,1),(444,4,2)]:
    out = (C.c_longlong * ctas)()
    iters = 480
    for _ in range(2):
        lib.sla_b200_diag_tma_bw(C.c_void_p(buf.data_ptr()), rows, ctas, slots, iters, prod, out)
    cyc = sorted(out[:ctas]); med = cyc[len(cyc)//2]
    per_sm = iters * 16384 * (ctas / 148) / med
    print(f"ctas {ctas} slots {slots} producers {prod}: median {med} cyc, {per_sm:.1f} B/cyc/SM, chip {per_sm*148*1.9e9/1e12:.1f} TB/s @1.9GHz")
