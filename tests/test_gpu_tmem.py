"""GPU test pinning the TMEM data-path layouts the kernels rely on (csrc/diag.cu):
tcgen05.ld.16x32bx2 thread map, and an M=64 MMA at lane offset 16 filling lanes 16-31."""
import ctypes as C

import pytest
import torch

from paper_2509_24006_b200 import _lib as L

pytestmark = pytest.mark.gpu


def test_tmem_layouts():
    f = L.diag_lib().sla_b200_diag_tmem
    f.argtypes = [C.c_void_p] * 4
    x2 = torch.zeros(128 * 16, dtype=torch.int32, device="cuda")
    lo = torch.zeros(256, device="cuda")
    hi = torch.zeros(256, device="cuda")
    assert f(x2.data_ptr(), lo.data_ptr(), hi.data_ptr(), None) == 0
    torch.cuda.synchronize()
    x2 = x2.view(4, 32, 16).cpu()
    for w in range(4):
        for t in range(32):
            lane = 32 * w + (t % 16)
            col0 = 0 if t < 16 else 16
            assert x2[w, t].tolist() == [lane * 1000 + col0 + c for c in range(16)]
    lo = lo.view(4, 32, 2).cpu()
    hi = hi.view(4, 32, 2).cpu()
    for w in range(4):
        for t in range(32):
            row = 16 * w + (t % 16) + 1   # D[m][n] = m + 1
            assert lo[w, t, 0] == (row if t < 16 else 0)
            assert hi[w, t, 0] == (row if t >= 16 else 0)
