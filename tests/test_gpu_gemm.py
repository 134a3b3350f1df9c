"""GPU test of the batched tcgen05 GEMM (gemm.cu) behind the linear branch: every operand
majorness, both M tiles, all N tiles, batched, against an fp32 matmul of the same bf16
inputs (the numerics reference for a floating-point kernel)."""
import ctypes as C

import pytest
import torch

from paper_2509_24006_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _gemm(A, B, M, N, K, batch, a_mn, b_mn, out_f32):
    lib = L.diag_lib()
    fn = lib.sla_b200_diag_gemm
    fn.argtypes = [C.c_void_p] * 3 + [C.c_int] * 7 + [C.c_void_p]
    out = torch.empty((batch, M, N), dtype=torch.float32 if out_f32 else torch.bfloat16, device="cuda")
    rc = fn(A.data_ptr(), B.data_ptr(), out.data_ptr(), batch, M, N, K, int(a_mn), int(b_mn),
            int(out_f32), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("M,N,K,batch", [(128, 256, 512, 2), (64, 128, 64, 3), (256, 64, 192, 1),
                                         (128, 128, 128, 5),
                                         # A-resident aggregation kernel: CTA tile ranges that
                                         # cross (batch, m) blocks, and a K tail
                                         (512, 4096, 512, 3), (384, 512, 200, 2),
                                         # 2-CTA multicast-B path (N-major B, bf16 out, even
                                         # M-tile count) with a K tail and an odd tile-pair count
                                         (256, 768, 200, 3)])
@pytest.mark.parametrize("out_f32", [True, False])
def test_gemm_matches_fp32_matmul(a_mn, b_mn, M, N, K, batch, out_f32):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K + batch)
    A = torch.randn((batch, M, K), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn((batch, K, N), device="cuda", generator=g).to(torch.bfloat16)
    ref = A.float() @ B.float()
    A_in = A.transpose(1, 2).contiguous() if a_mn else A.contiguous()   # [K][M] when M-major
    B_in = B.contiguous() if b_mn else B.transpose(1, 2).contiguous()   # [N][K] when K-major
    out = _gemm(A_in, B_in, M, N, K, batch, a_mn, b_mn, out_f32).float()
    tol = 1e-3 if out_f32 else 1e-2
    err = ((out - ref).abs().max() / ref.abs().max().clamp_min(1.0)).item()
    assert err <= tol, err


@pytest.mark.parametrize("M,N,K,batch,a_mn", [
    (512, 192, 512, 12, False),   # Z = M0 z at d = 64 (BN = 64 tiles)
    (512, 384, 512, 12, True),    # dZ_agg at d = 128 (M-major M0, BN = 128)
    (16, 16384, 16, 1, True),     # a partitioned view's dH_agg (BM = 64, K tail)
    (64, 4096, 200, 3, False),
    (128, 128, 32768, 12, True),  # split-K shaped dW chunks
    (16, 384, 128, 1, True),      # a partitioned view's dZ_agg (BM = 64, BN = 128)
    (16, 192, 128, 1, True),      # ... at d = 64 (BM = 64, BN = 64)
    (48, 384, 512, 2, False),
    (64, 64, 64, 6144, True),     # h_j = phi(K_j)^T V_j at d = 64 (BM = BN = 64), every key block
    (128, 128, 64, 6144, True),   # ... at d = 128
    # BN = 64 with several tiles per persistent CTA: a tile is one output chunk, so the TMA-store
    # staging parity must run across tiles (it once restarted per tile: 1 of 30 repeats differed)
    (128, 192, 64, 128, True),
])
@pytest.mark.parametrize("out_f32", [True, False])
def test_gemm_is_deterministic(M, N, K, batch, a_mn, out_f32):
    """Repeated launches of the same GEMM give bit-identical outputs (no races between the
    producer, MMA and epilogue roles), and match an fp32 matmul."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn((batch, M, K), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn((batch, K, N), device="cuda", generator=g).to(torch.bfloat16)
    A_in = A.transpose(1, 2).contiguous() if a_mn else A.contiguous()
    first = _gemm(A_in, B.contiguous(), M, N, K, batch, a_mn, True, out_f32)
    for _ in range(30):
        again = _gemm(A_in, B.contiguous(), M, N, K, batch, a_mn, True, out_f32)
        assert torch.equal(again, first)
    ref = A.float() @ B.float()
    err = ((first.float() - ref).abs().max() / ref.abs().max().clamp_min(1.0)).item()
    assert err <= (1e-3 if out_f32 else 1e-2), err
