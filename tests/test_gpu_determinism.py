"""Run-to-run determinism of the whole fast path: the same fwd+bwd repeated on the same inputs
must give bit-identical outputs every time.  Both backward passes own their outputs (no atomics,
backward.cpp:68 / :142), so any difference is a race between the asynchronous roles of a kernel
(TMA, tcgen05, epilogue warps) or between streams -- the kind of bug a tolerance-based parity
test can hide.  Shapes cover d = 64 and 128, every phi, ragged N and [B, N, H, d] tensors, and
enough blocks that the persistent kernels (rows pass, GEMMs) run several work items per CTA."""
import pytest
import torch

from paper_2509_24006_b200 import SLA, SlaConfig

pytestmark = pytest.mark.gpu

REPEATS = 8


@pytest.mark.parametrize("heads,n,d,phi,ragged,bnhd", [
    (4, 8192, 128, "softmax", False, False),
    (6, 8192, 64, "elu1", False, False),
    (3, 4160 - 8, 64, "relu", True, False),
    (2, 8192 - 24, 128, "softmax", True, True),
])
def test_repeated_steps_are_bit_identical(heads, n, d, phi, ragged, bnhd):
    g = torch.Generator(device="cuda").manual_seed(heads * 1000 + n + d)
    shape = (1, n, heads, d) if bnhd else (1, heads, n, d)
    q, k, v, do = (torch.randn(shape, generator=g, device="cuda").bfloat16() for _ in range(4))
    w = (torch.randn((heads, d, d), generator=g, device="cuda") * 0.1).bfloat16()
    op = SLA(1, heads, n, d, 64, 64, SlaConfig(k_h=10.0, k_l=20.0, phi=phi, ragged=ragged, bnhd=bnhd),
             torch.bfloat16)

    def step():
        st = op.forward(q, k, v, w)
        gr = op.backward(st, q, k, v, w, do)
        return {"o": st.o, "lse": st.lse, "labels": st.labels, "dq": gr.dq_total, "dk": gr.dk_total,
                "dv": gr.dv, "dw": gr.dproj}

    first = {nm: t.clone() for nm, t in step().items()}
    for it in range(REPEATS):
        out = step()
        for nm, t in out.items():
            assert torch.equal(t, first[nm]), (it, nm)
