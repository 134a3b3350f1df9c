"""The PyTorch caller (paper_2509_24006_b200/autograd.py): torch.autograd through the C-ABI.

Gradients must be exactly the ones the operator API returns for the same inputs (the
Function adds no arithmetic), layouts [B,H,N,d] and [B,N,H,d] must agree bit for bit, a
shared W must receive the head-summed dW, and one head is checked against the C oracle.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2509_24006_b200 import SLA, SlaConfig, SparseLinearAttention, sparse_linear_attention

pytestmark = pytest.mark.gpu

B, H, N, D = 1, 2, 1024, 64
CFG = SlaConfig(k_h=5.0, k_l=10.0, phi="softmax")


def _inputs(seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v, do = (torch.randn((B, H, N, D), generator=g, device="cuda").bfloat16() for _ in range(4))
    w = (torch.randn((H, D, D), generator=g, device="cuda") * 0.1).bfloat16()
    return q, k, v, w, do


def _grads(q, k, v, w, do, layout="bhnd"):
    leaves = [t.clone().requires_grad_(True) for t in (q, k, v, w)]
    o = sparse_linear_attention(*leaves, cfg=CFG, layout=layout)
    o.backward(do)
    return o.detach(), [t.grad for t in leaves]


def test_autograd_matches_operator_api():
    q, k, v, w, do = _inputs(1)
    o, (dq, dk, dv, dw) = _grads(q, k, v, w, do)
    op = SLA(B, H, N, D, 64, 64, CFG, torch.bfloat16)
    st = op.forward(q, k, v, w)
    g = op.backward(st, q, k, v, w, do)
    torch.cuda.synchronize()
    assert torch.equal(o, st.o)
    assert torch.equal(dq, g.dq_total) and torch.equal(dk, g.dk_total) and torch.equal(dv, g.dv)
    assert torch.equal(dw, g.dproj.bfloat16())


def test_bnhd_layout_matches_bhnd():
    q, k, v, w, do = _inputs(2)
    o1, g1 = _grads(q, k, v, w, do)
    t = lambda x: x.transpose(1, 2).contiguous()  # noqa: E731
    o2, g2 = _grads(t(q), t(k), t(v), w, t(do), layout="bnhd")
    assert torch.equal(o1, o2.transpose(1, 2))
    for a, b in zip(g1[:3], g2[:3]):
        assert torch.equal(a, b.transpose(1, 2))
    assert torch.equal(g1[3], g2[3])


def test_shared_projection_gets_head_sum():
    q, k, v, w, do = _inputs(3)
    w1 = w[0].clone()
    _, (_, _, _, dw_shared) = _grads(q, k, v, w1, do)
    _, (_, _, _, dw_heads) = _grads(q, k, v, w1.unsqueeze(0).expand(H, D, D).contiguous(), do)
    ref = dw_heads.float().sum(0)
    assert dw_shared.shape == (D, D)
    assert (dw_shared.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


def test_module_against_oracle():
    xs = []
    for h in range(H):
        rng = O.Rng(5100 + h)
        xs.append({nm: O.to_bf16_exact(rng.gaussian(N, D, 1.0)) for nm in ("q", "k", "v", "do")})
    wnp = O.to_bf16_exact(O.Rng(77).gaussian(D, D, 0.1))
    T = lambda a: torch.tensor(np.array(a), dtype=torch.float32, device="cuda").bfloat16()  # noqa: E731
    q, k, v, do = (T([[x[nm] for x in xs]]) for nm in ("q", "k", "v", "do"))
    m = SparseLinearAttention(H, D, CFG, layout="bhnd").cuda()
    with torch.no_grad():
        m.proj.copy_(T([wnp] * H))
    q.requires_grad_(True)
    o = m(q, k, v)
    o.backward(do)
    for h in range(H):
        x = xs[h]
        lab = O.dynamic_labels(x["q"], x["k"], 64, 64, 5.0, 10.0)
        want = O.step(x["q"], x["k"], x["v"], wnp, x["do"], lab, 64, 64, "softmax")
        assert O.rel_diff(o[0, h].detach().double().cpu().numpy(), want["o"], 1.0) <= 2e-2
        assert O.rel_diff(q.grad[0, h].double().cpu().numpy(), want["dq_total"], 1.0) <= 2e-2
