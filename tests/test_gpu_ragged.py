"""Ragged N (SLA_B200_FLAG_RAGGED) and the token-major
[B, N, H, d] layout (SLA_B200_FLAG_BNHD).

The reference rejects N % b != 0 (layout.cpp:12-17), so there is no reference output to match.
The semantics are pinned three ways:
  * mask: bit-exact against the C oracle's ragged restatement (oracle/sla_oracle.c
    orc_predict_ragged: last block pooled over its valid rows, mask.cpp:40-119 otherwise);
  * forward + backward: against a dense fp32 torch reference of the same operator (keys >= N
    excluded from both branches), gradients by torch.autograd, within the bf16 gate 2e-2;
  * N % 64 == 0 with the flag set is bit-identical to the unflagged (reference-exact) call.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2509_24006_b200 import SLA, SlaConfig

pytestmark = pytest.mark.gpu
B = 64


def _bf16(rng, n, d, scale=1.0):
    return O.to_bf16_exact(rng.gaussian(n, d, scale))


def _phi(x, kind):
    if kind == "softmax":
        return torch.softmax(x, dim=-1)
    if kind == "relu":
        return torch.relu(x)
    return torch.where(x >= 0, x + 1.0, torch.exp(x))  # elu1


def _dense_reference(q, k, v, w, labels, kind):
    """One unit, f32: O = O^s + O^l W with the block mask expanded to elements (keys < N only)."""
    n, d = q.shape
    blk = torch.arange(n, device=q.device) // B
    lab = labels[blk][:, blk]                      # [N, N] element labels
    crit, marg = lab == 1, lab == 0
    s = (q @ k.T) / d ** 0.5
    s = s.masked_fill(~crit, float("-inf"))
    has = crit.any(1, keepdim=True)
    p = torch.softmax(torch.where(has, s, torch.zeros_like(s)), dim=1) * has * crit
    o_s = p @ v
    fq, fk = _phi(q, kind), _phi(k, kind)
    a = (fq @ fk.T) * marg                         # linear-branch weights of marginal keys
    den = a.sum(1, keepdim=True)
    o_l = torch.where(den != 0, (a @ v) / torch.where(den != 0, den, torch.ones_like(den)),
                      torch.zeros_like(o_s))
    return o_s + o_l @ w


@pytest.mark.parametrize("n,d,phi", [(1000, 64, "softmax"), (1000, 64, "elu1"), (4040, 128, "softmax")])
def test_ragged_matches_dense_reference(n, d, phi):
    heads = 2
    cfg = SlaConfig(k_h=10.0, k_l=20.0, phi=phi, ragged=True)
    xs = []
    for h in range(heads):
        rng = O.Rng(8100 + 10 * h + n)
        xs.append({nm: _bf16(rng, n, d) for nm in ("q", "k", "v", "do")})
    wnp = O.to_bf16_exact(O.Rng(4).gaussian(d, d, 0.1))
    T = lambda a: torch.tensor(np.array(a), dtype=torch.float32, device="cuda")  # noqa: E731
    q, k, v, do = (T([[x[nm] for x in xs]]).bfloat16() for nm in ("q", "k", "v", "do"))
    wt = T([wnp] * heads).bfloat16()
    op = SLA(1, heads, n, d, B, B, cfg, torch.bfloat16)
    assert op.t_m == (n + B - 1) // B
    st = op.forward(q, k, v, wt)
    g = op.backward(st, q, k, v, wt, do)
    torch.cuda.synchronize()
    for h in range(heads):
        x = xs[h]
        want_lab = O.dynamic_labels_ragged(x["q"], x["k"], B, cfg.k_h, cfg.k_l)
        got_lab = st.labels[0, h].cpu().numpy()
        assert (got_lab == want_lab).all(), "ragged mask differs from the oracle restatement"
        leaves = [T(x[nm]).requires_grad_(True) for nm in ("q", "k", "v")]
        wl = T(wnp).requires_grad_(True)
        o_ref = _dense_reference(*leaves, wl, torch.tensor(want_lab, device="cuda"), phi)
        o_ref.backward(T(x["do"]))
        pairs = [(st.o[0, h], o_ref), (g.dq_total[0, h], leaves[0].grad), (g.dk_total[0, h], leaves[1].grad),
                 (g.dv[0, h], leaves[2].grad)]
        for got, ref in pairs:
            err = O.rel_diff(got.double().cpu().numpy(), ref.detach().double().cpu().numpy(), 1.0)
            assert err <= 2e-2, err
    for h in range(heads):  # per-head dW against the dense reference (summed W gradient per head)
        x = xs[h]
        leaves = [T(x[nm]) for nm in ("q", "k", "v")]
        wl = T(wnp).requires_grad_(True)
        lab = torch.tensor(O.dynamic_labels_ragged(x["q"], x["k"], B, cfg.k_h, cfg.k_l), device="cuda")
        _dense_reference(*leaves, wl, lab, phi).backward(T(x["do"]))
        err = O.rel_diff(g.dproj[h].double().cpu().numpy(), wl.grad.double().cpu().numpy(), 1.0)
        assert err <= 2e-2, err


def test_ragged_flag_is_inert_for_divisible_n():
    n, d, heads = 1024, 64, 2
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v, do = (torch.randn((1, heads, n, d), generator=g, device="cuda").bfloat16() for _ in range(4))
    w = (torch.randn((heads, d, d), generator=g, device="cuda") * 0.1).bfloat16()
    outs = []
    for ragged in (False, True):
        op = SLA(1, heads, n, d, B, B, SlaConfig(k_h=5.0, k_l=10.0, phi="softmax", ragged=ragged))
        st = op.forward(q, k, v, w)
        gr = op.backward(st, q, k, v, w, do)
        outs.append((st.o, st.lse, st.labels, gr.dq_total, gr.dk_total, gr.dv, gr.dproj))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_ragged_needs_the_flag_and_the_fast_path():
    with pytest.raises(ValueError, match="does not divide"):
        SLA(1, 1, 1000, 64, B, B, SlaConfig(), torch.bfloat16)
    with pytest.raises(ValueError, match="ragged"):
        SLA(1, 1, 1000, 64, B, B, SlaConfig(ragged=True), torch.float32)
    with pytest.raises(ValueError, match="ragged"):
        SLA(1, 1, 1000, 64, 32, 32, SlaConfig(ragged=True), torch.bfloat16)


@pytest.mark.parametrize("n", [1024, 1000])
def test_token_major_layout_matches_unit_major(n):
    """SLA_B200_FLAG_BNHD: [B, N, H, d] tensors (lse [B, N, H]) give the unit-major results bit
    for bit, with and without a ragged tail."""
    B, H, d = 2, 3, 64
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v, do = (torch.randn((B, H, n, d), generator=g, device="cuda").bfloat16() for _ in range(4))
    w = (torch.randn((H, d, d), generator=g, device="cuda") * 0.1).bfloat16()
    ragged = n % 64 != 0
    op1 = SLA(B, H, n, d, 64, 64, SlaConfig(k_h=10.0, k_l=20.0, phi="softmax", ragged=ragged))
    op2 = SLA(B, H, n, d, 64, 64, SlaConfig(k_h=10.0, k_l=20.0, phi="softmax", ragged=ragged, bnhd=True))
    t = lambda x: x.transpose(1, 2).contiguous()  # noqa: E731
    st1 = op1.forward(q, k, v, w)
    g1 = op1.backward(st1, q, k, v, w, do)
    st2 = op2.forward(t(q), t(k), t(v), w)
    g2 = op2.backward(st2, t(q), t(k), t(v), w, t(do))
    torch.cuda.synchronize()
    assert torch.equal(st1.labels, st2.labels)
    for x1, x2 in ((st1.o, st2.o), (st1.o_s, st2.o_s), (st1.o_l, st2.o_l), (g1.dq_total, g2.dq_total),
                   (g1.dk_total, g2.dk_total), (g1.dv, g2.dv)):
        assert torch.equal(x1, x2.transpose(1, 2))
    assert torch.equal(st1.lse, st2.lse.transpose(1, 2))
    assert torch.equal(g1.dproj, g2.dproj)
