"""GPU parity of the tcgen05 fast path (b_q = b_kv = 64, d in {64, 128}, bf16) against the C
oracle on the same bf16-exact inputs, including the edge cases the reference pins.

Tolerance: rel_diff (floor 1.0) <= 1.2e-2 for outputs and gradients -- bf16 operands (Q, K, V,
P, phi(Q), H, W) with fp32 accumulation and bf16 outputs; lse within 5e-6 absolute.  Measured on
B200 (profiles/r02_parity_small.md): worst rel_diff 5.3e-3 (dq_total), lse 1.2e-6."""
import numpy as np
import pytest
import torch

import _cases as cases
from oracle import oracle as O
from paper_2509_24006_b200 import SLA, SlaConfig

pytestmark = pytest.mark.gpu
TOL = 1.2e-2
LSE_TOL = 5e-6


def _inputs(seed, n, d, units=1):
    rng = O.Rng(seed)
    bf = O.to_bf16_exact
    xs = [dict(q=bf(rng.gaussian(n, d)), k=bf(rng.gaussian(n, d)), v=bf(rng.gaussian(n, d)),
               do=bf(rng.gaussian(n, d))) for _ in range(units)]
    w = bf(rng.gaussian(d, d, 0.1))
    return xs, w


def _T(a):
    return torch.tensor(np.array(a), dtype=torch.float32).to("cuda", torch.bfloat16).contiguous()


def _run(xs, w, n, d, cfg, labels=None, with_w=True, backward=True):
    U = len(xs)
    op = SLA(1, U, n, d, 64, 64, cfg, torch.bfloat16)
    assert op.path == "tcgen05"
    q, k, v, do = (_T([[x[nm] for x in xs]]) for nm in ("q", "k", "v", "do"))
    wt = _T([w] * U) if with_w else None
    mask = None if labels is None else torch.tensor(np.array([labels]), dtype=torch.int8)
    st = op.forward(q, k, v, wt, mask=mask)
    g = op.backward(st, q, k, v, wt, do) if backward else None
    torch.cuda.synchronize()
    return op, st, g


def _check_unit(st, g, h, x, w, lab, phi, with_w=True, backward=True):
    assert (st.labels[0, h].cpu().numpy() == lab).all()
    want = O.step(x["q"], x["k"], x["v"], w if with_w else np.zeros_like(w), x["do"], lab, 64, 64, phi)
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    for name, got in (("o_s", st.o_s[0, h]), ("o_l", st.o_l[0, h])):
        err = O.rel_diff(f(got), want[name], 1.0)
        cases.log_err(name, err, tol=TOL)
        assert err <= TOL, f"{name} {err:.3e}"
    if with_w:
        err = O.rel_diff(f(st.o[0, h]), want["o"], 1.0)
        cases.log_err("o", err, tol=TOL)
        assert err <= TOL, f"o {err:.3e}"
    lse = st.lse[0, h].cpu().numpy()
    live = want["lse"] > -1e299
    assert (lse[~live] == np.float32(-1e30)).all()
    if live.any():
        cases.log_err("lse", np.abs(lse[live] - want["lse"][live]).max(), tol=LSE_TOL)
        assert np.abs(lse[live] - want["lse"][live]).max() <= LSE_TOL
    if backward:
        for name, got in (("dq_total", g.dq_total[0, h]), ("dk_total", g.dk_total[0, h]), ("dv", g.dv[0, h])):
            err = O.rel_diff(f(got), want[name], 1.0)
            cases.log_err(name, err, tol=TOL)
            assert err <= TOL, f"{name} {err:.3e}"
    return want


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("phi", ["softmax", "elu1", "relu"])
def test_fast_dynamic_mask(d, phi):
    n = 2048
    xs, w = _inputs(11 + d + len(phi), n, d, units=2)
    cfg = SlaConfig(k_h=5.0, k_l=10.0, phi=phi)
    op, st, g = _run(xs, w, n, d, cfg)
    dw = np.zeros((d, d))
    for h, x in enumerate(xs):
        lab = O.dynamic_labels(x["q"], x["k"], 64, 64, 5.0, 10.0)
        want = _check_unit(st, g, h, x, w, lab, phi)
        dw = want["dw"]
        assert O.rel_diff(g.dproj[h].double().cpu().numpy(), dw, 1.0) <= TOL


@pytest.mark.parametrize("kind", ["all_critical", "all_marginal", "all_negligible", "empty_rows", "random"])
def test_fast_injected_masks(kind):
    n, d = 1024, 128
    xs, w = _inputs(21, n, d)
    t = n // 64
    rng = O.Rng(5)
    if kind == "all_critical":
        lab = np.ones((t, t), np.int8)
    elif kind == "all_marginal":
        lab = np.zeros((t, t), np.int8)
    elif kind == "all_negligible":
        lab = -np.ones((t, t), np.int8)
    elif kind == "empty_rows":
        lab = rng.random_mask(t, t, 0.2, 0.5, allow_empty_critical=True)
        lab[3] = np.where(lab[3] == 1, 0, lab[3])
        lab[7] = -1
    else:
        lab = rng.random_mask(t, t, 0.3, 0.4)
    cfg = SlaConfig(k_h=5.0, k_l=10.0, phi="elu1")
    op, st, g = _run(xs, w, n, d, cfg, labels=[lab])
    _check_unit(st, g, 0, xs[0], w, lab, "elu1")


def test_fast_without_projection():
    n, d = 1024, 64
    xs, w = _inputs(31, n, d)
    cfg = SlaConfig(k_h=10.0, k_l=10.0, phi="softmax")
    op, st, _ = _run(xs, w, n, d, cfg, with_w=False, backward=False)
    lab = O.dynamic_labels(xs[0]["q"], xs[0]["k"], 64, 64, 10.0, 10.0)
    _check_unit(st, None, 0, xs[0], w, lab, "softmax", with_w=False, backward=False)


def test_fast_matches_generic_kernels_wan_heads():
    """Two heads at the Wan2.1 shape: tcgen05 path vs the SIMT path on identical inputs."""
    n, d = 32768, 128
    g0 = torch.Generator(device="cuda").manual_seed(7)
    shape = (1, 2, n, d)
    q, k, v, do = (torch.randn(shape, generator=g0, device="cuda").to(torch.bfloat16) for _ in range(4))
    w = (torch.randn((2, d, d), generator=g0, device="cuda") * 0.1).to(torch.bfloat16)
    outs = {}
    for generic in (False, True):
        op = SLA(1, 2, n, d, 64, 64, SlaConfig(k_h=5.0, k_l=10.0, phi="softmax", force_generic=generic),
                 torch.bfloat16)
        st = op.forward(q, k, v, w)
        gr = op.backward(st, q, k, v, w, do)
        torch.cuda.synchronize()
        outs[generic] = (st, gr)
    a, b = outs[False], outs[True]
    assert torch.equal(a[0].labels, b[0].labels)
    for x, y, nm in ((a[0].o, b[0].o, "o"), (a[0].o_s, b[0].o_s, "o_s"), (a[0].o_l, b[0].o_l, "o_l"),
                     (a[1].dq_total, b[1].dq_total, "dq"), (a[1].dk_total, b[1].dk_total, "dk"),
                     (a[1].dv, b[1].dv, "dv")):
        err = ((x.float() - y.float()).abs().max() / y.float().abs().max().clamp_min(1.0)).item()
        assert err <= TOL, f"{nm} {err:.3e}"
