"""GPU tests of the reference-facing boundary beyond the fused training step:

  * sla_backward with INDEPENDENT cotangents (backward.hpp:25-38): dO^s and dO^l unrelated
    through W, as the reference accepts them -- sla_b200_backward_split on both paths;
  * the SlaGradients parts (dq, dk, dq_feat, dk_feat; backward.hpp:10-16) on the tcgen05 path;
  * combine_outputs (forward.cpp:187-195) and proj_backward (backward.cpp:12-22) on the device;
  * a forward state rebuilt around outputs the caller holds (sla_b200_build_state), as the C++
    drop-in's sla_backward uses it.

Checked against the C oracle (f64, reference order) on bf16-exact inputs.  Gates: bf16 path 1.5e-2
(rel_diff floor 1.0, see test_gpu_parity.py), f32 generic path 1e-4 (the reference's f32 gate)."""
import numpy as np
import pytest
import torch

import _cases as cases
from oracle import oracle as O
from paper_2509_24006_b200 import SLA, SlaConfig, sla_backward

pytestmark = pytest.mark.gpu
BF16_TOL, F32_TOL = 1.5e-2, 1e-4


def _inputs(seed, n, d):
    rng = O.Rng(seed)
    bf = O.to_bf16_exact
    x = {nm: bf(rng.gaussian(n, d)) for nm in ("q", "k", "v", "do", "dos", "dol")}
    x["w"] = bf(rng.gaussian(d, d, 0.1))
    return x


def _t(a, dtype, shape):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64).to("cuda", dtype).reshape(shape).contiguous()


def _np(t):
    return t.detach().double().cpu().numpy()


def _close(got, want, tol, key):
    err = O.rel_diff(got, want, 1.0)
    cases.log_err(key, err, tol=tol)
    assert err <= tol, f"{key}: rel_diff {err:.3e} > {tol}"


@pytest.mark.parametrize("path", ["tcgen05", "generic_f32"])
@pytest.mark.parametrize("phi", ["softmax", "elu1"])
def test_backward_split_independent_cotangents(path, phi):
    n, d = (2048, 128) if path == "tcgen05" else (256, 16)
    b = 64 if path == "tcgen05" else 16
    dtype, tol = (torch.bfloat16, BF16_TOL) if path == "tcgen05" else (torch.float32, F32_TOL)
    x = _inputs(41 + len(phi), n, d)
    cfg = SlaConfig(k_h=10.0, k_l=20.0, phi=phi, force_generic=path != "tcgen05")
    op = SLA(1, 1, n, d, b, b, cfg, dtype)
    assert op.path == ("tcgen05" if path == "tcgen05" else "generic")
    T = lambda a: _t(a, dtype, (1, 1, n, d))  # noqa: E731
    q, k, v = T(x["q"]), T(x["k"]), T(x["v"])
    st = op.forward(q, k, v, _t(x["w"], dtype, (1, d, d)))
    lab = st.labels[0, 0].cpu().numpy()
    g = sla_backward(st, q, k, v, T(x["dos"]), T(x["dol"]), parts=True)
    torch.cuda.synchronize()
    ost = O.forward(x["q"], x["k"], x["v"], lab, b, b, phi, want_state=True)
    want = O.backward(x["q"], x["k"], x["v"], lab, ost, x["dos"], x["dol"], b, b, phi)
    for key, got in (("dq_total", g.dq_total), ("dk_total", g.dk_total), ("dv", g.dv), ("dq", g.dq),
                     ("dk", g.dk), ("dq_feat", g.dq_feat), ("dk_feat", g.dk_feat)):
        _close(_np(got)[0, 0], want[key], tol, key)
    _close(_np(g.dproj)[0], want["dproj"], tol, "dproj")


def test_combined_equals_split_with_projected_cotangent():
    """The fused call (dO^l = dO W^T in-kernel) against the split call on dO^l computed by
    sla_b200_proj_backward: the same gradients up to the bf16 rounding of dO^l."""
    n, d = 2048, 128
    x = _inputs(77, n, d)
    op = SLA(1, 1, n, d, 64, 64, SlaConfig(k_h=5.0, k_l=10.0, phi="softmax"), torch.bfloat16)
    T = lambda a: _t(a, torch.bfloat16, (1, 1, n, d))  # noqa: E731
    q, k, v, do = T(x["q"]), T(x["k"]), T(x["v"]), T(x["do"])
    w = _t(x["w"], torch.bfloat16, (1, d, d))
    st = op.forward(q, k, v, w)
    gc = op.backward(st, q, k, v, w, do)
    dos, dol, dw = op.proj_backward(do, st.o_l, w)
    gs = op.backward(st, q, k, v, None, dos, d_out_linear=dol)
    torch.cuda.synchronize()
    for key in ("dq_total", "dk_total", "dv", "dproj"):
        _close(_np(getattr(gs, key)), _np(getattr(gc, key)), 5e-3, key)
    assert torch.equal(dw, gc.dproj) or O.rel_diff(_np(dw), _np(gc.dproj), 1.0) <= 1e-5


def test_parts_on_tcgen05_path():
    n, d = 2048, 64
    x = _inputs(91, n, d)
    op = SLA(1, 1, n, d, 64, 64, SlaConfig(k_h=5.0, k_l=10.0, phi="softmax"), torch.bfloat16)
    assert op.path == "tcgen05"
    T = lambda a: _t(a, torch.bfloat16, (1, 1, n, d))  # noqa: E731
    q, k, v, do = T(x["q"]), T(x["k"]), T(x["v"]), T(x["do"])
    w = _t(x["w"], torch.bfloat16, (1, d, d))
    st = op.forward(q, k, v, w)
    g = op.backward(st, q, k, v, w, do, parts=True)
    torch.cuda.synchronize()
    lab = st.labels[0, 0].cpu().numpy()
    want = O.step(x["q"], x["k"], x["v"], x["w"], x["do"], lab, 64, 64, "softmax")
    for key in ("dq", "dk", "dq_feat", "dk_feat", "dq_total", "dk_total"):
        got = getattr(g, key)
        _close(_np(got)[0, 0], want[key], BF16_TOL, key)
    # the parts compose to the totals (backward.cpp:211-214) -- checked through the oracle's VJP
    recomposed = O.phi_vjp(x["q"], "softmax", _np(g.dq_feat)[0, 0]) + _np(g.dq)[0, 0]
    _close(_np(g.dq_total)[0, 0], recomposed, 1e-2, "dq_total=vjp(dq_feat)+dq")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_combine_and_proj_backward_on_device(dtype):
    n, d = 1024, 128
    x = _inputs(13, n, d)
    b = 64
    cfg = SlaConfig(k_h=5.0, k_l=10.0, phi="elu1", force_generic=dtype == torch.float32)
    op = SLA(1, 1, n, d, b, b, cfg, dtype)
    T = lambda a: _t(a, dtype, (1, 1, n, d))  # noqa: E731
    q, k, v, do = T(x["q"]), T(x["k"]), T(x["v"]), T(x["do"])
    w = _t(x["w"], dtype, (1, d, d))
    st = op.forward(q, k, v, w)
    o = op.combine(st, w)
    dos, dol, dw = op.proj_backward(do, st.o_l, w)
    torch.cuda.synchronize()
    tol = BF16_TOL if dtype == torch.bfloat16 else F32_TOL
    want_o = O.combine(_np(st.o_s)[0, 0], _np(st.o_l)[0, 0], x["w"])
    _close(_np(o)[0, 0], want_o, tol / 2, "combine")
    _close(_np(o)[0, 0], _np(st.o)[0, 0], tol / 2, "combine vs fused")
    ds_w, dl_w, dw_w = O.proj_backward(x["do"], _np(st.o_l)[0, 0], x["w"])
    assert dos.data_ptr() == do.data_ptr()
    _close(_np(dol)[0, 0], dl_w, tol / 2, "proj dO^l")
    _close(_np(dw)[0], dw_w, tol / 2, "proj dW")


def test_state_rebuilt_around_caller_outputs():
    """The drop-in's path: outputs of a forward the caller holds (here the oracle's, rounded to
    bf16) plus its label grid -> sla_b200_build_state -> split backward."""
    n, d = 1024, 128
    x = _inputs(57, n, d)
    lab = O.dynamic_labels(x["q"], x["k"], 64, 64, 5.0, 10.0)
    ost = O.forward(x["q"], x["k"], x["v"], lab, 64, 64, "softmax", want_state=True)
    op = SLA(1, 1, n, d, 64, 64, SlaConfig(k_h=5.0, k_l=10.0, phi="softmax"), torch.bfloat16)
    T = lambda a: _t(a, torch.bfloat16, (1, 1, n, d))  # noqa: E731
    q, k, v = T(x["q"]), T(x["k"]), T(x["v"])
    lse = torch.tensor(ost["lse"], dtype=torch.float32, device="cuda").reshape(1, 1, n)
    st = op.state_from(q, k, v, torch.tensor(lab).reshape(1, 1, *lab.shape), T(ost["o_s"]), T(ost["o_l"]), lse)
    assert (st.labels[0, 0].cpu().numpy() == lab).all()
    g = sla_backward(st, q, k, v, T(x["dos"]), T(x["dol"]), parts=True)
    torch.cuda.synchronize()
    want = O.backward(x["q"], x["k"], x["v"], lab, ost, x["dos"], x["dol"], 64, 64, "softmax")
    for key in ("dq_total", "dk_total", "dv", "dq", "dk", "dq_feat", "dk_feat"):
        _close(_np(getattr(g, key))[0, 0], want[key], BF16_TOL, key)
