"""GPU parity tests: the CUDA path (through the C-ABI) against the C oracle and the
reference's golden vectors on identical inputs.

Tolerances (rel_diff = max|a-b| / max(max|b|, 1), mat.hpp:169-178 with floor 1.0):
  * labels: bit-exact (f64 mask path); the f32 mask variant may only flip near-ties.
  * f32 inputs (generic kernels, fp32 arithmetic): 1e-4, the reference's own f32 gate
    (acceptance_main.cpp:51-102).
  * bf16 inputs (fp32 accumulation, bf16 outputs): 1.5e-2 for outputs and gradients (measured
    worst 6.7e-3, dq_total at b = 64 d = 64; profiles/r02_parity_small.md), lse 1e-4.
"""
import os

import numpy as np
import pytest
import torch

import _cases as cases
from oracle import oracle as O
from paper_2509_24006_b200 import SLA, SlaConfig

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DEV = "cuda"
BF16_TOL = 1.5e-2
BF16_LSE_TOL = 1e-4


def _t(x, dtype):
    return torch.tensor(np.ascontiguousarray(x), dtype=torch.float64).to(DEV, dtype).contiguous()


def _np(t):
    return t.detach().to(torch.float64).cpu().numpy()


def _run_step(x, b, phi, dtype, labels=None, k_h=5.0, k_l=10.0, generic=False, parts=False):
    n, d = x["q"].shape
    cfg = SlaConfig(k_h=k_h, k_l=k_l, phi=phi, force_generic=generic)
    op = SLA(1, 1, n, d, b, b, cfg, dtype)
    q, k, v, w, do = (_t(x[nm], dtype).view(1, 1, *x[nm].shape) for nm in ("q", "k", "v", "w", "do"))
    w = w.view(1, d, d)
    mask = None if labels is None else torch.tensor(labels, dtype=torch.int8).view(1, 1, *labels.shape)
    st = op.forward(q, k, v, w, mask=mask)
    g = op.backward(st, q, k, v, w, do, parts=parts)
    torch.cuda.synchronize()
    out = dict(o=_np(st.o)[0, 0], o_s=_np(st.o_s)[0, 0], o_l=_np(st.o_l)[0, 0],
               lse=_np(st.lse)[0, 0], labels=st.labels.cpu().numpy()[0, 0],
               dq_total=_np(g.dq_total)[0, 0], dk_total=_np(g.dk_total)[0, 0],
               dv=_np(g.dv)[0, 0], dw=_np(g.dproj)[0])
    if parts:
        for nm in ("dq", "dk", "dq_feat", "dk_feat"):
            out[nm] = _np(getattr(g, nm))[0, 0]
    return out, op


def _close(got, want, tol, keys=("o", "o_s", "o_l", "dq_total", "dk_total", "dv", "dw")):
    for key in keys:
        err = O.rel_diff(got[key], want[key], 1.0)
        cases.log_err(key, err, tol=tol)
        assert err <= tol, f"{key}: rel_diff {err:.3e} > {tol}"


def _lse_close(got, want, tol):
    live = want > -1e29
    assert np.all(got[~live] == np.float32(-1e30))
    if live.any():
        cases.log_err("lse", np.abs(got[live] - want[live]).max(), tol=tol)
        assert np.abs(got[live] - want[live]).max() <= tol


# ---------------------------------------------------------------------------------------
# masks (K1+K2): bit-exact against the reference at C1 and at the Wan2.1 shape
# ---------------------------------------------------------------------------------------
def _classify(q, k, b, k_h, k_l, precision="f64", dtype=torch.bfloat16, weights=False):
    n, d = q.shape
    op = SLA(1, 1, n, d, b, b, SlaConfig(k_h=k_h, k_l=k_l, mask_precision=precision), dtype)
    out = op.classify(_t(q, dtype).view(1, 1, n, d), _t(k, dtype).view(1, 1, n, d), weights=weights)
    torch.cuda.synchronize()
    if weights:
        return out[0].cpu().numpy()[0, 0], out[1].cpu().numpy()[0, 0]
    return out.cpu().numpy()[0, 0]


@pytest.mark.parametrize("name", list(cases.C2_MASKS))
def test_mask_bit_exact_wan_shape(name):
    seed, peaked = cases.C2_MASKS[name]
    q, k = cases.c2_qk(seed, peaked)
    g = np.load(os.path.join(GOLDEN, "c2_masks.npz"))
    lab = _classify(q, k, 64, 5.0, 10.0)
    flips = int((lab != g[f"{name}/labels"]).sum())
    assert flips == 0, f"{flips} label flips vs reference"


def test_mask_weights_match_reference_predict():
    q, k = cases.c2_qk(7, False, n=4096)
    lab, p_c = _classify(q, k, 64, 5.0, 10.0, weights=True)
    ref = O.predict(q, k, 64, 64)
    assert np.abs(p_c - ref).max() <= 4 * np.finfo(np.float64).eps * ref.max()
    assert (lab == O.classify(ref, 5.0, 10.0)).all()


def test_mask_bit_exact_many_seeds_c1():
    flips = 0
    for seed in range(40):
        rng = O.Rng(90000 + seed)
        q, k = O.to_bf16_exact(rng.gaussian(1024, 64)), O.to_bf16_exact(rng.gaussian(1024, 64))
        lab = _classify(q, k, 64, 5.0, 10.0)
        flips += int((lab != O.dynamic_labels(q, k, 64, 64, 5.0, 10.0)).sum())
    assert flips == 0


@pytest.mark.parametrize("t_n,k_h,k_l", [(16, 25, 25), (40, 20, 30), (128, 2.5, 10), (1182, 5, 10)])
def test_mask_counts_and_order_statistics(t_n, k_h, k_l):
    rng = O.Rng(777 + t_n)
    n = t_n * 16
    q, k = O.to_bf16_exact(rng.gaussian(n, 32)), O.to_bf16_exact(rng.gaussian(n, 32))
    lab = _classify(q, k, 16, k_h, k_l)
    want = O.dynamic_labels(q, k, 16, 16, k_h, k_l)
    n1, nn = O.counts(t_n, k_h, k_l)
    assert ((lab == 1).sum(1) == n1).all() and ((lab == -1).sum(1) == nn).all()
    assert (lab == want).all()


def test_mask_f32_variant_flips_only_on_near_ties():
    q, k = cases.c2_qk(8, False)
    g = np.load(os.path.join(GOLDEN, "c2_masks.npz"))
    lab = _classify(q, k, 64, 5.0, 10.0, precision="f32")
    ref = g["iid_s8/labels"]
    bad_rows = np.where((lab != ref).any(1))[0]
    p_c = O.predict(q, k, 64, 64)
    for i in bad_rows:  # every disagreement must sit on a boundary gap of a few f32 ulps
        srt = np.sort(p_c[i])[::-1]
        gaps = [abs(srt[25] - srt[26]) / srt[25], abs(srt[-52] - srt[-51]) / srt[-52]]
        assert min(gaps) < 1e-5, (i, gaps)
    print(f"f32 mask: {len(bad_rows)} rows of 512 differ (near-tie)")


# ---------------------------------------------------------------------------------------
# forward + backward against the golden reference steps (reference test shapes)
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("c", cases.SMALL, ids=[c["name"] for c in cases.SMALL])
def test_step_f32_generic_matches_reference(c):
    g = np.load(os.path.join(GOLDEN, "small_steps.npz"))
    x = cases.small_inputs(c)
    got, op = _run_step(x, c["b"], c["phi"], torch.float32, labels=x["labels"], generic=True)
    want = {key: g[f"{c['name']}/f32/{key}"] for key in ("o", "o_s", "o_l", "lse", "dq_total", "dk_total", "dv", "dw")}
    assert (got["labels"] == x["labels"]).all()
    _close(got, want, 1e-4)
    _lse_close(got["lse"], want["lse"], 1e-4)


@pytest.mark.parametrize("c", cases.SMALL, ids=[c["name"] for c in cases.SMALL])
def test_step_bf16_matches_oracle(c):
    x = {k: (O.to_bf16_exact(v) if v.dtype != np.int8 else v) for k, v in cases.small_inputs(c).items()}
    got, _ = _run_step(x, c["b"], c["phi"], torch.bfloat16, labels=x["labels"])
    want = O.step(x["q"], x["k"], x["v"], x["w"], x["do"], x["labels"], c["b"], c["b"], c["phi"])
    _close(got, want, BF16_TOL)
    _lse_close(got["lse"], want["lse"], BF16_LSE_TOL)


def test_step_parts_match_oracle():
    c = cases.SMALL[0]
    x = cases.small_inputs(c)
    got, _ = _run_step(x, c["b"], c["phi"], torch.float32, labels=x["labels"], generic=True, parts=True)
    want = O.step(x["q"], x["k"], x["v"], x["w"], x["do"], x["labels"], c["b"], c["b"], c["phi"])
    _close(got, want, 1e-4, keys=("dq", "dk", "dq_feat", "dk_feat"))


def test_c1_step_bf16_matches_reference():
    """BASELINE configs[0]: B=1 H=2 N=1024 d=64 b=64 k_h=5 k_l=10 (dynamic mask)."""
    g = np.load(os.path.join(GOLDEN, "c1_step.npz"))
    for h in range(cases.C1["heads"]):
        x = cases.c1_inputs(h)
        got, op = _run_step(x, 64, cases.C1["phi"], torch.bfloat16)
        assert (got["labels"] == g[f"h{h}/labels"]).all()
        _lse_close(got["lse"], g[f"h{h}/lse"], BF16_LSE_TOL)
        if h == 0:
            _close(got, {k: g[f"h0/{k}"] for k in ("o", "dq_total", "dk_total", "dv", "dw")}, BF16_TOL,
                   keys=("o", "dq_total", "dk_total", "dv", "dw"))


# ---------------------------------------------------------------------------------------
# edge cases the reference tests pin
# ---------------------------------------------------------------------------------------
def _small_x(seed, n=64, d=8):
    rng = O.Rng(seed)
    return dict(q=rng.gaussian(n, d), k=rng.gaussian(n, d), v=rng.gaussian(n, d),
                w=rng.gaussian(d, d, 0.5), do=rng.gaussian(n, d))


@pytest.mark.parametrize("fill", [1, 0, -1])
def test_degenerate_masks(fill):  # forward_test.cpp:60-85; all-negligible -> zeros
    x = _small_x(32)
    lab = np.full((4, 4), fill, np.int8)
    got, _ = _run_step(x, 16, "elu1", torch.float32, labels=lab, generic=True)
    want = O.step(x["q"], x["k"], x["v"], x["w"], x["do"], lab, 16, 16, "elu1")
    _close(got, want, 1e-4)
    if fill != 1:
        assert np.abs(got["o_s"]).max() == 0 and (got["lse"] == np.float32(-1e30)).all()
    if fill != 0:
        assert np.abs(got["o_l"]).max() == 0


def test_rows_without_critical_blocks():  # mask.hpp:21-23
    x = _small_x(41, n=128, d=16)
    rng = O.Rng(41)
    lab = rng.random_mask(8, 8, 0.2, 0.5, allow_empty_critical=True)
    lab[3] = np.where(lab[3] == 1, 0, lab[3])
    got, _ = _run_step(x, 16, "softmax", torch.float32, labels=lab, generic=True)
    want = O.step(x["q"], x["k"], x["v"], x["w"], x["do"], lab, 16, 16, "softmax")
    _close(got, want, 1e-4)
    assert (got["lse"][48:64] == np.float32(-1e30)).all()


def test_relu_zero_denominator_rows():  # backward_test.cpp:247-264
    rng = O.Rng(58)
    q = rng.gaussian(16, 4)
    q[2] = -np.abs(q[2]) - 0.5
    x = dict(q=q, k=rng.gaussian(16, 4), v=rng.gaussian(16, 4), w=np.eye(4), do=rng.gaussian(16, 4))
    lab = np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1], np.int8).reshape(4, 4)
    got, _ = _run_step(x, 4, "relu", torch.float32, labels=lab, generic=True, parts=True)
    assert (got["o_l"][2] == 0).all() and (got["dq_feat"][2] == 0).all()


def test_zero_cotangent_gives_zero_gradients():  # backward_test.cpp:59-73
    x = _small_x(51, n=32, d=4)
    x["do"] = np.zeros_like(x["do"])
    lab = O.Rng(51).random_mask(4, 4)
    got, _ = _run_step(x, 8, "elu1", torch.float32, labels=lab, generic=True)
    for key in ("dq_total", "dk_total", "dv", "dw"):
        assert np.abs(got[key]).max() == 0


def test_non_finite_input_reports_coordinates():  # forward_test.cpp:271-281
    x = _small_x(43, n=32, d=4)
    q = _t(x["q"], torch.float32).view(1, 1, 32, 4)
    q[0, 0, 5, 2] = float("inf")
    op = SLA(1, 1, 32, 4, 8, 8, SlaConfig(check_finite=True), torch.float32)
    k, v = (_t(x[n], torch.float32).view(1, 1, 32, 4) for n in ("k", "v"))
    with pytest.raises(ValueError, match=r"Q has non-finite entry at \(5, 2\)"):
        op.forward(q, k, v, mask=torch.ones(1, 1, 4, 4, dtype=torch.int8))


def test_invalid_label_rejected_when_checking():
    x = _small_x(44, n=32, d=4)
    op = SLA(1, 1, 32, 4, 8, 8, SlaConfig(check_finite=True), torch.float32)
    q, k, v = (_t(x[n], torch.float32).view(1, 1, 32, 4) for n in ("q", "k", "v"))
    bad = torch.ones(1, 1, 4, 4, dtype=torch.int8)
    bad[0, 0, 1, 1] = 3
    with pytest.raises(ValueError, match="label must be -1, 0 or 1"):
        op.forward(q, k, v, mask=bad)


def test_batched_units_match_per_unit_oracle():
    B, H, n, d, b = 2, 3, 128, 16, 16
    rng = O.Rng(4242)
    q = [[rng.gaussian(n, d) for _ in range(H)] for _ in range(B)]
    k = [[rng.gaussian(n, d) for _ in range(H)] for _ in range(B)]
    v = [[rng.gaussian(n, d) for _ in range(H)] for _ in range(B)]
    w = [rng.gaussian(d, d, 0.5) for _ in range(H)]
    do = [[rng.gaussian(n, d) for _ in range(H)] for _ in range(B)]
    cfg = SlaConfig(k_h=25, k_l=25, phi="softmax", force_generic=True)
    op = SLA(B, H, n, d, b, b, cfg, torch.float32)
    T = lambda a: _t(np.array(a), torch.float32)  # noqa: E731
    st = op.forward(T(q), T(k), T(v), T(w))
    g = op.backward(st, T(q), T(k), T(v), T(w), T(do))
    dw_sum = [np.zeros((d, d)) for _ in range(H)]
    for bi in range(B):
        for h in range(H):
            lab = O.dynamic_labels(q[bi][h], k[bi][h], b, b, 25, 25)
            assert (st.labels[bi, h].cpu().numpy() == lab).all()
            want = O.step(q[bi][h], k[bi][h], v[bi][h], w[h], do[bi][h], lab, b, b, "softmax")
            assert O.rel_diff(_np(st.o[bi, h]), want["o"], 1.0) <= 1e-4
            assert O.rel_diff(_np(g.dq_total[bi, h]), want["dq_total"], 1.0) <= 1e-4
            assert O.rel_diff(_np(g.dk_total[bi, h]), want["dk_total"], 1.0) <= 1e-4
            assert O.rel_diff(_np(g.dv[bi, h]), want["dv"], 1.0) <= 1e-4
            dw_sum[h] += want["dw"]
    for h in range(H):  # W is per head and shared over the batch
        assert O.rel_diff(_np(g.dproj[h]), dw_sum[h], 1.0) <= 1e-4
