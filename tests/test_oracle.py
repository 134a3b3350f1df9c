"""CPU tests: pin the C restatement (oracle/sla_oracle.c) against the reference's own
known-answer tests, against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and, when oracle/_ref exists, against the reference live.

Citations: /root/reference/proj/tests/*.cpp."""
import os

import numpy as np
import pytest

import _cases as cases
from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _npz(name):
    return np.load(os.path.join(GOLDEN, name))


# ---- mask_test.cpp ----------------------------------------------------------------------
def test_mean_pooling_known_answers():  # mask_test.cpp:9-26
    x = np.array([[1, 3], [3, 5]], float)
    p = O.pool_mean(x, 2)
    assert p.shape == (1, 2) and p[0, 0] == 2.0 and p[0, 1] == 4.0
    assert (O.pool_mean(x, 1) == x).all()
    c = np.full((6, 3), 4.25)
    assert (O.pool_mean(c, 3) == 4.25).all()
    with pytest.raises(ValueError):
        O.pool_mean(x, 3)


def test_predict_known_answers():  # mask_test.cpp:28-84
    z = np.zeros((32, 4))
    assert np.allclose(O.predict(z, z, 8, 8), 0.25, rtol=0, atol=1e-15)
    rng = O.Rng(3)
    q, k = rng.gaussian(32, 4), rng.gaussian(32, 4)
    assert np.allclose(O.predict(q, k, 8, 32), 1.0)
    rng = O.Rng(8)
    q, k = rng.gaussian(64, 8), rng.gaussian(64, 8)
    w = O.predict(q, k, 16, 16)
    pq = q.reshape(4, 16, 8).sum(1) / 16
    pk = k.reshape(4, 16, 8).sum(1) / 16
    s = pq @ pk.T / np.sqrt(8.0)
    ref = np.exp(s - s.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert O.rel_diff(w, ref) <= 1e-12
    assert np.allclose(w.sum(1), 1.0, atol=1e-10)


def test_classification_known_answers():  # mask_test.cpp:86-162
    assert O.classify(np.array([[0.4, 0.3, 0.2, 0.1]]), 25, 25).tolist() == [[1, 0, 0, -1]]
    assert O.classify(np.array([[0.25] * 4]), 25, 25).tolist() == [[1, 0, 0, -1]]
    rng = O.Rng(21)
    m = O.classify(rng.uniform_mat(3, 512, 0.0, 1.0), 5, 10)
    assert ((m == 1).sum(1) == 26).all() and ((m == -1).sum(1) == 51).all() and ((m == 0).sum(1) == 435).all()
    rng = O.Rng(22)
    assert ((O.classify(rng.uniform_mat(4, 8, 0.0, 1.0), 1, 50) == 1).sum(1) >= 1).all()
    rng = O.Rng(24)
    w = rng.uniform_mat(6, 32, 0.0, 1.0)
    m = O.classify(w, 20, 30)
    for i in range(6):
        assert w[i][m[i] == 1].min() >= w[i][m[i] == 0].max() >= w[i][m[i] == -1].max()
    rng = O.Rng(25)
    w = rng.uniform_mat(4, 16, 0.0, 1.0)
    assert (O.classify(w, 25, 25) == O.classify(0.3 * w + 7.0, 25, 25)).all()
    with pytest.raises(ValueError):
        O.classify(w, 60, 50)


def test_counts_formula():  # mask.cpp:98-101
    assert O.counts(512, 5, 10) == (26, 51)
    assert O.counts(16, 5, 10) == (1, 2)
    assert O.counts(1182, 5, 10) == (59, 118)
    assert O.counts(128, 2.5, 10) == (3, 13)
    assert O.counts(4, 100, 0) == (4, 0)


# ---- forward_test.cpp --------------------------------------------------------------------
def test_summaries_hand_case():  # forward_test.cpp:23-57
    h, z = O.summaries(np.array([[1, 0], [0, 1.0]]), np.array([[2, 0], [0, 4.0]]), 2)
    assert h[0, 0, 0] == 2 and h[0, 1, 1] == 4 and h[0, 0, 1] == 0 and (z[0] == 1).all()
    rng = O.Rng(31)
    k, v = rng.gaussian(64, 8), rng.gaussian(64, 8)
    kf = O.phi(k, "elu1")
    h, _ = O.summaries(kf, v, 16)
    assert O.rel_diff(h.sum(0), kf.T @ v) <= 1e-12


def _naive_attention(q, k, v):
    s = q @ k.T / np.sqrt(q.shape[1])
    p = np.exp(s - s.max(1, keepdims=True))
    return (p / p.sum(1, keepdims=True)) @ v


def test_degenerate_masks():  # forward_test.cpp:60-85
    rng = O.Rng(32)
    q, k, v = rng.gaussian(64, 8), rng.gaussian(64, 8), rng.gaussian(64, 8)
    st = O.forward(q, k, v, np.ones((4, 4), np.int8), 16, 16)
    assert O.rel_diff(st["o_s"], _naive_attention(q, k, v)) <= 1e-10
    assert np.abs(st["o_l"]).max() == 0
    st = O.forward(q, k, v, np.zeros((4, 4), np.int8), 16, 16)
    qf, kf = O.phi(q, "elu1"), O.phi(k, "elu1")
    ref = (qf @ (kf.T @ v)) / (qf @ kf.sum(0))[:, None]
    assert O.rel_diff(st["o_l"], ref) <= 1e-10
    assert np.abs(st["o_s"]).max() == 0 and (st["lse"] == O.LSE_SENTINEL_F64).all()


def test_forward_known_relu_zero_rows():  # backward_test.cpp:247-264 (forward half)
    rng = O.Rng(58)
    q = rng.gaussian(16, 4)
    q[2] = -np.abs(q[2]) - 0.5
    k, v = rng.gaussian(16, 4), rng.gaussian(16, 4)
    lab = np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1], np.int8).reshape(4, 4)
    st = O.forward(q, k, v, lab, 4, 4, "relu")
    assert (st["o_l"][2] == 0).all()


def test_flops_ratio_published_point():  # acceptance_main.cpp:253-266
    rng = O.Rng(5000)
    lab = O.classify(rng.uniform_mat(512, 512, 0.0, 1.0), 5.0, 10.0)
    f = O.flops(32768, 128, 64, 64, lab)
    ratio = f["total"] / f["full"]
    assert abs(ratio - 0.054832) < 5e-7 and 0.050 <= ratio <= 0.055


def test_backward_finite_differences():  # acceptance_main.cpp:138-192 (3 of the 20 seeds)
    worst = 0.0
    for seed in (0, 1, 2):
        n, d, b = 16 * (1 + seed % 4), (8 if seed % 2 else 4), (8 if seed % 3 else 16)
        b = min(b, n)
        rng = O.Rng(3000 + seed)
        q, k, v = rng.gaussian(n, d), rng.gaussian(n, d), rng.gaussian(n, d)
        w = rng.gaussian(d, d, 0.5)
        lab = rng.random_mask(n // b, n // b)
        phi = ["softmax", "elu1", "relu"][seed % 3]

        def loss():
            st = O.forward(q, k, v, lab, b, b, phi)
            return 0.5 * (O.combine(st["o_s"], st["o_l"], w) ** 2).sum()

        st = O.forward(q, k, v, lab, b, b, phi, want_state=True)
        out = O.combine(st["o_s"], st["o_l"], w)
        g = O.step(q, k, v, w, out, lab, b, b, phi)
        for t, gr in ((q, g["dq_total"]), (k, g["dk_total"]), (v, g["dv"]), (w, g["dw"])):
            flat, gflat = t.reshape(-1), gr.reshape(-1)
            for e in range(0, flat.size, 5):
                s = flat[e]
                flat[e] = s + 1e-5
                up = loss()
                flat[e] = s - 1e-5
                dn = loss()
                flat[e] = s
                fd = (up - dn) / 2e-5
                worst = max(worst, abs(gflat[e] - fd) / max(1.0, abs(fd)))
    assert worst <= 1e-5


# ---- golden vectors made by the reference itself -----------------------------------------
@pytest.mark.parametrize("c", cases.SMALL, ids=[c["name"] for c in cases.SMALL])
def test_oracle_matches_reference_golden_small(c):
    g = _npz("small_steps.npz")
    x = cases.small_inputs(c)
    r = O.step(x["q"], x["k"], x["v"], x["w"], x["do"], x["labels"], c["b"], c["b"], c["phi"])
    for key in ("o", "o_s", "o_l", "dq_total", "dk_total", "dv", "dw"):
        if c["d"] <= 16:  # the f64 reference: bit-for-bit up to summation-free identity
            assert O.rel_diff(r[key], g[f"{c['name']}/f64/{key}"], 1.0) <= 1e-13, key
        assert O.rel_diff(r[key], g[f"{c['name']}/f32/{key}"], 1.0) <= 1e-4, key
    lse_ref = g[f"{c['name']}/f32/lse"]
    live = lse_ref > -1e29
    assert np.abs(r["lse"][live] - lse_ref[live]).max() <= 1e-4
    assert (r["lse"][~live] == O.LSE_SENTINEL_F64).all()


def test_oracle_matches_reference_golden_c1():
    g = _npz("c1_step.npz")
    for h in range(cases.C1["heads"]):
        x = cases.c1_inputs(h)
        lab = O.dynamic_labels(x["q"], x["k"], 64, 64, 5.0, 10.0)
        assert (lab == g[f"h{h}/labels"]).all()
        if h:
            continue
        r = O.step(x["q"], x["k"], x["v"], x["w"], x["do"], lab, 64, 64, cases.C1["phi"])
        for key in ("o", "dq_total", "dk_total", "dv", "dw"):
            assert O.rel_diff(r[key], g[f"h0/{key}"], 1.0) <= 1e-4, key


@pytest.mark.parametrize("name", list(cases.C2_MASKS))
def test_oracle_mask_matches_reference_golden_c2(name):
    seed, peaked = cases.C2_MASKS[name]
    q, k = cases.c2_qk(seed, peaked)
    lab = O.dynamic_labels(q, k, 64, 64, 5.0, 10.0)
    g = _npz("c2_masks.npz")
    assert (lab == g[f"{name}/labels"]).all()
    assert ((lab == 1).sum(1) == 26).all() and ((lab == -1).sum(1) == 51).all()


@pytest.mark.skipif(not O.Reference.available(), reason="oracle/_ref not built here")
def test_oracle_matches_reference_live():
    R = O.Reference
    for c in range(6):
        n, d, b = [64, 128, 256][c % 3], [8, 16][(c // 3) % 2], 16
        phi = ["elu1", "relu", "softmax"][c % 3]
        rng = O.Rng(1000 + c)
        q, k, v = rng.gaussian(n, d), rng.gaussian(n, d), rng.gaussian(n, d)
        lab = rng.random_mask(n // b, n // b)
        w, do = rng.gaussian(d, d, 0.5), rng.gaussian(n, d)
        ref = R.run(q, k, v, b, b, phi_kind=phi, w=w, labels=lab, d_out=do, dtype=np.float64)
        orc = O.step(q, k, v, w, do, lab, b, b, phi)
        for key in ("o_s", "o_l", "o", "dq_total", "dk_total", "dv", "dw", "dq", "dk", "dq_feat", "dk_feat"):
            assert (orc[key] == ref[key]).all(), key


def test_ragged_predict_restatement():
    """orc_predict_ragged (the SLA_B200_FLAG_RAGGED extension) equals predict bit for bit when
    b divides N, and pools the partial last block over its valid rows only."""
    rng = O.Rng(4242)
    q, k = O.to_bf16_exact(rng.gaussian(512, 16)), O.to_bf16_exact(rng.gaussian(512, 16))
    assert np.array_equal(O.predict_ragged(q, k, 64), O.predict(q, k, 64, 64))
    qr, kr = q[:500], k[:500]
    p = O.predict_ragged(qr, kr, 64)
    pool = lambda x: np.array([x[i * 64:min(500, (i + 1) * 64)].mean(0) for i in range(8)])  # noqa: E731
    s_ = pool(qr) @ pool(kr).T / 4.0
    want = np.exp(s_ - s_.max(1, keepdims=True))
    want /= want.sum(1, keepdims=True)
    assert p.shape == (8, 8) and np.allclose(p, want, rtol=1e-12, atol=0)
