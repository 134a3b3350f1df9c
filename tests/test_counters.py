"""Device accounting, CPU half: the oracle's restatement of
flops_report (flops.cpp:7-33) and of the forward's ExecCounters (forward.hpp:46-50,
forward.cpp:117-161, aggregation.cpp:40-156) pinned against the reference itself
(oracle/_ref) and the reference's own flops tests (core_test.cpp:85-150)."""
import numpy as np
import pytest

from oracle import oracle as O

needs_ref = pytest.mark.skipif(not O.Reference.available(), reason="oracle/_ref not built")


def _inputs(seed, n, d, relu_zero_rows=()):
    rng = O.Rng(seed)
    q, k, v = (O.to_bf16_exact(rng.gaussian(n, d)) for _ in range(3))
    for r in relu_zero_rows:  # relu empties these rows' features: den == 0 (forward.cpp:136)
        q[r] = -np.abs(q[r]) - 0.25
    return q, k, v


@needs_ref
@pytest.mark.parametrize("phi", ["elu1", "relu", "softmax"])
@pytest.mark.parametrize("fractions", [(0.3, 0.4), (0.05, 0.1), (0.1, 0.85), (0.5, 0.45)])
def test_exec_counters_restatement_matches_reference(phi, fractions):
    n, d, b = 256, 16, 16
    q, k, v = _inputs(11, n, d, relu_zero_rows=(3, 40, 41, 200))
    lab = O.Rng(12).random_mask(n // b, n // b, *fractions)
    for agg in ("direct", "complement", "four_russians", "auto"):
        for g in (1, 3, 4, 16):
            want = O.Reference.exec_counters(q, k, v, lab, b, b, phi, agg, g)
            assert O.exec_counters(q, k, lab, b, b, phi, agg, g) == want, (agg, g)
    if phi == "relu":  # the zero rows really are skipped
        assert O.exec_counters(q, k, lab, b, b, phi)[1] < n


@needs_ref
def test_flops_restatement_matches_reference():
    for seed, (n, d, b) in enumerate([(1024, 32, 32), (256, 16, 16), (512, 64, 64)]):
        lab = O.Rng(70 + seed).random_mask(n // b, n // b, 0.25, 0.5)
        u, ratio, sparsity = O.Reference.flops_report(n, d, b, b, lab)
        f = O.flops(n, d, b, b, lab)
        assert [f[x] for x in ("full", "sparse", "linear", "proj", "mask", "total")] == u
        assert ratio == f["total"] / f["full"]
        assert sparsity == 1.0 - (lab == 1).sum() / lab.size


def test_flops_known_answers():  # core_test.cpp:106-150
    t = 16
    f = O.flops(256, 16, 16, 16, np.ones((t, t), np.int8))
    assert f["total"] / f["full"] >= 1.0 and f["linear"] == 0
    f = O.flops(256, 16, 16, 16, -np.ones((t, t), np.int8))
    assert f["total"] == f["proj"] + f["mask"]
    prev = -1.0
    for p1 in (0.05, 0.1, 0.2, 0.3, 0.4, 0.5):
        rng = O.Rng(11)
        u = np.array([rng.uniform() for _ in range(32 * 32)]).reshape(32, 32)
        lab = np.where(u < p1, 1, np.where((u >= 0.5) & (u < 0.75), 0, -1)).astype(np.int8)
        f = O.flops(512, 16, 16, 16, lab)
        assert f["total"] / f["full"] >= prev
        prev = f["total"] / f["full"]


def test_resolve_strategy_thresholds():  # aggregation.cpp:147-156, config.hpp:30-31
    assert O.resolve_strategy(O.AGG["auto"], 0.25) == O.AGG["direct"]
    assert O.resolve_strategy(O.AGG["auto"], 0.5) == O.AGG["four_russians"]
    assert O.resolve_strategy(O.AGG["auto"], 0.75) == O.AGG["complement"]
    assert O.resolve_strategy(O.AGG["complement"], 0.1) == O.AGG["complement"]
