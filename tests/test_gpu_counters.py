"""Device accounting: flops_report and ExecCounters computed on
the GPU from the block LUT the classification / forward left in the state
(csrc/counters.cu, sla_b200_flops_report / sla_b200_exec_counters), against the oracle's
restatement (pinned to the reference in tests/test_counters.py) and, where oracle/_ref was
built, the reference itself.  Counts are integers: exact equality."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2509_24006_b200 import SLA, SlaConfig

pytestmark = pytest.mark.gpu


def _unit_inputs(units, n, d, seed):
    xs = []
    for u in range(units):
        rng = O.Rng(seed + u)
        q, k, v = (O.to_bf16_exact(rng.gaussian(n, d)) for _ in range(3))
        q[5] = -np.abs(q[5]) - 0.25  # a relu zero row
        xs.append((q, k, v))
    return xs


def _dev(arrs, dtype):
    return torch.tensor(np.array(arrs), dtype=torch.float32, device="cuda").to(dtype).unsqueeze(0).contiguous()


@pytest.mark.parametrize("phi", ["elu1", "relu", "softmax"])
@pytest.mark.parametrize("b,dtype,generic", [(64, torch.bfloat16, False), (16, torch.float32, True)])
def test_exec_counters_and_flops_match_oracle(phi, b, dtype, generic):
    units, n, d = 3, 1024, 64
    xs = _unit_inputs(units, n, d, 900)
    t = n // b
    masks = [O.Rng(950 + u).random_mask(t, t, *fr) for u, fr in enumerate([(0.3, 0.4), (0.05, 0.9), (0.4, 0.1)])]
    masks[0][2] = -1  # a block row with no marginal block: no linear rows, no aggregation
    q, k, v = (_dev([x[i] for x in xs], dtype) for i in range(3))
    op = SLA(1, units, n, d, b, b, SlaConfig(phi=phi, force_generic=generic), dtype)
    st = op.forward(q, k, v, mask=torch.tensor(np.array(masks)).unsqueeze(0))
    torch.cuda.synchronize()
    fl = op.flops_report(st)
    for u in range(units):
        f = O.flops(n, d, b, b, masks[u])
        got = fl[u]
        assert [got[x] for x in ("full_flops", "sparse_flops", "linear_flops", "proj_flops", "mask_flops",
                                 "sla_total")] == [f[x] for x in ("full", "sparse", "linear", "proj", "mask", "total")]
        assert got["ratio"] == f["total"] / f["full"]
        assert got["sparsity"] == 1.0 - (masks[u] == 1).sum() / masks[u].size
    keys = ("sparse_block_matmuls", "linear_row_products", "additions", "subtractions", "lookups",
            "table_build_additions")
    for agg in ("direct", "complement", "four_russians", "auto"):
        got = op.exec_counters(st, q, agg, 4)
        want = np.sum([O.exec_counters(*xs[u][:2], masks[u], b, b, phi, agg, 4) for u in range(units)], axis=0)
        assert [got[x] for x in keys] == [int(w) for w in want], agg
        if O.Reference.available() and dtype == torch.float32:
            ref = np.sum([O.Reference.exec_counters(*xs[u], masks[u], b, b, phi, agg, 4) for u in range(units)],
                         axis=0)
            assert [got[x] for x in keys] == [int(w) for w in ref], agg


def test_counters_of_a_dynamic_mask_c1():
    """C1: the dynamic mask's counts, 1 / 2 / 13 per row."""
    n, d, b = 1024, 64, 64
    xs = _unit_inputs(2, n, d, 40)
    q, k, v = (_dev([x[i] for x in xs], torch.bfloat16) for i in range(3))
    op = SLA(1, 2, n, d, b, b, SlaConfig(k_h=5.0, k_l=10.0, phi="softmax"), torch.bfloat16)
    st = op.forward(q, k, v)
    c = op.exec_counters(st, q)
    assert c["sparse_block_matmuls"] == 2 * 2 * 16 * 1
    assert c["additions"] == 2 * 16 * 12 and c["subtractions"] == 0
    fl = op.flops_report(st)
    assert all(f["sparsity"] == 1.0 - 1 / 16 for f in fl)


def test_counters_reject_bad_strategy_and_group():
    op = SLA(1, 1, 1024, 64, 64, 64, SlaConfig(), torch.bfloat16)
    q = torch.randn((1, 1, 1024, 64), device="cuda").bfloat16()
    st = op.forward(q, q, q)
    with pytest.raises(ValueError, match="unknown aggregation"):
        op.exec_counters(st, q, "sparse")
    with pytest.raises(ValueError, match="g > 20"):
        op.exec_counters(st, q, "four_russians", 21)
