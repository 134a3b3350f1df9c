"""GPU tests of the classification stage's rank kernel (classify.cu k_classify_rank): labels from
the raw pooled-score ranks, exact P_c only where a rank boundary is not strictly separated.

Labels must equal the reference's (mask.cpp:57-119, through the C oracle pinned to it) on
tie-heavy inputs (all-equal scores, duplicated key blocks), across T in {16 .. 2048} (and 2049,
the block-per-row kernel), on the forced-exact path (weights requested), and the exact fallback
must be rare on iid data (it is the slow path)."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2509_24006_b200 import SLA, SlaConfig
from paper_2509_24006_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _classify(q, k, b, k_h, k_l, weights=False, dtype=torch.bfloat16):
    n, d = q.shape
    op = SLA(1, 1, n, d, b, b, SlaConfig(k_h=k_h, k_l=k_l), dtype)
    t = lambda a: torch.tensor(a, dtype=torch.float64).to("cuda", dtype).view(1, 1, n, d)  # noqa: E731
    out = op.classify(t(q), t(k), weights=weights)
    torch.cuda.synchronize()
    return out[0].cpu().numpy()[0, 0] if weights else out.cpu().numpy()[0, 0]


class ExactRows:
    """Counts the rows k_classify_rank resolves through the exact P_c path."""

    def __enter__(self):
        self.c = torch.zeros(1, dtype=torch.int32, device="cuda")
        L.diag_lib().sla_b200_diag_classify_exact(C.c_void_p(self.c.data_ptr()))
        return self

    def __exit__(self, *a):
        L.diag_lib().sla_b200_diag_classify_exact(None)

    @property
    def value(self):
        torch.cuda.synchronize()
        return int(self.c.item())


def test_all_equal_scores_rank_by_index():
    """Q = 0: every pooled score is 0 (mask_test.cpp:96-103 -- ties resolve by column index)."""
    n, d, b = 1024, 64, 64
    rng = O.Rng(3)
    q = np.zeros((n, d))
    k = O.to_bf16_exact(rng.gaussian(n, d))
    with ExactRows() as ex:
        lab = _classify(q, k, b, 25.0, 25.0)
    assert (lab == O.dynamic_labels(q, k, b, b, 25.0, 25.0)).all()
    t = n // b
    assert (lab[:, :4] == 1).all() and (lab[:, -4:] == -1).all()
    assert ex.value == 0  # a single tie class and nothing above or below it: no exact pass needed
    _ = t


@pytest.mark.parametrize("distinct", [3, 8, 37])
def test_duplicated_key_blocks(distinct):
    """Key blocks repeat with period `distinct`: every score value appears T / distinct times, so
    tie classes straddle both rank boundaries."""
    n, d, b = 8192, 64, 64
    rng = O.Rng(100 + distinct)
    q = O.to_bf16_exact(rng.gaussian(n, d))
    blocks = O.to_bf16_exact(rng.gaussian(distinct * b, d)).reshape(distinct, b, d)
    k = np.concatenate([blocks[j % distinct] for j in range(n // b)])
    lab = _classify(q, k, b, 5.0, 10.0)
    assert (lab == O.dynamic_labels(q, k, b, b, 5.0, 10.0)).all()


@pytest.mark.parametrize("t_n,b,d", [(16, 64, 64), (65, 64, 64), (100, 16, 32), (300, 16, 32), (512, 64, 128),
                                     (600, 16, 32), (1182, 64, 128), (2048, 16, 32), (2049, 16, 32)])
def test_rank_kernel_matches_reference_across_t(t_n, b, d):
    rng = O.Rng(5000 + t_n)
    n = t_n * b
    q, k = O.to_bf16_exact(rng.gaussian(n, d)), O.to_bf16_exact(rng.gaussian(n, d))
    with ExactRows() as ex:
        lab = _classify(q, k, b, 5.0, 10.0)
    want = O.dynamic_labels(q, k, b, b, 5.0, 10.0)
    assert (lab == want).all(), int((lab != want).sum())
    if t_n <= 2048:
        assert ex.value <= max(1, t_n // 100), ex.value  # iid scores: near-ties at 2^-50 are rare


def test_forced_exact_path_agrees():
    """weights=True makes every row take the exact P_c path; the labels must not change."""
    n, d, b = 32768, 128, 64
    rng = O.Rng(11)
    q, k = O.to_bf16_exact(rng.gaussian(n, d)), O.to_bf16_exact(rng.gaussian(n, d))
    lab_fast = _classify(q, k, b, 5.0, 10.0)
    with ExactRows() as ex:
        lab_exact = _classify(q, k, b, 5.0, 10.0, weights=True)
    assert ex.value == n // b
    assert (lab_fast == lab_exact).all()
