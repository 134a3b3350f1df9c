"""CPU tests of the C-ABI boundary (no GPU compute): the library loads, exports every entry
point include/sla_b200.h declares, and validates problems with the reference's messages
(layout.cpp:8-26, config.cpp:7-19, mask.cpp:98-101)."""
import ctypes as C
import os
import re

import pytest

from paper_2509_24006_b200 import _lib as L
from paper_2509_24006_b200 import sla as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "sla_b200.h")).read()
    return sorted(set(re.findall(r"\b(sla_b200_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    names = _declared()
    assert len(names) >= 10
    for nm in names:
        assert hasattr(lib, nm), nm
    assert lib.sla_b200_abi_version() == 2


def _p(**kw):
    base = dict(batch=1, heads=1, n=1024, d=64, b_q=64, b_kv=64, k_h=5.0, k_l=10.0)
    base.update(kw)
    p = L.Problem()
    for k, v in base.items():
        setattr(p, k, v)
    p.phi, p.dtype, p.mask_precision, p.flags = 0, L.DTYPE_BF16, L.MASK_F64, 0
    return p


@pytest.mark.parametrize("kw,msg", [
    (dict(n=32760, d=128), "make_block_layout: b_q=64 does not divide N=32760"),
    (dict(b_kv=48), "make_block_layout: b_kv=48 does not divide N=1024"),
    (dict(n=0), "make_block_layout: all sizes must be positive"),
    (dict(k_h=0.0), "config: k_h must be in (0, 100]"),
    (dict(k_h=101.0), "config: k_h must be in (0, 100]"),
    (dict(k_l=100.0), "config: k_l must be in [0, 100)"),
    (dict(k_h=60.0, k_l=50.0), "config: k_h + k_l must be <= 100"),
])
def test_validation_messages(kw, msg):
    p = _p(**kw)
    rc = L.lib().sla_b200_validate(C.byref(p))
    assert rc == L.ERR_INVALID
    assert L.lib().sla_b200_last_error().decode() == msg


def test_make_block_layout_raises_value_error():
    with pytest.raises(ValueError, match="does not divide N=32760"):
        S.make_block_layout(32760, 128, 64, 64)
    lay = S.make_block_layout(32768, 128, 64, 64)
    assert (lay.t_m, lay.t_n) == (512, 512)


@pytest.mark.parametrize("n,n1,nn", [(1024, 1, 2), (32768, 26, 51), (75648, 59, 118)])
def test_query_counts_match_reference_formula(n, n1, nn):
    p = _p(n=n, d=128)
    info = L.Info()
    assert L.lib().sla_b200_query(C.byref(p), C.byref(info)) == 0
    assert (info.n1, info.n_neg, info.t_m, info.t_n) == (n1, nn, n // 64, n // 64)


def test_sizes_scale_with_problem():
    small, big = _p(), _p(heads=12, n=32768, d=128)
    out = []
    for p in (small, big):
        sb, wb = C.c_size_t(), C.c_size_t()
        assert L.lib().sla_b200_sizes(C.byref(p), C.byref(sb), C.byref(wb)) == 0
        out.append((sb.value, wb.value))
    assert 0 < out[0][0] < out[1][0] and 0 < out[0][1] < out[1][1]


def test_generic_shape_limits_are_reported():
    p = _p(n=1024, d=1024, b_q=256, b_kv=256)
    p.flags = L.FLAG_GENERIC
    assert L.lib().sla_b200_validate(C.byref(p)) == L.ERR_INVALID
    assert "shared memory" in L.lib().sla_b200_last_error().decode()


def test_autograd_caller_validates_shapes_before_any_launch():
    import torch
    from paper_2509_24006_b200 import sparse_linear_attention
    q = torch.zeros(1, 2, 128, 64)
    with pytest.raises(ValueError):
        sparse_linear_attention(q, q[:, :1], q, torch.zeros(64, 64))
    with pytest.raises(ValueError):
        sparse_linear_attention(q, q, q, torch.zeros(3, 64, 64))
    with pytest.raises(ValueError):
        sparse_linear_attention(q, q, q, torch.zeros(64, 64), layout="nhd")


def test_fast_forward_rejects_null_branch_outputs():
    """The tcgen05 forward stores O^s and O^l by TMA: NULL is an InvalidArgument, returned before
    any device work (fake device pointers are never dereferenced)."""
    p = _p(d=128)
    fake = C.c_void_p(0x1000)
    rc = L.lib().sla_b200_forward(C.byref(p), fake, fake, fake, None, None, None, None, fake, fake, fake,
                                  fake, None)
    assert rc == L.ERR_INVALID
    assert "o_s and o_l are required" in L.lib().sla_b200_last_error().decode()


def test_split_backward_requires_linear_cotangent():
    p = _p(d=128)
    fake = C.c_void_p(0x1000)
    rc = L.lib().sla_b200_backward_split(C.byref(p), *([fake] * 7), None, *([fake] * 4), None, fake, fake, None)
    assert rc == L.ERR_INVALID
    assert "cotangent" in L.lib().sla_b200_last_error().decode()


def test_launch_count_survives_queries():
    """sla_b200_state_labels / validate / query / sizes launch nothing and leave the previous
    call's launch count readable (bench.py counts kernels through it)."""
    p = _p()
    before = L.lib().sla_b200_last_launch_count()
    assert L.lib().sla_b200_validate(C.byref(p)) == 0
    info = L.Info()
    assert L.lib().sla_b200_query(C.byref(p), C.byref(info)) == 0
    assert L.lib().sla_b200_last_launch_count() == before
