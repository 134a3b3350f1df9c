"""ctypes binding of libsla_b200.so (include/sla_b200.h).

This is the reference-side binding a maintainer would add for Python callers; C++ callers
use include/sla_b200.hpp.  The library is loaded from the package directory; a missing
library is an error (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsla_b200.so")
DIAG_PATH = os.path.join(HERE, "libsla_b200_diag.so")  # microbenchmarks / layout probes, not the product

OK, ERR_RUNTIME, ERR_INVALID = 0, 1, 2
PHI = {"elu1": 0, "relu": 1, "softmax": 2}
DTYPE_BF16, DTYPE_F32 = 0, 1
MASK_F64, MASK_F32 = 0, 1
FLAG_CHECK_FINITE, FLAG_GENERIC, FLAG_RAGGED, FLAG_BNHD = 1, 2, 4, 8


class Problem(C.Structure):
    _fields_ = [
        ("batch", C.c_int64), ("heads", C.c_int64), ("n", C.c_int64), ("d", C.c_int64),
        ("b_q", C.c_int64), ("b_kv", C.c_int64), ("k_h", C.c_double), ("k_l", C.c_double),
        ("phi", C.c_int32), ("dtype", C.c_int32), ("mask_precision", C.c_int32),
        ("flags", C.c_uint32), ("n_kv", C.c_int64),
    ]


class Info(C.Structure):
    _fields_ = [("path", C.c_int32), ("n1", C.c_int32), ("n_neg", C.c_int32),
                ("t_m", C.c_int32), ("t_n", C.c_int32), ("gpu_launches", C.c_int64)]


class Flops(C.Structure):
    """sla_b200_flops: flops_report (flops.cpp:7-33) of one unit."""
    _fields_ = [("full_flops", C.c_uint64), ("sparse_flops", C.c_uint64), ("linear_flops", C.c_uint64),
                ("proj_flops", C.c_uint64), ("mask_flops", C.c_uint64), ("sla_total", C.c_uint64),
                ("ratio", C.c_double), ("sparsity", C.c_double)]


class Counters(C.Structure):
    """sla_b200_counters: ExecCounters (forward.hpp:46-50) with its AggCounters."""
    _fields_ = [("sparse_block_matmuls", C.c_uint64), ("linear_row_products", C.c_uint64),
                ("additions", C.c_uint64), ("subtractions", C.c_uint64), ("lookups", C.c_uint64),
                ("table_build_additions", C.c_uint64)]


AGG = {"direct": 0, "complement": 1, "four_russians": 2, "auto": 3}


class GradParts(C.Structure):
    _fields_ = [("dq_sparse", C.c_void_p), ("dk_sparse", C.c_void_p),
                ("dq_feat", C.c_void_p), ("dk_feat", C.c_void_p)]


_lib = None

EXPORTS = [
    "sla_b200_last_error", "sla_b200_abi_version", "sla_b200_validate", "sla_b200_sizes",
    "sla_b200_query", "sla_b200_last_launch_count", "sla_b200_classify", "sla_b200_forward",
    "sla_b200_backward", "sla_b200_backward_ex", "sla_b200_state_labels",
    "sla_b200_flops_report", "sla_b200_exec_counters", "sla_b200_backward_split",
    "sla_b200_combine_outputs", "sla_b200_proj_backward", "sla_b200_build_state",
    "sla_b200_backward_rows", "sla_b200_backward_cols",
]


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"sla_b200: CUDA library not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER(Problem)
    vp = C.c_void_p
    L.sla_b200_last_error.restype = C.c_char_p
    L.sla_b200_abi_version.restype = C.c_int
    L.sla_b200_last_launch_count.restype = C.c_int64
    L.sla_b200_validate.argtypes = [P]
    L.sla_b200_sizes.argtypes = [P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
    L.sla_b200_query.argtypes = [P, C.POINTER(Info)]
    L.sla_b200_classify.argtypes = [P, vp, vp, vp, vp, vp, vp, vp]
    L.sla_b200_forward.argtypes = [P] + [vp] * 12
    L.sla_b200_backward.argtypes = [P] + [vp] * 15
    L.sla_b200_backward_ex.argtypes = [P] + [vp] * 12 + [C.POINTER(GradParts)] + [vp] * 3
    L.sla_b200_state_labels.argtypes = [P, vp, C.POINTER(C.c_void_p)]
    L.sla_b200_backward_split.argtypes = [P] + [vp] * 12 + [C.POINTER(GradParts)] + [vp] * 3
    L.sla_b200_combine_outputs.argtypes = [P] + [vp] * 5
    L.sla_b200_proj_backward.argtypes = [P] + [vp] * 7
    L.sla_b200_build_state.argtypes = [P] + [vp] * 7
    L.sla_b200_backward_rows.argtypes = [P] + [vp] * 17
    L.sla_b200_backward_cols.argtypes = [P] + [vp] * 14
    L.sla_b200_flops_report.argtypes = [P, vp, C.POINTER(Flops), vp, vp]
    L.sla_b200_exec_counters.argtypes = [P, vp, vp, C.c_int, C.c_int, C.POINTER(Counters), vp, vp]
    for name in EXPORTS:
        getattr(L, name)
    _lib = L
    return L


_diag = None


def diag_lib():
    """libsla_b200_diag.so: csrc/diag.cu (TMEM layout probes, tcgen05 / TMA microbenchmarks, the
    bare GEMM) for tests/test_gpu_gemm.py, tests/test_gpu_tmem.py and profiles/."""
    global _diag
    if _diag is None:
        lib()  # the product library first (the diag library links against it)
        _diag = C.CDLL(DIAG_PATH)
    return _diag


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().sla_b200_last_error().decode()
    if rc == ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(msg)
