"""ctypes/numpy front end for the parity checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs import this module.  It never sits on the product path.

* ``Oracle``    -- the C restatement in oracle/sla_oracle.c (f64, reference loop order).
* ``Reference`` -- the unmodified reference library (oracle/_ref/libsla_ref.so) built
  from /root/reference/proj/core by oracle/Makefile.  Absent on machines that never
  had /root/reference; callers must handle ``Reference.available() is False``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libsla_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsla_ref.so")

PHI = {"elu1": 0, "relu": 1, "softmax": 2}
LSE_SENTINEL_F64 = -1e300
LSE_SENTINEL_F32 = np.float32(-1e30)

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_i8 = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def build(ref: bool = True) -> None:
    """Compile the checkers (gcc/g++ only).  ref=True also builds oracle/_ref when
    /root/reference exists."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/core"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class _Opt:
    """NULL-able double* argument."""

    @staticmethod
    def from_param(a):
        if a is None:
            return None
        if not (isinstance(a, np.ndarray) and a.flags.c_contiguous):
            raise TypeError("expected C-contiguous ndarray")
        return a.ctypes.data_as(C.c_void_p)


class Oracle:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                build(ref=False)
            lib = C.CDLL(ORACLE_SO)
            lib.orc_rng_next.argtypes = [C.POINTER(C.c_uint64)]
            lib.orc_rng_next.restype = C.c_uint64
            lib.orc_rng_uniform.argtypes = [C.POINTER(C.c_uint64)]
            lib.orc_rng_uniform.restype = C.c_double
            lib.orc_rng_gaussian.argtypes = [C.POINTER(C.c_uint64), _dp, _sz, C.c_double]
            lib.orc_rng_uniform_range.argtypes = [C.POINTER(C.c_uint64), _dp, _sz, C.c_double, C.c_double]
            lib.orc_random_mask.argtypes = [C.POINTER(C.c_uint64), _sz, _sz, C.c_double, C.c_double, C.c_int, _i8]
            lib.orc_validate.argtypes = [_sz, _sz, _sz, _sz, C.c_double, C.c_double, C.c_char_p, _sz]
            lib.orc_pool_mean.argtypes = [_dp, _sz, _sz, _sz, _dp]
            lib.orc_predict.argtypes = [_dp, _dp, _sz, _sz, _sz, _sz, _dp]
            lib.orc_predict_ragged.argtypes = [_dp, _dp, _sz, _sz, _sz, _dp]
            lib.orc_scores.argtypes = [_dp, _dp, _sz, _sz, _sz, _sz, _dp]
            lib.orc_counts.argtypes = [_sz, C.c_double, C.c_double, C.POINTER(_sz), C.POINTER(_sz)]
            lib.orc_classify.argtypes = [_dp, _sz, _sz, C.c_double, C.c_double, _i8]
            lib.orc_phi.argtypes = [_dp, _sz, _sz, C.c_int, _dp]
            lib.orc_phi_vjp.argtypes = [_dp, _sz, _sz, C.c_int, _dp, _dp]
            lib.orc_summaries.argtypes = [_dp, _dp, _sz, _sz, _sz, _dp, _dp]
            lib.orc_aggregate_direct.argtypes = [_dp, _dp, _sz, _u32, _sz, _dp, _dp]
            lib.orc_forward.argtypes = [_dp, _dp, _dp, _i8, _sz, _sz, _sz, _sz, C.c_int,
                                        C.c_void_p, _sz, _dp, _dp, _dp, _Opt, _Opt]
            lib.orc_combine.argtypes = [_dp, _dp, _dp, _sz, _sz, _dp]
            lib.orc_proj_backward.argtypes = [_dp, _dp, _dp, _sz, _sz, _dp, _dp, _dp]
            lib.orc_backward.argtypes = [_dp, _dp, _dp, _i8] + [_dp] * 7 + [_sz, _sz, _sz, _sz, C.c_int] + [_dp] * 8
            lib.orc_flops.argtypes = [_sz, _sz, _sz, _sz, _i8, np.ctypeslib.ndpointer(dtype=np.uint64)]
            cls._lib = lib
        return cls._lib


class Rng:
    """SplitMix64 stream (rng.hpp:22-64) -- bit-identical to the reference's fixtures."""

    def __init__(self, seed: int):
        self.state = C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def next(self) -> int:
        return int(Oracle.lib().orc_rng_next(C.byref(self.state)))

    def uniform(self) -> float:
        return float(Oracle.lib().orc_rng_uniform(C.byref(self.state)))

    def gaussian(self, rows: int, cols: int, stddev: float = 1.0) -> np.ndarray:
        out = np.empty((rows, cols), np.float64)
        Oracle.lib().orc_rng_gaussian(C.byref(self.state), out, out.size, stddev)
        return out

    def uniform_mat(self, rows: int, cols: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        out = np.empty((rows, cols), np.float64)
        Oracle.lib().orc_rng_uniform_range(C.byref(self.state), out, out.size, lo, hi)
        return out

    def random_mask(self, t_m, t_n, p_critical=0.3, p_marginal=0.4, allow_empty_critical=False):
        out = np.empty((t_m, t_n), np.int8)
        Oracle.lib().orc_random_mask(C.byref(self.state), t_m, t_n, p_critical, p_marginal,
                                     int(allow_empty_critical), out)
        return out


def to_bf16_exact(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float64 holding exactly those values."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------------------
# thin numpy wrappers over the C restatement
# ---------------------------------------------------------------------------------------
def counts(t_n: int, k_h: float, k_l: float):
    a, b = _sz(), _sz()
    Oracle.lib().orc_counts(t_n, k_h, k_l, C.byref(a), C.byref(b))
    return a.value, b.value


def validate(n, d, b_q, b_kv, k_h, k_l):
    buf = C.create_string_buffer(200)
    rc = Oracle.lib().orc_validate(n, d, b_q, b_kv, k_h, k_l, buf, 200)
    return rc, buf.value.decode()


def pool_mean(x, b):
    x = _f64(x)
    out = np.empty((x.shape[0] // b, x.shape[1]))
    if Oracle.lib().orc_pool_mean(x, x.shape[0], x.shape[1], b, out):
        raise ValueError("pool_mean: b must divide rows")
    return out


def scores(q, k, b_q, b_kv):
    q, k = _f64(q), _f64(k)
    n, d = q.shape
    out = np.empty((n // b_q, n // b_kv))
    Oracle.lib().orc_scores(q, k, n, d, b_q, b_kv, out)
    return out


def predict(q, k, b_q, b_kv):
    q, k = _f64(q), _f64(k)
    n, d = q.shape
    out = np.empty((n // b_q, n // b_kv))
    if Oracle.lib().orc_predict(q, k, n, d, b_q, b_kv, out):
        raise ValueError("predict: bad layout")
    return out


def predict_ragged(q, k, b):
    """Ragged-N extension of predict (sla_oracle.c orc_predict_ragged): T = ceil(N / b), the
    last block's pooled mean over its valid rows.  No reference counterpart (layout.cpp:12-17
    rejects ragged N)."""
    q, k = _f64(q), _f64(k)
    n, d = q.shape
    t = (n + b - 1) // b
    out = np.empty((t, t))
    if Oracle.lib().orc_predict_ragged(q, k, n, d, b, out):
        raise ValueError("predict_ragged: bad layout")
    return out


def dynamic_labels_ragged(q, k, b, k_h, k_l):
    return classify(predict_ragged(q, k, b), k_h, k_l)


def classify(p_c, k_h, k_l):
    p_c = _f64(p_c)
    out = np.empty(p_c.shape, np.int8)
    if Oracle.lib().orc_classify(p_c, p_c.shape[0], p_c.shape[1], k_h, k_l, out):
        raise ValueError("classify_mask: k_h + k_l > 100")
    return out


def phi(x, kind):
    x = _f64(x)
    out = np.empty_like(x)
    Oracle.lib().orc_phi(x, x.shape[0], x.shape[1], PHI[kind], out)
    return out


def phi_vjp(x, kind, g):
    x, g = _f64(x), _f64(g)
    out = np.empty_like(x)
    Oracle.lib().orc_phi_vjp(x, x.shape[0], x.shape[1], PHI[kind], g, out)
    return out


def summaries(k_feat, v, b_kv):
    k_feat, v = _f64(k_feat), _f64(v)
    n, d = v.shape
    h = np.empty((n // b_kv, d, d))
    z = np.empty((n // b_kv, d))
    Oracle.lib().orc_summaries(k_feat, v, n, d, b_kv, h, z)
    return h, z


def aggregate_direct(h, z, idx):
    h, z = _f64(h), _f64(z)
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    d = h.shape[-1]
    ho, zo = np.empty((d, d)), np.empty(d)
    Oracle.lib().orc_aggregate_direct(h, z, d, idx, idx.size, ho, zo)
    return ho, zo


def forward(q, k, v, labels, b_q, b_kv, phi_kind="elu1", block_rows=None, want_state=False):
    """sla_forward_with_mask (forward.cpp:81-172). Returns dict(o_s, o_l, lse[, row_h, row_z])."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    labels = np.ascontiguousarray(labels, dtype=np.int8)
    n, d = q.shape
    t_m = n // b_q
    o_s = np.zeros((n, d))
    o_l = np.zeros((n, d))
    lse = np.full(n, LSE_SENTINEL_F64)
    row_h = np.zeros((t_m, d, d)) if want_state else None
    row_z = np.zeros((t_m, d)) if want_state else None
    br = None
    nbr = 0
    if block_rows is not None:
        br = np.ascontiguousarray(block_rows, dtype=np.int32)
        nbr = br.size
    rc = Oracle.lib().orc_forward(q, k, v, labels, n, d, b_q, b_kv, PHI[phi_kind],
                                  None if br is None else br.ctypes.data_as(C.c_void_p), nbr,
                                  o_s, o_l, lse, row_h, row_z)
    if rc == 2:
        raise ValueError("sla_forward: invalid input")
    if rc == 1:
        raise RuntimeError("sla_forward: non-finite output")
    out = dict(o_s=o_s, o_l=o_l, lse=lse)
    if want_state:
        out.update(row_h=row_h, row_z=row_z)
    return out


def combine(o_s, o_l, w):
    o_s, o_l, w = _f64(o_s), _f64(o_l), _f64(w)
    out = np.empty_like(o_s)
    Oracle.lib().orc_combine(o_s, o_l, w, o_s.shape[0], o_s.shape[1], out)
    return out


def proj_backward(d_out, o_l, w):
    d_out, o_l, w = _f64(d_out), _f64(o_l), _f64(w)
    n, d = d_out.shape
    ds, dl, dw = np.empty((n, d)), np.empty((n, d)), np.empty((d, d))
    Oracle.lib().orc_proj_backward(d_out, o_l, w, n, d, ds, dl, dw)
    return ds, dl, dw


def backward(q, k, v, labels, state, d_out_s, d_out_l, b_q, b_kv, phi_kind="elu1"):
    """sla_backward (backward.cpp:24-216).  state = forward(..., want_state=True)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    labels = np.ascontiguousarray(labels, dtype=np.int8)
    n, d = q.shape
    outs = [np.empty((n, d)) for _ in range(5)] + [np.empty((d, d))] + [np.empty((n, d)) for _ in range(2)]
    Oracle.lib().orc_backward(q, k, v, labels, _f64(state["o_s"]), _f64(state["o_l"]),
                              _f64(state["lse"]), _f64(state["row_h"]), _f64(state["row_z"]),
                              _f64(d_out_s), _f64(d_out_l), n, d, b_q, b_kv, PHI[phi_kind], *outs)
    names = ["dq", "dk", "dv", "dq_feat", "dk_feat", "dproj", "dq_total", "dk_total"]
    return dict(zip(names, outs))


def step(q, k, v, w, d_out, labels, b_q, b_kv, phi_kind="elu1"):
    """Full training step as the reference's callers run it (finetune.cpp:24-68)."""
    st = forward(q, k, v, labels, b_q, b_kv, phi_kind, want_state=True)
    o = combine(st["o_s"], st["o_l"], w)
    dos, dol, dw = proj_backward(d_out, st["o_l"], w)
    g = backward(q, k, v, labels, st, dos, dol, b_q, b_kv, phi_kind)
    g["dw"] = dw
    g.update(st)
    g["o"] = o
    return g


def dynamic_labels(q, k, b_q, b_kv, k_h, k_l):
    """sla_forward's mask (forward.cpp:174-185): predict in f64, then classify."""
    return classify(predict(q, k, b_q, b_kv), k_h, k_l)


def flops(n, d, b_q, b_kv, labels):
    out = np.zeros(6, np.uint64)
    Oracle.lib().orc_flops(n, d, b_q, b_kv, np.ascontiguousarray(labels, np.int8), out)
    return dict(zip(["full", "sparse", "linear", "proj", "mask", "total"], [int(x) for x in out]))


AGG = {"direct": 0, "complement": 1, "four_russians": 2, "auto": 3}


def resolve_strategy(kind, marginal_fraction, direct_max=0.25, complement_min=0.75):
    """aggregation.cpp:147-156 with the config.hpp:30-31 default thresholds."""
    if kind != AGG["auto"]:
        return kind
    if marginal_fraction <= direct_max:
        return AGG["direct"]
    if marginal_fraction >= complement_min:
        return AGG["complement"]
    return AGG["four_russians"]


def exec_counters(q, k, labels, b_q, b_kv, phi_kind="elu1", aggregation="direct", group_size=4):
    """ExecCounters of sla_forward_with_mask (forward.hpp:46-50) restated from the label grid:
    2 block matmuls per critical block (forward.cpp:46, 123-124); one linear row product per
    row of a block row with a marginal block whose den = phi(q) . Z_i is non-zero
    (forward.cpp:130-146; phi >= 0 and z >= 0, so den == 0 iff every product is 0); the
    aggregation counts of the resolved strategy: direct = marginal - 1 additions per non-empty
    row (aggregation.cpp:40-56), complement = one subtraction per excluded block
    (aggregation.cpp:58-70), Four-Russians = one lookup per group holding a marginal block and
    lookups - 1 additions per row, plus 2^size - 1 table additions per group
    (aggregation.cpp:72-145).  Returns [sparse, linear_rows, additions, subtractions, lookups,
    table_build_additions]."""
    lab = np.asarray(labels)
    t_m, t_n = lab.shape
    qf, kf = phi(np.asarray(q, np.float64), phi_kind), phi(np.asarray(k, np.float64), phi_kind)
    z = kf.reshape(t_n, b_kv, -1).sum(axis=1)
    marg = lab == 0
    strat = resolve_strategy(AGG[aggregation] if isinstance(aggregation, str) else aggregation,
                             marg.sum() / (t_m * t_n))
    out = [2 * int((lab == 1).sum()), 0, 0, 0, 0, 0]
    g = group_size
    groups = [(b, min(b + g, t_n)) for b in range(0, t_n, g)]
    if strat == AGG["four_russians"]:
        out[5] = sum((1 << (e - b)) - 1 for b, e in groups)
    for i in range(t_m):
        m = marg[i]
        cnt = int(m.sum())
        if strat == AGG["direct"]:
            out[2] += max(cnt - 1, 0)
        elif strat == AGG["complement"]:
            out[3] += t_n - cnt
        else:
            hit = sum(1 for b, e in groups if m[b:e].any())
            out[4] += hit
            out[2] += max(hit - 1, 0)
        if cnt:
            zi = z[m].sum(axis=0)
            rows = qf[i * b_q:(i + 1) * b_q]
            out[1] += int(((rows * zi) != 0).any(axis=1).sum())
    return out


def rel_diff(a, b, floor=1e-300):
    """mat.hpp:169-178 max-norm relative difference."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    num = float(np.max(np.abs(a - b))) if a.size else 0.0
    den = max(floor, float(np.max(np.abs(b))) if b.size else 0.0)
    return num / den


# ---------------------------------------------------------------------------------------
# the real reference (oracle/_ref)
# ---------------------------------------------------------------------------------------
class Reference:
    _lib = None

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            lib = C.CDLL(REF_SO)
            for name, ptr in (("ref_run_f32", C.c_void_p), ("ref_run_f64", C.c_void_p)):
                f = getattr(lib, name)
                f.argtypes = [_sz, _sz, _sz, _sz, C.c_double, C.c_double, C.c_int, C.c_uint] + \
                             [C.c_void_p] * 19 + [C.c_char_p, _sz]
                f.restype = C.c_int
            lib.ref_predict.argtypes = [_sz, _sz, _sz, _sz, _dp, _dp, _dp, C.c_char_p, _sz]
            lib.ref_classify.argtypes = [_sz, _sz, _dp, C.c_double, C.c_double, _i8, C.c_char_p, _sz]
            lib.ref_exec_counters.argtypes = [_sz, _sz, _sz, _sz, C.c_int, C.c_int, _sz] + \
                                             [C.c_void_p] * 5 + [C.c_char_p, _sz]
            lib.ref_flops_report.argtypes = [_sz, _sz, _sz, _sz] + [C.c_void_p] * 3 + [C.c_char_p, _sz]
            cls._lib = lib
        return cls._lib

    @classmethod
    def run(cls, q, k, v, b_q, b_kv, k_h=5.0, k_l=10.0, phi_kind="elu1", threads=1, w=None,
            labels=None, d_out=None, dtype=np.float32):
        """sla_forward[_with_mask] -> combine -> proj_backward -> sla_backward."""
        dt = np.dtype(dtype)
        q, k, v = (np.ascontiguousarray(x, dt) for x in (q, k, v))
        n, d = q.shape
        t_m, t_n = n // b_q, n // b_kv
        out = {}
        ptr = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
        labels_out = np.empty((t_m, t_n), np.int8)
        o_s, o_l, lse = np.empty((n, d), dt), np.empty((n, d), dt), np.empty(n, dt)
        w_ = None if w is None else np.ascontiguousarray(w, dt)
        do_ = None if d_out is None else np.ascontiguousarray(d_out, dt)
        lab_in = None if labels is None else np.ascontiguousarray(labels, np.int8)
        o = np.empty((n, d), dt) if w_ is not None else None
        grads = {}
        if do_ is not None:
            for nm in ("dq_total", "dk_total", "dv", "dq", "dk", "dq_feat", "dk_feat"):
                grads[nm] = np.empty((n, d), dt)
            grads["dw"] = np.empty((d, d), dt)
        g = lambda nm: ptr(grads.get(nm))  # noqa: E731
        err = C.create_string_buffer(300)
        f = cls.lib().ref_run_f32 if dt == np.float32 else cls.lib().ref_run_f64
        rc = f(n, d, b_q, b_kv, k_h, k_l, PHI[phi_kind], threads, ptr(q), ptr(k), ptr(v), ptr(w_),
               ptr(lab_in), ptr(do_), ptr(labels_out), ptr(o_s), ptr(o_l), ptr(o), ptr(lse),
               g("dq_total"), g("dk_total"), g("dv"), g("dw"), g("dq"), g("dk"), g("dq_feat"),
               g("dk_feat"), err, 300)
        if rc == 2:
            raise ValueError(err.value.decode())
        if rc:
            raise RuntimeError(err.value.decode())
        out.update(labels=labels_out, o_s=o_s, o_l=o_l, lse=lse)
        if o is not None:
            out["o"] = o
        out.update(grads)
        return out

    @classmethod
    def predict(cls, q, k, b_q, b_kv):
        q, k = _f64(q), _f64(k)
        n, d = q.shape
        out = np.empty((n // b_q, n // b_kv))
        err = C.create_string_buffer(300)
        if cls.lib().ref_predict(n, d, b_q, b_kv, q, k, out, err, 300):
            raise ValueError(err.value.decode())
        return out

    @classmethod
    def exec_counters(cls, q, k, v, labels, b_q, b_kv, phi_kind="elu1", aggregation="direct", group_size=4):
        """ExecCounters of the reference's sla_forward_with_mask<float> on this label grid."""
        q, k, v = (np.ascontiguousarray(x, np.float32) for x in (q, k, v))
        lab = np.ascontiguousarray(labels, np.int8)
        out = np.zeros(6, np.uint64)
        err = C.create_string_buffer(300)
        agg = AGG[aggregation] if isinstance(aggregation, str) else aggregation
        rc = cls.lib().ref_exec_counters(q.shape[0], q.shape[1], b_q, b_kv, PHI[phi_kind], agg, group_size,
                                         q.ctypes.data, k.ctypes.data, v.ctypes.data, lab.ctypes.data,
                                         out.ctypes.data, err, 300)
        if rc:
            raise ValueError(err.value.decode())
        return [int(x) for x in out]

    @classmethod
    def flops_report(cls, n, d, b_q, b_kv, labels):
        """flops.cpp:7-33: ([full, sparse, linear, proj, mask, total], ratio, sparsity)."""
        lab = np.ascontiguousarray(labels, np.int8)
        u, f = np.zeros(6, np.uint64), np.zeros(2)
        err = C.create_string_buffer(300)
        if cls.lib().ref_flops_report(n, d, b_q, b_kv, lab.ctypes.data, u.ctypes.data, f.ctypes.data, err, 300):
            raise ValueError(err.value.decode())
        return [int(x) for x in u], float(f[0]), float(f[1])

    @classmethod
    def classify(cls, p_c, k_h, k_l):
        p_c = _f64(p_c)
        out = np.empty(p_c.shape, np.int8)
        err = C.create_string_buffer(300)
        if cls.lib().ref_classify(p_c.shape[0], p_c.shape[1], p_c, k_h, k_l, out, err, 300):
            raise ValueError(err.value.decode())
        return out
