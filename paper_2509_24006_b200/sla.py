"""Host-side mirror of the reference's SLA operator API over the B200 C-ABI.

The names, argument meaning and error behaviour follow the reference
(/root/reference/proj/core):

  SlaConfig              config.hpp:21-32       (k_h, k_l, phi; f64 mask by default)
  make_block_layout      layout.cpp:8-26        raises ValueError (std::invalid_argument)
  sla_forward            forward.cpp:174-185    dynamic mask from q, k
  sla_forward_with_mask  forward.cpp:81-172     injected label grid
  combine_outputs        forward.cpp:187-195    fused into the forward kernel epilogue (and a
                                                device kernel for a standalone call)
  proj_backward          backward.cpp:12-22     device dO W^T and dW = O^l^T dO
  sla_backward           backward.cpp:24-216    independent cotangents (dO^s, dO^l), as the
                                                reference takes them
  SLA.backward           proj_backward + sla_backward fused, from the combined cotangent

Tensors are CUDA tensors (torch is only the device-memory / stream plumbing); every op
runs through libsla_b200.so.  Shapes: [N, d] for one (batch, head) unit as in the
reference, or [B, H, N, d] for batched use; W is [d, d] or [H, d, d].
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _lib as L

LSE_SENTINEL = -1e30  # forward.hpp:18-24 (f32)


@dataclass
class SlaConfig:
    """config.hpp:21-32 (aggregation strategy is fixed: the device aggregates with GEMMs)."""

    k_h: float = 25.0
    k_l: float = 25.0
    phi: str = "elu1"
    mask_precision: str = "f64"   # "f64" (reference-exact) | "f32" (north-star fp32 variant)
    check_finite: bool = False    # reproduce the reference's non-finite input/output errors
    force_generic: bool = False   # run the shape-generic SIMT kernels
    ragged: bool = False          # allow N % 64 != 0 (SLA_B200_FLAG_RAGGED; not in the reference)
    bnhd: bool = False            # tensors are [B, N, H, d], lse [B, N, H] (SLA_B200_FLAG_BNHD)


@dataclass
class BlockLayout:
    n: int
    d: int
    b_q: int
    b_kv: int
    t_m: int = 0
    t_n: int = 0


def _problem(batch, heads, n, d, b_q, b_kv, cfg: SlaConfig, dtype, n_kv: int = 0) -> L.Problem:
    if cfg.phi not in L.PHI:
        raise ValueError(f"unknown feature map: {cfg.phi}")
    p = L.Problem()
    p.batch, p.heads, p.n, p.d, p.b_q, p.b_kv = batch, heads, n, d, b_q, b_kv
    p.n_kv = n_kv
    p.k_h, p.k_l = float(cfg.k_h), float(cfg.k_l)
    p.phi = L.PHI[cfg.phi]
    if dtype == torch.bfloat16:
        p.dtype = L.DTYPE_BF16
    elif dtype == torch.float32:
        p.dtype = L.DTYPE_F32
    else:
        raise ValueError(f"unsupported dtype {dtype}")
    p.mask_precision = {"f64": L.MASK_F64, "f32": L.MASK_F32}[cfg.mask_precision]
    p.flags = ((L.FLAG_CHECK_FINITE if cfg.check_finite else 0) | (L.FLAG_GENERIC if cfg.force_generic else 0)
               | (L.FLAG_RAGGED if cfg.ragged else 0) | (L.FLAG_BNHD if cfg.bnhd else 0))
    return p


def make_block_layout(n: int, d: int, b_q: int, b_kv: int) -> BlockLayout:
    """layout.cpp:8-26 -- raises ValueError when a block size does not divide N."""
    p = _problem(1, 1, n, d, b_q, b_kv, SlaConfig(), torch.float32)
    L.check(L.lib().sla_b200_validate(C.byref(p)))
    return BlockLayout(n, d, b_q, b_kv, n // b_q, n // b_kv)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


@dataclass
class SlaForwardState:
    """forward.hpp:33-43.  Device tensors; `state` holds the label grid, lookups, H and Z."""

    o: Optional[torch.Tensor]
    o_s: torch.Tensor
    o_l: torch.Tensor
    lse: torch.Tensor
    labels: torch.Tensor
    op: "SLA" = field(repr=False)
    state: torch.Tensor = field(repr=False)


@dataclass
class SlaGradients:
    """backward.hpp:10-16 (dq_total / dk_total are the composed totals)."""

    dq_total: torch.Tensor
    dk_total: torch.Tensor
    dv: torch.Tensor
    dproj: torch.Tensor
    dq: Optional[torch.Tensor] = None
    dk: Optional[torch.Tensor] = None
    dq_feat: Optional[torch.Tensor] = None
    dk_feat: Optional[torch.Tensor] = None


class SLA:
    """One SLA operator instance for a fixed problem shape: owns its state/workspace."""

    def __init__(self, batch: int, heads: int, n: int, d: int, b_q: int = 64, b_kv: int = 64,
                 cfg: Optional[SlaConfig] = None, dtype=torch.bfloat16, device="cuda", n_kv: int = 0):
        """n_kv (one unit only): a rectangular view -- n query rows against n_kv key rows, the
        building block of partitioned execution (runner.py)."""
        self.cfg = cfg or SlaConfig()
        self.batch, self.heads, self.n, self.d = batch, heads, n, d
        self.b_q, self.b_kv = b_q, b_kv
        self.dtype = dtype
        self.device = torch.device(device)
        self.n_kv = n_kv or n
        self.p = _problem(batch, heads, n, d, b_q, b_kv, self.cfg, dtype, n_kv if n_kv != n else 0)
        sb, wb = C.c_size_t(), C.c_size_t()
        L.check(L.lib().sla_b200_sizes(C.byref(self.p), C.byref(sb), C.byref(wb)))
        self.state_bytes, self.workspace_bytes = sb.value, wb.value
        info = L.Info()
        L.check(L.lib().sla_b200_query(C.byref(self.p), C.byref(info)))
        self.info = info
        self.t_m, self.t_n = info.t_m, info.t_n
        self._workspaces = {}

    @property
    def _workspace(self) -> torch.Tensor:
        """Scratch of the current stream: calls issued on different streams must not share it
        (the C-ABI is re-entrant per stream, sla_b200.h)."""
        key = torch.cuda.current_stream(self.device).cuda_stream
        ws = self._workspaces.get(key)
        if ws is None:
            ws = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=self.device)
            self._workspaces[key] = ws
        return ws

    @property
    def path(self) -> str:
        return "tcgen05" if self.info.path == 1 else "generic"

    # -- helpers ----------------------------------------------------------------------
    def _unit_shape(self):
        if self.cfg.bnhd:
            return (self.batch, self.n, self.heads, self.d)
        return (self.batch, self.heads, self.n, self.d)

    def _kv_shape(self):
        if self.cfg.bnhd:
            return (self.batch, self.n_kv, self.heads, self.d)
        return (self.batch, self.heads, self.n_kv, self.d)

    def _check(self, name, t, shape=None, dtype=None):
        shape = shape or self._unit_shape()
        dtype = dtype or self.dtype
        if t.numel() != int(torch.tensor(shape).prod()):
            raise ValueError(f"sla_forward: {name} must be N x d")
        if t.dtype != dtype or not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"sla_b200: {name} must be a contiguous {dtype} CUDA tensor")

    def _w(self, w):
        if w is None:
            return None
        if w.numel() == self.d * self.d and self.heads > 1:
            w = w.reshape(1, self.d, self.d).expand(self.heads, self.d, self.d).contiguous()
        self._check("W", w, (self.heads, self.d, self.d))
        return w

    def new_state(self) -> torch.Tensor:
        return torch.empty(self.state_bytes, dtype=torch.uint8, device=self.device)

    def labels_of(self, state: torch.Tensor) -> torch.Tensor:
        ptr = C.c_void_p()
        L.check(L.lib().sla_b200_state_labels(C.byref(self.p), _ptr(state), C.byref(ptr)))
        off = ptr.value - state.data_ptr()
        n = self.batch * self.heads * self.t_m * self.t_n
        return state[off:off + n].view(torch.int8).view(self.batch, self.heads, self.t_m, self.t_n)

    # -- API ------------------------------------------------------------------------
    def classify(self, q, k, weights: bool = False):
        """predict_compressed_weights + classify_mask (mask.cpp:57-119)."""
        self._check("Q", q)
        self._check("K", k, self._kv_shape())
        state = self.new_state()
        labels = torch.empty((self.batch, self.heads, self.t_m, self.t_n), dtype=torch.int8,
                             device=self.device)
        p_c = torch.empty((self.batch, self.heads, self.t_m, self.t_n), dtype=torch.float64,
                          device=self.device) if weights else None
        with torch.cuda.device(self.device):
            L.check(L.lib().sla_b200_classify(C.byref(self.p), _ptr(q), _ptr(k), _ptr(labels),
                                              _ptr(p_c), _ptr(state), _ptr(self._workspace), _stream(self.device)))
        return (labels, p_c) if weights else labels

    def forward(self, q, k, v, w=None, mask=None, state=None, out=None) -> SlaForwardState:
        """sla_forward (mask None) / sla_forward_with_mask, fused with combine_outputs."""
        self._check("Q", q)
        self._check("K", k, self._kv_shape())
        self._check("V", v, self._kv_shape())
        w = self._w(w)
        if mask is not None:
            mask = mask.to(device=self.device, dtype=torch.int8).contiguous()
            if mask.numel() != self.batch * self.heads * self.t_m * self.t_n:
                raise ValueError("sla_forward: mask does not match layout")
        shape = self._unit_shape()
        state = self.new_state() if state is None else state
        if out is None:
            o = torch.empty(shape, dtype=self.dtype, device=self.device) if w is not None else None
            o_s = torch.empty(shape, dtype=self.dtype, device=self.device)
            o_l = torch.empty(shape, dtype=self.dtype, device=self.device)
            lse = torch.empty(shape[:-1], dtype=torch.float32, device=self.device)
        else:
            o, o_s, o_l, lse = out
        with torch.cuda.device(self.device):
            L.check(L.lib().sla_b200_forward(C.byref(self.p), _ptr(q), _ptr(k), _ptr(v), _ptr(w),
                                             _ptr(mask), _ptr(o), _ptr(o_s), _ptr(o_l), _ptr(lse),
                                             _ptr(state), _ptr(self._workspace), _stream(self.device)))
        return SlaForwardState(o, o_s, o_l, lse, self.labels_of(state), self, state)

    def backward(self, st: SlaForwardState, q, k, v, w, d_out, parts: bool = False,
                 out=None, d_out_linear=None) -> SlaGradients:
        """proj_backward + sla_backward (backward.cpp:12-216) from the combined cotangent d_out;
        with `d_out_linear`, sla_backward alone on independent cotangents (d_out = dO^s,
        backward.hpp:25-38; w is not used and dproj = O^l^T dO^s)."""
        if d_out_linear is None:
            w = self._w(w)
        else:
            self._check("dO^l", d_out_linear)
        self._check("dO", d_out)
        shape = self._unit_shape()
        if out is None:
            dq = torch.empty(shape, dtype=self.dtype, device=self.device)
            dk = torch.empty_like(dq)
            dv = torch.empty_like(dq)
            dw = torch.empty((self.heads, self.d, self.d), dtype=torch.float32, device=self.device)
        else:
            dq, dk, dv, dw = out
        gp = None
        extra = {}
        if parts:
            for nm in ("dq", "dk", "dq_feat", "dk_feat"):
                extra[nm] = torch.empty(shape, dtype=torch.float32, device=self.device)
            gp = L.GradParts(extra["dq"].data_ptr(), extra["dk"].data_ptr(),
                             extra["dq_feat"].data_ptr(), extra["dk_feat"].data_ptr())
        with torch.cuda.device(self.device):
            if d_out_linear is None:
                rc = L.lib().sla_b200_backward_ex(
                    C.byref(self.p), _ptr(q), _ptr(k), _ptr(v), _ptr(w), _ptr(st.o_s), _ptr(st.o_l),
                    _ptr(st.lse), _ptr(d_out), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dw),
                    None if gp is None else C.byref(gp), _ptr(st.state), _ptr(self._workspace),
                    _stream(self.device))
            else:
                rc = L.lib().sla_b200_backward_split(
                    C.byref(self.p), _ptr(q), _ptr(k), _ptr(v), _ptr(st.o_s), _ptr(st.o_l), _ptr(st.lse),
                    _ptr(d_out), _ptr(d_out_linear), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dw),
                    None if gp is None else C.byref(gp), _ptr(st.state), _ptr(self._workspace),
                    _stream(self.device))
        L.check(rc)
        return SlaGradients(dq, dk, dv, dw, **extra)

    # -- the backward in two phases, for partitioned execution (runner.py) ---------------
    def backward_rows(self, st: SlaForwardState, q, k, v, w, d_out, d_out_linear=None, want_dw: bool = True):
        """Row phase of this view's query rows (sla_b200_backward_rows): returns dq_total, the dW
        partial over these rows (or None), and the row summaries the column phase of every key
        range needs: D^s [N], dH_i [T_m, d, d] (bf16), dZ_i as three bf16 parts [T_m, 3 d]."""
        if d_out_linear is None:
            w = self._w(w)
        dev, d = self.device, self.d
        dq = torch.empty(self._unit_shape(), dtype=self.dtype, device=dev)
        dw = torch.empty((self.heads, d, d), dtype=torch.float32, device=dev) if want_dw else None
        U = self.batch * self.heads
        ds = torch.empty((U, self.n), dtype=torch.float32, device=dev)
        dh = torch.empty((U, self.t_m, d, d), dtype=torch.bfloat16, device=dev)
        dz = torch.empty((U, self.t_m, 3 * d), dtype=torch.bfloat16, device=dev)
        with torch.cuda.device(dev):
            L.check(L.lib().sla_b200_backward_rows(
                C.byref(self.p), _ptr(q), _ptr(k), _ptr(v), _ptr(w), _ptr(st.o_s), _ptr(st.o_l), _ptr(st.lse),
                _ptr(d_out), _ptr(d_out_linear), _ptr(dq), _ptr(dw), _ptr(ds), _ptr(dh), _ptr(dz), _ptr(st.state),
                _ptr(self._workspace), _stream(dev)))
        return dq, dw, ds, dh, dz

    def backward_cols(self, q, k, v, lse, d_out, ds, dh, dz, labels):
        """Column phase of this view's key blocks against every query row (sla_b200_backward_cols):
        q, d_out, lse, ds, dh, dz cover all query rows; labels [T_m, T_n] are all rows' labels
        restricted to these key blocks.  Returns dk_total, dv of these keys."""
        self._check("K", k, self._kv_shape())
        dk = torch.empty(self._kv_shape(), dtype=self.dtype, device=self.device)
        dv = torch.empty_like(dk)
        labels = labels.to(device=self.device, dtype=torch.int8).contiguous()
        state = self.new_state()
        with torch.cuda.device(self.device):
            L.check(L.lib().sla_b200_backward_cols(
                C.byref(self.p), _ptr(q), _ptr(k), _ptr(v), _ptr(lse), _ptr(d_out), _ptr(ds), _ptr(dh), _ptr(dz),
                _ptr(labels), _ptr(dk), _ptr(dv), _ptr(state), _ptr(self._workspace), _stream(self.device)))
        return dk, dv

    def combine(self, st: SlaForwardState, w) -> torch.Tensor:
        """combine_outputs (forward.cpp:187-195) on the device: O = O^s + O^l W."""
        w = self._w(w)
        o = torch.empty_like(st.o_s)
        with torch.cuda.device(self.device):
            L.check(L.lib().sla_b200_combine_outputs(C.byref(self.p), _ptr(st.o_s), _ptr(st.o_l), _ptr(w), _ptr(o),
                                                     _stream(self.device)))
        return o

    def proj_backward(self, d_out, o_l, w):
        """proj_backward (backward.cpp:12-22) on the device: (dO^s = dO, dO^l = dO W^T,
        dW = O^l^T dO summed over the batch per head)."""
        w = self._w(w)
        self._check("dO", d_out)
        self._check("O^l", o_l)
        d_out_l = torch.empty_like(d_out)
        dw = torch.empty((self.heads, self.d, self.d), dtype=torch.float32, device=self.device)
        with torch.cuda.device(self.device):
            L.check(L.lib().sla_b200_proj_backward(C.byref(self.p), _ptr(d_out), _ptr(o_l), _ptr(w), _ptr(d_out_l),
                                                   _ptr(dw), _ptr(self._workspace), _stream(self.device)))
        return d_out, d_out_l, dw

    def state_from(self, q, k, v, labels, o_s, o_l, lse) -> SlaForwardState:
        """A SlaForwardState around outputs the caller holds (e.g. a reference forward's O^s,
        O^l, lse and label grid): the device state (lookups, H, Z) is rebuilt from the labels by
        sla_b200_build_state, without rerunning the attention kernel."""
        for nm, t in (("Q", q), ("K", k), ("V", v), ("O^s", o_s), ("O^l", o_l)):
            self._check(nm, t)
        labels = labels.to(device=self.device, dtype=torch.int8).contiguous()
        state = self.new_state()
        with torch.cuda.device(self.device):
            L.check(L.lib().sla_b200_build_state(C.byref(self.p), _ptr(q), _ptr(k), _ptr(v), _ptr(labels),
                                                 _ptr(state), _ptr(self._workspace), _stream(self.device)))
        return SlaForwardState(None, o_s, o_l, lse, self.labels_of(state), self, state)

    def flops_report(self, st) -> list:
        """flops_report (flops.cpp:7-33) of every (batch, head) unit, from the device LUT of a
        forward state (SlaForwardState or its state tensor).  Synchronises the stream."""
        state = st.state if isinstance(st, SlaForwardState) else st
        arr = (L.Flops * (self.batch * self.heads))()
        L.check(L.lib().sla_b200_flops_report(C.byref(self.p), _ptr(state), arr, _ptr(self._workspace),
                                              _stream(self.device)))
        return [{f: getattr(x, f) for f, _ in L.Flops._fields_} for x in arr]

    def exec_counters(self, st: SlaForwardState, q, aggregation: str = "direct", group_size: int = 4) -> dict:
        """ExecCounters of the forward that produced `st` (forward.hpp:46-50), as the reference
        counts them for `aggregation` (config.hpp:19-31), summed over units."""
        self._check("Q", q)
        if aggregation not in L.AGG:
            raise ValueError(f"unknown aggregation strategy '{aggregation}'")
        c = L.Counters()
        L.check(L.lib().sla_b200_exec_counters(C.byref(self.p), _ptr(q), _ptr(st.state), L.AGG[aggregation],
                                               group_size, C.byref(c), _ptr(self._workspace), _stream(self.device)))
        return {f: int(getattr(c, f)) for f, _ in L.Counters._fields_}

    def launches(self) -> int:
        """Kernels launched by the last C-ABI call on this thread."""
        return int(L.lib().sla_b200_last_launch_count())


# ---- reference-named single-unit functional API ([N, d] tensors) -------------------------
def _op_for(q, cfg: SlaConfig, layout: BlockLayout) -> SLA:
    if q.dim() != 2 or q.shape[0] != layout.n or q.shape[1] != layout.d:
        raise ValueError("sla_forward: Q must be N x d")
    return SLA(1, 1, layout.n, layout.d, layout.b_q, layout.b_kv, cfg, q.dtype, q.device)


def sla_forward(q, k, v, cfg: SlaConfig, layout: BlockLayout, w=None) -> SlaForwardState:
    """forward.cpp:174-185 -- the mask is re-predicted from the live q, k."""
    return _op_for(q, cfg, layout).forward(q, k, v, w)


def sla_forward_with_mask(q, k, v, mask, cfg: SlaConfig, layout: BlockLayout, w=None) -> SlaForwardState:
    """forward.cpp:81-172 -- injected label grid (rows may have no critical block)."""
    return _op_for(q, cfg, layout).forward(q, k, v, w, mask=mask)


def combine_outputs(state: SlaForwardState, w) -> torch.Tensor:
    """forward.cpp:187-195: O = O^s + O^l W on the device.  (sla_forward with w already returns the
    fused result in state.o.)"""
    return state.op.combine(state, w)


def proj_backward(d_out, linear_out, w):
    """backward.cpp:12-22: (dO^s, dO^l, dW) = (dO, dO W^T, O^l^T dO) for one [N, d] unit."""
    if d_out.shape != linear_out.shape:
        raise ValueError("proj_backward: shape mismatch")
    n, d = d_out.shape[-2:]
    op = SLA(1, 1, n, d, 64 if n % 64 == 0 else n, 64 if n % 64 == 0 else n, SlaConfig(), d_out.dtype,
             d_out.device)
    dos, dol, dw = op.proj_backward(d_out.reshape(1, 1, n, d).contiguous(),
                                    linear_out.reshape(1, 1, n, d).contiguous(), w.reshape(1, d, d))
    return dos.reshape(d_out.shape), dol.reshape(d_out.shape), dw.reshape(d, d)


def sla_backward(state: SlaForwardState, q, k, v, d_out_sparse, d_out_linear, parts: bool = False) -> SlaGradients:
    """backward.hpp:25-38: gradients through both branches from independent cotangents
    (dO^s for the sparse branch, dO^l for the linear one); dproj = O^l^T dO^s."""
    return state.op.backward(state, q, k, v, None, d_out_sparse, parts=parts, d_out_linear=d_out_linear)


def sla_step_backward(state: SlaForwardState, q, k, v, w, d_out, parts: bool = False) -> SlaGradients:
    """proj_backward + sla_backward fused, from the combined-output cotangent (the reference's
    training-step sequence, finetune.cpp:44-61)."""
    return state.op.backward(state, q, k, v, w, d_out, parts=parts)
