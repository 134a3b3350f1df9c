"""PyTorch caller of the SLA operator: a torch.autograd.Function over the C-ABI.

SURVEY.md section 8(f) item 2: the real caller of SLA in a DiT is an attention layer that
wants `o = sla(q, k, v)` with autograd.  The reference's own caller is the fine-tuning loop
(finetune.cpp:44-61): forward (sla_forward + combine_outputs), then proj_backward +
sla_backward from the cotangent of the combined output.  `SparseLinearAttention` does the
same through libsla_b200.so:

  forward : mask prediction, fused sparse + linear forward, O = O^s + O^l W  (one C-ABI call)
  backward: dQ_total, dK_total, dV and dW                                   (one C-ABI call)

Layouts: "bhnd" ([B, H, N, d], the library's native unit-major layout) or "bnhd" ([B, N, H, d],
the usual DiT projection output, passed as-is with SLA_B200_FLAG_BNHD).  W is the per-head projection [H, d, d] (indexed [in][out]) or one
shared [d, d] matrix; its gradient comes back in the same shape (a shared W receives the
sum over heads).  Operators are cached per (shape, config, dtype, device).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Optional, Tuple

import torch

from .sla import SLA, SlaConfig, SlaForwardState

_OPS: Dict[Tuple, SLA] = {}


def _op(batch: int, heads: int, n: int, d: int, b_q: int, b_kv: int, cfg: SlaConfig,
        dtype: torch.dtype, device: torch.device) -> SLA:
    key = (batch, heads, n, d, b_q, b_kv, cfg.k_h, cfg.k_l, cfg.phi, cfg.mask_precision,
           cfg.check_finite, cfg.force_generic, cfg.ragged, cfg.bnhd, dtype, device)
    op = _OPS.get(key)
    if op is None:
        op = SLA(batch, heads, n, d, b_q, b_kv, cfg, dtype, device)
        _OPS[key] = op
    return op


class _SlaFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, w, op: SLA):  # q, k, v: [B, H, N, d] contiguous
        st = op.forward(q, k, v, w)
        ctx.op = op
        # the forward state is kept as saved tensors only (no Python reference to the returned O:
        # that would form the cycle o.grad_fn -> ctx -> state -> o and hold each step's buffers
        # until the cyclic GC runs); it is rebuilt around them in backward
        ctx.save_for_backward(q, k, v, w, st.o_s, st.o_l, st.lse, st.state)
        return st.o

    @staticmethod
    def backward(ctx, d_out):
        q, k, v, w, o_s, o_l, lse, state = ctx.saved_tensors
        op = ctx.op
        st = SlaForwardState(None, o_s, o_l, lse, op.labels_of(state), op, state)
        g = op.backward(st, q, k, v, w, d_out.contiguous())
        return g.dq_total, g.dk_total, g.dv, g.dproj.to(w.dtype), None


def sparse_linear_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, w: torch.Tensor,
                            cfg: Optional[SlaConfig] = None, layout: str = "bhnd",
                            b_q: int = 64, b_kv: int = 64) -> torch.Tensor:
    """O = SLA(q, k, v) with the linear-branch projection W; differentiable in q, k, v, W."""
    cfg = cfg or SlaConfig(k_h=5.0, k_l=10.0, phi="softmax")
    if layout not in ("bhnd", "bnhd"):
        raise ValueError(f"sparse_linear_attention: unknown layout {layout!r}")
    if q.dim() != 4 or k.shape != q.shape or v.shape != q.shape:
        raise ValueError("sparse_linear_attention: q, k, v must share one 4-D shape")
    q, k, v = (t.contiguous() for t in (q, k, v))
    if layout == "bnhd":  # token-major tensors go to the library as they are (SLA_B200_FLAG_BNHD)
        cfg = dataclasses.replace(cfg, bnhd=True)
        batch, n, heads, d = q.shape
    else:
        batch, heads, n, d = q.shape
    shared_w = w.dim() == 2
    if shared_w:
        if w.shape != (d, d):
            raise ValueError("sparse_linear_attention: W must be [d, d] or [H, d, d]")
        w_h = w.unsqueeze(0).expand(heads, d, d)
    else:
        if w.shape != (heads, d, d):
            raise ValueError("sparse_linear_attention: W must be [d, d] or [H, d, d]")
        w_h = w
    w_h = w_h.to(q.dtype).contiguous()
    op = _op(batch, heads, n, d, b_q, b_kv, cfg, q.dtype, q.device)
    return _SlaFn.apply(q, k, v, w_h, op)


class SparseLinearAttention(torch.nn.Module):
    """Attention core of a DiT block: o = SLA(q, k, v) with a learned per-head projection W
    of the linear branch (initialised to zero, as the paper's fine-tuning starts from the
    sparse branch alone)."""

    def __init__(self, heads: int, head_dim: int, cfg: Optional[SlaConfig] = None,
                 layout: str = "bnhd", shared_proj: bool = False, dtype=torch.bfloat16):
        super().__init__()
        self.cfg = cfg or SlaConfig(k_h=5.0, k_l=10.0, phi="softmax")
        self.layout = layout
        shape = (head_dim, head_dim) if shared_proj else (heads, head_dim, head_dim)
        self.proj = torch.nn.Parameter(torch.zeros(shape, dtype=dtype))

    def forward(self, q, k, v):
        return sparse_linear_attention(q, k, v, self.proj, self.cfg, self.layout)
