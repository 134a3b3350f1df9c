"""Host-buffer training step with copy / compute overlap.

The reference's API works on host matrices (forward.hpp / backward.hpp take `Mat<T>` in host
memory), so a drop-in that is handed host buffers pays PCIe both ways.  `HostTrainStep` runs
the fused SLA forward + backward on pinned host tensors and hides most of that traffic: the
(batch, head) units are independent, so it splits them into contiguous chunks (over heads when
batch == 1, over the batch otherwise) and overlaps, on three CUDA streams,

    H2D(chunk c+1)  |  forward + backward(chunk c)  |  D2H(chunk c-1)

with `slots` device-side buffers (3 by default: a chunk's inputs can land while the previous
two chunks still compute and drain).  Slots rotate across calls, so with `pipelined=True` the
next call's uploads start while this call's last downloads drain (a training loop's next batch
streaming in under the previous step's results); the caller then orders its stream after the
step(s) with `finish()`.  Every chunk runs through the same C-ABI calls as `SLA` (one
`SLA` instance per distinct chunk shape).  dW is per head: chunks over heads write disjoint
head rows; chunks over the batch accumulate into one dW (backward.cpp:46 sums over the batch).
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import torch

from .sla import SLA, SlaConfig


def _split(n: int, parts: int) -> List[Tuple[int, int]]:
    parts = max(1, min(parts, n))
    base, extra = divmod(n, parts)
    out, s = [], 0
    for i in range(parts):
        e = s + base + (1 if i < extra else 0)
        out.append((s, e))
        s = e
    return out


class HostTrainStep:
    """fwd+bwd of an SLA layer on pinned host tensors [B, H, N, d] (bf16), W [H, d, d].

    Outputs (host): o [B, H, N, d], dq, dk, dv [B, H, N, d] (bf16) and dW [H, d, d] (f32).
    The call is stream-ordered after the caller's current stream and the caller's current
    stream is made to wait for the last device->host copy, so CUDA events recorded around the
    call time the whole step.  With pipelined=True only the first call after construction or
    `finish()` waits for the caller's stream, no call makes the caller's stream wait, and
    consecutive calls overlap; `finish()` makes the caller's stream wait for every issued call.
    The host inputs of a call must not be modified until that call has finished.
    """

    def __init__(self, batch: int, heads: int, n: int, d: int, b_q: int = 64, b_kv: int = 64,
                 cfg: Optional[SlaConfig] = None, dtype=torch.bfloat16, device="cuda", chunks: int = 4,
                 slots: int = 3, pipelined: bool = False):
        self.batch, self.heads, self.n, self.d = batch, heads, n, d
        self.device = torch.device(device)
        self.dtype = dtype
        self.by_heads = batch == 1
        self.ranges = _split(heads if self.by_heads else batch, chunks)
        self.ops = {}
        for s, e in self.ranges:
            shape = (1, e - s) if self.by_heads else (e - s, heads)
            if shape not in self.ops:
                self.ops[shape] = SLA(shape[0], shape[1], n, d, b_q, b_kv, cfg, dtype, device)
        span = max(e - s for s, e in self.ranges)
        cshape = (1, span, n, d) if self.by_heads else (span, heads, n, d)
        mk = lambda dt=dtype: torch.empty(cshape, dtype=dt, device=self.device)  # noqa: E731
        self.nslots = max(2, slots)
        self.slots = []
        for _ in range(self.nslots):
            self.slots.append({
                "q": mk(), "k": mk(), "v": mk(), "do": mk(),
                "o": mk(), "o_s": mk(), "o_l": mk(), "lse": mk(torch.float32)[..., 0].contiguous(),
                "dq": mk(), "dk": mk(), "dv": mk(),
            })
        self.states = {shape: op.new_state() for shape, op in self.ops.items()}
        # W and dW alternate between two buffers across calls (call k+1's W upload may run while
        # call k still computes, and its dW while call k's dW still downloads)
        self.wb = [torch.empty((heads, d, d), dtype=dtype, device=self.device) for _ in range(2)]
        self.dwb = [torch.empty((heads, d, d), dtype=torch.float32, device=self.device) for _ in range(2)]
        self.dw_part = None if self.by_heads else torch.empty_like(self.dwb[0])
        self.s_in, self.s_c, self.s_out = (torch.cuda.Stream(self.device) for _ in range(3))
        self.ev_in = [torch.cuda.Event() for _ in range(self.nslots)]
        self.ev_c = [torch.cuda.Event() for _ in range(self.nslots)]
        self.ev_out = [torch.cuda.Event() for _ in range(self.nslots)]
        self.ev_wfree = [torch.cuda.Event() for _ in range(2)]
        self.ev_dwout = [torch.cuda.Event() for _ in range(2)]
        self.used = [False] * self.nslots
        self.wused = [False, False]
        self.pipelined = pipelined
        self.fresh = True
        self.calls = 0
        self.chunk_ctr = 0
        self.launches = 0

    def h2d_bytes(self) -> int:
        return 4 * self.batch * self.heads * self.n * self.d * 2 + self.heads * self.d * self.d * 2

    def d2h_bytes(self) -> int:
        return 4 * self.batch * self.heads * self.n * self.d * 2 + self.heads * self.d * self.d * 4

    def __call__(self, hq, hk, hv, hw, hdo, ho, hdq, hdk, hdv, hdw) -> None:
        cur = torch.cuda.current_stream(self.device)
        if not self.pipelined or self.fresh:
            for s in (self.s_in, self.s_c, self.s_out):
                s.wait_stream(cur)
            self.fresh = False
        self.launches = 0
        par = self.calls & 1
        self.calls += 1
        w_all, dw_all = self.wb[par], self.dwb[par]
        with torch.cuda.stream(self.s_in):
            if self.wused[par]:
                self.s_in.wait_event(self.ev_wfree[par])  # the compute of the call before last read W
            w_all.copy_(hw, non_blocking=True)
        S = self.nslots
        for c, (s, e) in enumerate(self.ranges):
            i = self.chunk_ctr % S  # slots rotate across calls
            self.chunk_ctr += 1
            slot = self.slots[i]
            shape = (1, e - s) if self.by_heads else (e - s, self.heads)
            op, state = self.ops[shape], self.states[shape]
            sl = (slice(0, 1), slice(s, e)) if self.by_heads else (slice(s, e),)
            view = lambda t: t[: shape[0], : shape[1]]  # noqa: E731  (slot tensors are max-span)
            with torch.cuda.stream(self.s_in):
                if self.used[i]:
                    self.s_in.wait_event(self.ev_c[i])  # the slot's previous compute is done with its inputs
                for nm, src in (("q", hq), ("k", hk), ("v", hv), ("do", hdo)):
                    view(slot[nm]).copy_(src[sl], non_blocking=True)
                self.ev_in[i].record(self.s_in)
            with torch.cuda.stream(self.s_c):
                self.s_c.wait_event(self.ev_in[i])
                if self.used[i]:
                    self.s_c.wait_event(self.ev_out[i])  # the slot's previous D2H is done with its outputs
                if c == 0 and self.wused[par]:
                    self.s_c.wait_event(self.ev_dwout[par])  # dW of the call before last has left
                q, k, v, do = (view(slot[nm]) for nm in ("q", "k", "v", "do"))
                w = w_all[s:e] if self.by_heads else w_all
                dw = dw_all[s:e] if self.by_heads else (dw_all if c == 0 else self.dw_part)
                st = op.forward(q, k, v, w, state=state,
                                out=(view(slot["o"]), view(slot["o_s"]), view(slot["o_l"]), view(slot["lse"])))
                self.launches += op.launches()
                op.backward(st, q, k, v, w, do, out=(view(slot["dq"]), view(slot["dk"]), view(slot["dv"]), dw))
                self.launches += op.launches()
                if not self.by_heads and c > 0:
                    dw_all.add_(self.dw_part)
                self.ev_c[i].record(self.s_c)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_c[i])
                for nm, dst in (("o", ho), ("dq", hdq), ("dk", hdk), ("dv", hdv)):
                    dst[sl].copy_(view(slot[nm]), non_blocking=True)
                self.ev_out[i].record(self.s_out)
            self.used[i] = True
        self.ev_wfree[par].record(self.s_c)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_stream(self.s_c)
            hdw.copy_(dw_all, non_blocking=True)
            self.ev_dwout[par].record(self.s_out)
        self.wused[par] = True
        if not self.pipelined:
            cur.wait_stream(self.s_out)

    def finish(self) -> None:
        """The caller's current stream waits for every call issued so far."""
        torch.cuda.current_stream(self.device).wait_stream(self.s_out)
        self.fresh = True
