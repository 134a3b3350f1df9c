"""Multi-rank SLA step: the (batch x head) units of ONE global problem partitioned over ranks.

SURVEY.md 8(e): every (batch, head) unit is independent in the forward and the backward (the
reference has no cross-head state; block rows and columns of a
unit are independent, backward.cpp:68,142), so rank r runs the contiguous unit range
`partition_units(B*H, world, r)` with no collective on the data path.  The one real exchange
of a training step is dW: W is per head and shared by the batch (forward.hpp:27-30,
backward.cpp:12-22), so when a head's batch elements sit on different ranks its d x d
partials are summed -- one all-reduce of [H, d, d] f32 at the end of the step.  The
validation gather of per-unit checksums (and optionally whole units) runs outside any timed
region.

The per-unit compute is pluggable: `CudaUnits` runs the rank's units as one [1, count, N, d]
problem through libsla_b200.so; the CPU tests plug in the C oracle (tests/test_multigpu.py)
and drive this same `ShardedStep`.
"""
from __future__ import annotations

from typing import Dict, List, Optional

import torch
import torch.distributed as dist

from .shard import Shard, partition_units


def unit_seed(base: int, unit: int) -> int:
    """Inputs of unit u are a function of (base, u) only, so the global problem is the same at
    every world size and sharded results can be compared with the one-rank run."""
    return base + 7919 * unit


class UnitCompute:
    """Interface of the per-rank compute.  Tensors are per local unit: [count, N, d] / [count, d, d]."""

    def step(self) -> None:  # fwd + bwd of every local unit
        raise NotImplementedError

    def dw_units(self) -> torch.Tensor:  # [count, d, d] f32: O^l_u^T dO_u of each unit
        raise NotImplementedError

    def outputs(self) -> Dict[str, torch.Tensor]:  # o, dq, dk, dv: [count, N, d]
        raise NotImplementedError


class CudaUnits(UnitCompute):
    """The rank's units as one SLA problem (batch 1, `count` heads) on one GPU, inputs generated
    on the device from the per-unit seeds.  W of a unit is its head's W."""

    def __init__(self, shard: Shard, heads: int, n: int, d: int, b: int, cfg, device, seed: int = 1234):
        from .sla import SLA

        self.shard, self.heads, self.n, self.d = shard, heads, n, d
        self.device = torch.device(device)
        cnt = shard.count
        self.op = SLA(1, cnt, n, d, b, b, cfg, torch.bfloat16, self.device)
        shape = (1, cnt, n, d)
        mk = lambda: torch.empty(shape, dtype=torch.bfloat16, device=self.device)  # noqa: E731
        self.q, self.k, self.v, self.do = mk(), mk(), mk(), mk()
        g = torch.Generator(device=self.device)
        for i, u in enumerate(shard.units):
            g.manual_seed(unit_seed(seed, u))
            for t in (self.q, self.k, self.v, self.do):
                t[0, i].copy_(torch.randn((n, d), generator=g, device=self.device))
        w_heads = torch.empty((heads, d, d), dtype=torch.bfloat16, device=self.device)
        for h in range(heads):
            g.manual_seed(unit_seed(seed + 1, 1_000_000 + h))
            w_heads[h].copy_(torch.randn((d, d), generator=g, device=self.device) * 0.1)
        self.w_heads = w_heads
        idx = torch.tensor([u % heads for u in shard.units], dtype=torch.long, device=self.device)
        self.w = w_heads.index_select(0, idx).contiguous() if cnt else w_heads[:0]
        self.state = self.op.new_state()
        self.o, self.o_s, self.o_l = mk(), mk(), mk()
        self.lse = torch.empty(shape[:-1], dtype=torch.float32, device=self.device)
        self.dq, self.dk, self.dv = mk(), mk(), mk()
        self.dw = torch.empty((cnt, d, d), dtype=torch.float32, device=self.device)
        self.launches = 0

    def step(self) -> None:
        st = self.op.forward(self.q, self.k, self.v, self.w, state=self.state,
                             out=(self.o, self.o_s, self.o_l, self.lse))
        n1 = self.op.launches()
        self.op.backward(st, self.q, self.k, self.v, self.w, self.do, out=(self.dq, self.dk, self.dv, self.dw))
        self.launches += n1 + self.op.launches()
        self.last_state = st

    def dw_units(self) -> torch.Tensor:
        return self.dw

    def outputs(self) -> Dict[str, torch.Tensor]:
        return {"o": self.o[0], "dq": self.dq[0], "dk": self.dk[0], "dv": self.dv[0]}


class ShardedStep:
    """One rank's share of a B x H SLA fwd+bwd step (rank/world from torch.distributed, or 0/1)."""

    def __init__(self, batch: int, heads: int, d: int, world: int = 1, rank: int = 0,
                 group=None):
        self.batch, self.heads, self.d = batch, heads, d
        self.world, self.rank, self.group = world, rank, group
        self.n_units = batch * heads
        self.shard = partition_units(self.n_units, world, rank)
        self.compute: Optional[UnitCompute] = None
        self.dw: Optional[torch.Tensor] = None
        self._dw_idx: Dict[torch.device, torch.Tensor] = {}

    @property
    def units(self) -> List[int]:
        return list(self.shard.units)

    def attach(self, compute: UnitCompute) -> "ShardedStep":
        self.compute = compute
        return self

    def reduce_dw(self) -> torch.Tensor:
        """dW[h] = sum over every unit (b, h) of O^l_u^T dO_u (backward.cpp:46 summed over the
        batch): local scatter-add, then one all-reduce when the world is larger than one."""
        part = self.compute.dw_units()
        dw = torch.zeros((self.heads, self.d, self.d), dtype=torch.float32, device=part.device)
        if self.shard.count:
            idx = self._dw_idx.get(part.device)
            if idx is None:  # built once per device: no host->device copy inside a step (graph capture)
                idx = torch.tensor([u % self.heads for u in self.units], dtype=torch.long, device=part.device)
                self._dw_idx[part.device] = idx
            dw.index_add_(0, idx, part.float())
        if self.world > 1:
            if dw.is_cuda and dist.get_backend(self.group) == "gloo":  # gloo moves host tensors
                host = dw.cpu()
                dist.all_reduce(host, group=self.group)
                dw.copy_(host)
            else:
                dist.all_reduce(dw, group=self.group)
        self.dw = dw
        return dw

    def step(self) -> None:
        self.compute.step()
        self.reduce_dw()

    # ---- validation (outside timed regions) ------------------------------------------------
    def unit_checksums(self) -> torch.Tensor:
        """[count, 8] f64 per local unit: sum and sum of |x| of o, dq, dk, dv."""
        outs = self.compute.outputs()
        cols = []
        for nm in ("o", "dq", "dk", "dv"):
            x = outs[nm].double().reshape(self.shard.count, -1)
            cols += [x.sum(1), x.abs().sum(1)]
        return torch.stack(cols, 1) if self.shard.count else torch.zeros((0, 8), dtype=torch.float64)

    def gather_checksums(self, device=None) -> Optional[torch.Tensor]:
        """All units' checksums on rank 0 ([B*H, 8]); None elsewhere (NCCL or gloo)."""
        from .shard import gather_units

        local = self.unit_checksums()
        if device is not None:
            local = local.to(device)
        return gather_units(local, self.shard, self.n_units, group=self.group)

    def gather_outputs(self, name: str) -> Optional[torch.Tensor]:
        from .shard import gather_units

        return gather_units(self.compute.outputs()[name].contiguous(), self.shard, self.n_units, group=self.group)


# ---------------------------------------------------------------------------------------------
# Finer than a (batch, head) unit: one head split over ranks (SURVEY.md 8(e) "sub-head split",
# 8(f) item 4 "sequence-sharded SLA").  Block rows and block columns of a unit are independent
# (backward.cpp:68 row phase, :142 column phase), so rank r owns a range of query blocks R_r for
# the forward and the row phase, and a range of key blocks C_r for the column phase.  The phases
# exchange only row summaries: D^s, lse, dH_i, dZ_i and the label grid of every row (the column
# phase of C_r needs them for all rows), and the per-rank dW partials are summed.
#   mode "subhead":  Q, K, V, dO replicated on every rank (C2 / C3 over 8 GPUs: 12 heads x 8 ranges)
#   mode "sequence": rank r holds only its token slice of Q, K, V, dO (context parallel): K and V
#                    are all-gathered for the forward / row phase, Q and dO for the column phase
# Every exchange is a rank-ordered concatenation along rows (`Exchange.gather_rows`) or a sum.
# ---------------------------------------------------------------------------------------------
class Exchange:
    """Collectives of the partitioned head over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, world: int, rank: int, group=None):
        self.world, self.rank, self.group = world, rank, group

    def gather_rows(self, x: torch.Tensor, counts: List[int]) -> torch.Tensor:
        """Concatenate every rank's x (x.shape[0] == counts[rank]) along dim 0 in rank order."""
        if self.world == 1:
            return x
        dev = x.device
        if x.is_cuda and dist.get_backend(self.group) == "gloo":  # gloo moves host tensors
            return self.gather_rows(x.cpu(), counts).to(dev)
        big = max(counts)
        pad = torch.zeros((big,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        pad[: x.shape[0]] = x
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad, group=self.group)
        return torch.cat([b[:c] for b, c in zip(bufs, counts)], 0)

    def sum(self, x: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            if x.is_cuda and dist.get_backend(self.group) == "gloo":
                y = x.cpu()
                dist.all_reduce(y, group=self.group)
                x.copy_(y)
            else:
                dist.all_reduce(x, group=self.group)
        return x


def block_ranges(t: int, world: int) -> List[range]:
    """Contiguous balanced block ranges of a T-block axis, one per rank."""
    return [partition_units(t, world, r).units for r in range(world)]


class HeadPartition:
    """One rank's part of one head's fwd + bwd: query blocks R_r, key blocks C_r (64-row blocks).

    The compute runs through two rectangular views of the library (sla_b200_problem.n_kv):
    `fwd`: this rank's query rows against all keys; `cols`: all query rows against this rank's
    keys.  Use `forward`, `backward_rows`, `exchange`, `backward_cols` in that order on every rank,
    or `step` with an Exchange."""

    def __init__(self, n: int, d: int, cfg, world: int, rank: int, device, block: int = 64):
        from .sla import SLA

        self.n, self.d, self.world, self.rank = n, d, world, rank
        t = n // block
        self.q_blocks = block_ranges(t, world)
        self.k_blocks = block_ranges(t, world)
        self.rows = [len(r) * block for r in self.q_blocks]
        self.krows = [len(r) * block for r in self.k_blocks]
        R, Cc = self.q_blocks[rank], self.k_blocks[rank]
        self.r0, self.r1 = R.start * block, R.stop * block
        self.c0, self.c1 = Cc.start * block, Cc.stop * block
        self.cfg = cfg
        self.fwd_op = SLA(1, 1, self.r1 - self.r0, d, block, block, cfg, torch.bfloat16, device, n_kv=n) \
            if self.r1 > self.r0 else None
        self.cols_op = SLA(1, 1, n, d, block, block, cfg, torch.bfloat16, device, n_kv=self.c1 - self.c0) \
            if self.c1 > self.c0 else None

    def forward(self, q_rows, k, v, w):
        """q_rows [1, 1, rows_r, d]; k, v all keys [1, 1, N, d]; w [1, d, d]."""
        self.st = self.fwd_op.forward(q_rows, k, v, w)
        return self.st

    def backward_rows(self, q_rows, k, v, w, do_rows, d_out_linear=None):
        dq, dw, ds, dh, dz = self.fwd_op.backward_rows(self.st, q_rows, k, v, w, do_rows, d_out_linear)
        self.part = {"ds": ds[0], "lse": self.st.lse.reshape(-1), "dh": dh[0], "dz": dz[0],
                     "labels": self.st.labels.reshape(self.st.labels.shape[-2], -1)}
        return dq, dw

    def exchange(self, ex: "Exchange") -> Dict[str, torch.Tensor]:
        """All rows' summaries, rank-ordered: D^s and lse by rows, dH / dZ / labels by block rows."""
        br = [len(r) for r in self.q_blocks]
        p = self.part
        self.full = {"ds": ex.gather_rows(p["ds"], self.rows), "lse": ex.gather_rows(p["lse"], self.rows),
                     "dh": ex.gather_rows(p["dh"], br), "dz": ex.gather_rows(p["dz"], br),
                     "labels": ex.gather_rows(p["labels"], br)}
        return self.full

    def backward_cols(self, q, k_own, v_own, do, full=None):
        """q, do: all query rows [1, 1, N, d]; k_own, v_own: this rank's keys [1, 1, c1 - c0, d]."""
        f = full or self.full
        t0, t1 = self.k_blocks[self.rank].start, self.k_blocks[self.rank].stop
        labels = f["labels"][:, t0:t1].contiguous()
        return self.cols_op.backward_cols(q, k_own, v_own, f["lse"].reshape(1, 1, -1), do, f["ds"].reshape(1, -1),
                                          f["dh"].unsqueeze(0), f["dz"].unsqueeze(0), labels.unsqueeze(0))

    def step(self, ex: "Exchange", q, k, v, w, do, mode: str = "subhead"):
        """fwd + bwd of this rank's part.  mode "subhead": q, k, v, do are the full head on every
        rank; "sequence": this rank's token slice (rows r0:r1 == keys c0:c1).  Returns
        (o_rows, dq_rows, dk_own, dv_own, dw summed over the ranks)."""
        if mode == "sequence":
            q_rows, do_rows, k_own, v_own = q, do, k, v
            k = ex.gather_rows(k_own[0, 0], self.krows).reshape(1, 1, self.n, self.d)
            v = ex.gather_rows(v_own[0, 0], self.krows).reshape(1, 1, self.n, self.d)
        else:
            q_rows, do_rows = q[:, :, self.r0:self.r1], do[:, :, self.r0:self.r1]
            k_own, v_own = k[:, :, self.c0:self.c1], v[:, :, self.c0:self.c1]
        st = self.forward(q_rows.contiguous(), k, v, w)
        dq, dw = self.backward_rows(q_rows.contiguous(), k, v, w, do_rows.contiguous())
        self.exchange(ex)
        if mode == "sequence":
            q = ex.gather_rows(q_rows[0, 0], self.rows).reshape(1, 1, self.n, self.d)
            do = ex.gather_rows(do_rows[0, 0], self.rows).reshape(1, 1, self.n, self.d)
        dk, dv = self.backward_cols(q, k_own.contiguous(), v_own.contiguous(), do)
        return st.o, dq, dk, dv, ex.sum(dw)
