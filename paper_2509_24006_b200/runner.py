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
            idx = torch.tensor([u % self.heads for u in self.units], dtype=torch.long, device=part.device)
            dw.index_add_(0, idx, part.float())
        if self.world > 1:
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
