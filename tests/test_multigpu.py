"""CPU tests of the multi-rank path (world_size 2, gloo): the same `ShardedStep` runner that
bench.py drives with NCCL and `CudaUnits`, here with the per-unit compute plugged to the C
oracle (test infrastructure).  Under test: the (batch x head) partition, the dW all-reduce over
a head's batch elements split across ranks (backward.cpp:46 summed over the batch), and the
validation gathers -- sharded results must equal the one-rank run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_24006_b200.runner import ShardedStep, UnitCompute, unit_seed
from paper_2509_24006_b200.shard import batch_slices, gather_units, partition_units

N, D, BLK = 64, 8, 16


@pytest.mark.parametrize("n,world", [(12, 8), (320, 8), (5, 2), (2, 4), (1, 1)])
def test_partition_covers_every_unit_once(n, world):
    seen = []
    for r in range(world):
        s = partition_units(n, world, r)
        seen.extend(s.units)
        assert abs(s.count - n / world) < 1
    assert seen == list(range(n))


def test_batch_slices_order():
    s = partition_units(8 * 40, 8, 3)
    pairs = batch_slices(8, 40, s)
    assert pairs[0] == (3, 0) and pairs[-1] == (3, 39)


class OracleUnits(UnitCompute):
    """Per-unit fwd+bwd through the C oracle: O.step on seeded inputs (unit_seed)."""

    def __init__(self, shard, heads):
        self.shard, self.heads = shard, heads

    def step(self):
        from oracle import oracle as O

        outs = {"o": [], "dq": [], "dk": [], "dv": []}
        dws = []
        for u in self.shard.units:
            rng = O.Rng(unit_seed(700, u))
            q, k, v, do = (rng.gaussian(N, D) for _ in range(4))
            w = O.Rng(unit_seed(701, 1_000_000 + u % self.heads)).gaussian(D, D, 0.1)
            lab = O.dynamic_labels(q, k, BLK, BLK, 25.0, 25.0)
            r = O.step(q, k, v, w, do, lab, BLK, BLK, "softmax")
            for nm, key in (("o", "o"), ("dq", "dq_total"), ("dk", "dk_total"), ("dv", "dv")):
                outs[nm].append(r[key])
            dws.append(r["dw"])
        mk = lambda xs, shp: torch.tensor(np.stack(xs)) if xs else torch.zeros((0,) + shp, dtype=torch.float64)  # noqa: E731
        self._out = {nm: mk(xs, (N, D)) for nm, xs in outs.items()}
        self._dw = mk(dws, (D, D))

    def dw_units(self):
        return self._dw

    def outputs(self):
        return self._out


def _run(batch, heads, world, rank):
    st = ShardedStep(batch, heads, D, world, rank)
    st.attach(OracleUnits(st.shard, heads))
    st.step()
    res = {"dw": st.dw.clone(), "sums": st.gather_checksums(), "dq": st.gather_outputs("dq")}
    return res


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, batch, heads, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _run(batch, heads, world, rank)
        if rank == 0:
            torch.save(res, out_path)
        else:
            assert res["sums"] is None and res["dq"] is None
            torch.save(res["dw"], out_path + ".r1")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch,heads", [(1, 3), (2, 2), (3, 1)])
def test_sharded_step_matches_single_process(tmp_path, batch, heads):
    """2 ranks (gloo) against 1: per-unit checksums, gathered dQ and the per-head dW (whose
    batch elements straddle the ranks for (2, 2) and (3, 1)) must equal the one-rank run."""
    out = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, _free_port(), batch, heads, out), nprocs=2, join=True)
    got = torch.load(out)
    want = _run(batch, heads, 1, 0)
    assert torch.equal(got["sums"], want["sums"])
    assert torch.equal(got["dq"], want["dq"])
    # dW: the all-reduce of per-rank partial sums may order the batch additions differently
    assert torch.allclose(got["dw"], want["dw"], rtol=1e-12, atol=1e-14)
    assert torch.allclose(torch.load(out + ".r1"), want["dw"], rtol=1e-12, atol=1e-14)


def test_gather_units_uneven():
    """gather_units on a single process (world 1) is the identity."""
    s = partition_units(3, 1, 0)
    x = torch.arange(6.0).view(3, 2)
    assert torch.equal(gather_units(x, s, 3), x)


def _exchange_worker(rank, world, port, out_path):
    from paper_2509_24006_b200.runner import Exchange, block_ranges

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = 13  # block rows of one head, split 7 / 6
        ranges = block_ranges(t, world)
        mine = ranges[rank]
        counts = [len(r) for r in ranges]
        ex = Exchange(world, rank)
        rows = torch.arange(mine.start, mine.stop, dtype=torch.float64).view(-1, 1).repeat(1, 3)
        full = ex.gather_rows(rows, counts)
        total = ex.sum(torch.full((2, 2), float(rank + 1)))
        torch.save({"full": full, "total": total}, f"{out_path}.{rank}")
    finally:
        dist.destroy_process_group()


def test_partition_exchange_gathers_rank_ordered_rows(tmp_path):
    """runner.Exchange (the collectives of the sub-head / sequence-sharded head): uneven
    rank-ordered row gathers and the dW sum, world size 2 over gloo."""
    out = str(tmp_path / "ex")
    mp.spawn(_exchange_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        res = torch.load(f"{out}.{r}")
        assert torch.equal(res["full"][:, 0], torch.arange(13, dtype=torch.float64))
        assert torch.equal(res["total"], torch.full((2, 2), 3.0))


def test_block_ranges_cover_the_axis():
    from paper_2509_24006_b200.runner import block_ranges

    for t, w in ((512, 8), (13, 2), (1182, 8), (3, 4)):
        rs = block_ranges(t, w)
        assert [i for r in rs for i in r] == list(range(t))
