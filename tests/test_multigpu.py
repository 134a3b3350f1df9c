"""CPU tests of the multi-rank path (world_size 2, gloo): (batch x head) partitioning, the
validation gather, and that sharded per-unit results equal the single-process run.  The per-unit
compute here is the C oracle (test infrastructure) -- the property under test is the host-side
sharding logic that bench.py and the GPU runner use with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_24006_b200.shard import batch_slices, gather_units, partition_units


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


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _unit_result(u):
    """A (batch, head) unit's forward output through the C oracle (seeded, deterministic)."""
    from oracle import oracle as O

    rng = O.Rng(700 + u)
    n, d, b = 64, 8, 16
    q, k, v = rng.gaussian(n, d), rng.gaussian(n, d), rng.gaussian(n, d)
    lab = O.dynamic_labels(q, k, b, b, 25.0, 25.0)
    st = O.forward(q, k, v, lab, b, b, "softmax")
    return np.concatenate([st["o_s"], st["o_l"]], 1)


def _worker(rank, world, port, n_units, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = partition_units(n_units, world, rank)
        local = torch.tensor(np.stack([_unit_result(u) for u in shard.units]) if shard.count else
                             np.zeros((0, 64, 16)), dtype=torch.float64)
        full = gather_units(local, shard, n_units)
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_units", [3, 4])
def test_sharded_run_matches_single_process(tmp_path, n_units):
    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), n_units, out), nprocs=2, join=True)
    got = np.load(out)
    want = np.stack([_unit_result(u) for u in range(n_units)])
    assert got.shape == want.shape
    assert (got == want).all()
