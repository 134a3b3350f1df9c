"""GPU test of the partitioned head (runner.HeadPartition): one head's fwd + bwd split over W ranks
by query-block ranges (forward, row phase) and key-block ranges (column phase), through the
rectangular views of the library (sla_b200_problem.n_kv) and the two backward phases
(sla_b200_backward_rows / _cols).  The ranks run one after another in this process; the
exchanges are the rank-ordered concatenations the NCCL path performs (runner.Exchange).

Block rows and columns are independent (backward.cpp:68, :142), so the concatenated O, dQ, dK, dV
must be BIT-identical to the one-op run; dW is a sum of per-rank partials (reassociated)."""
import numpy as np
import pytest
import torch

from paper_2509_24006_b200 import SLA, SlaConfig
from paper_2509_24006_b200.runner import HeadPartition

pytestmark = pytest.mark.gpu


class _Local:
    """Exchange stand-in for ranks run sequentially in one process."""

    def __init__(self, parts):
        self.parts = parts


def _inputs(n, d, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    mk = lambda s=1.0: (torch.randn((1, 1, n, d), generator=g, device="cuda") * s).to(torch.bfloat16)  # noqa: E731
    q, k, v, do = mk(), mk(), mk(), mk()
    w = (torch.randn((1, d, d), generator=g, device="cuda") * 0.1).to(torch.bfloat16)
    return q, k, v, do, w


@pytest.mark.parametrize("world,n,d,phi", [(2, 4096, 128, "softmax"), (3, 4160, 64, "elu1"), (8, 8192, 128, "softmax")])
def test_partitioned_head_matches_single_op(world, n, d, phi):
    cfg = SlaConfig(k_h=10.0, k_l=20.0, phi=phi)
    q, k, v, do, w = _inputs(n, d, 7 + world)
    op = SLA(1, 1, n, d, 64, 64, cfg, torch.bfloat16)
    st = op.forward(q, k, v, w)
    g = op.backward(st, q, k, v, w, do)
    torch.cuda.synchronize()

    parts = [HeadPartition(n, d, cfg, world, r, "cuda") for r in range(world)]
    dqs, dws = [], []
    for p in parts:  # forward + row phase of every rank
        qr, dor = q[:, :, p.r0:p.r1].contiguous(), do[:, :, p.r0:p.r1].contiguous()
        p.forward(qr, k, v, w)
        dq, dw = p.backward_rows(qr, k, v, w, dor)
        dqs.append(dq)
        dws.append(dw)
    # the exchange: rank-ordered concatenations of every rank's row summaries
    full = {key: torch.cat([p.part[key] for p in parts], 0) for key in ("ds", "lse", "dh", "dz", "labels")}
    dks, dvs = [], []
    for p in parts:
        dk, dv = p.backward_cols(q, k[:, :, p.c0:p.c1].contiguous(), v[:, :, p.c0:p.c1].contiguous(), do, full)
        dks.append(dk)
        dvs.append(dv)
    torch.cuda.synchronize()
    o = torch.cat([p.st.o for p in parts], 2)
    assert torch.equal(full["labels"].view(1, 1, n // 64, n // 64), st.labels)
    assert torch.equal(o, st.o)
    assert torch.equal(full["lse"].view(1, 1, n), st.lse)
    assert torch.equal(torch.cat(dqs, 2), g.dq_total)
    assert torch.equal(torch.cat(dks, 2), g.dk_total)
    assert torch.equal(torch.cat(dvs, 2), g.dv)
    dw = sum(dws)
    err = ((dw - g.dproj).abs().max() / g.dproj.abs().max()).item()
    assert err <= 1e-5, err


def test_rectangular_view_rejects_multi_unit():
    with pytest.raises(ValueError, match="partitioned view"):
        SLA(1, 2, 1024, 64, 64, 64, SlaConfig(), torch.bfloat16, "cuda", n_kv=2048)


def _worker(rank, world, port, mode, n, d, out):
    import os

    import torch.distributed as dist

    from paper_2509_24006_b200.runner import Exchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = SlaConfig(k_h=10.0, k_l=20.0, phi="softmax")
        q, k, v, do, w = _inputs(n, d, 99)
        p = HeadPartition(n, d, cfg, world, rank, "cuda")
        if mode == "sequence":  # this rank holds only its token slice
            sl = slice(p.r0, p.r1)
            args = (q[:, :, sl], k[:, :, sl], v[:, :, sl], w, do[:, :, sl])
        else:
            args = (q, k, v, w, do)
        o, dq, dk, dv, dw = p.step(Exchange(world, rank), *args, mode=mode)
        torch.cuda.synchronize()
        torch.save({"o": o.cpu(), "dq": dq.cpu(), "dk": dk.cpu(), "dv": dv.cpu(), "dw": dw.cpu()}, f"{out}.{rank}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["subhead", "sequence"])
def test_partitioned_step_two_processes(tmp_path, mode):
    """HeadPartition.step in 2 processes (gloo; both on cuda:0): sub-head split with replicated
    inputs, and sequence sharding where each rank holds its token slice and K / V / Q / dO are
    all-gathered.  Concatenated results equal the one-op run."""
    import socket

    import torch.multiprocessing as mp

    n, d, world = 4096, 128, 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / "part")
    mp.spawn(_worker, args=(world, port, mode, n, d, out), nprocs=world, join=True)
    q, k, v, do, w = _inputs(n, d, 99)
    op = SLA(1, 1, n, d, 64, 64, SlaConfig(k_h=10.0, k_l=20.0, phi="softmax"), torch.bfloat16)
    st = op.forward(q, k, v, w)
    g = op.backward(st, q, k, v, w, do)
    res = [torch.load(f"{out}.{r}") for r in range(world)]
    for key, want in (("o", st.o), ("dq", g.dq_total), ("dk", g.dk_total), ("dv", g.dv)):
        got = torch.cat([r[key] for r in res], 2)
        assert torch.equal(got, want.cpu()), key
    for r in res:
        assert ((r["dw"] - g.dproj.cpu()).abs().max() / g.dproj.abs().max().cpu()).item() <= 1e-5
