"""bench.py's multi-rank path end to end on one GPU: `--gpus 2` re-launches itself under
torch.distributed.run; the two ranks share the device (collectives over gloo, as on a one-GPU
box; NCCL on a multi-GPU node).  The global problem at N = 2 (weak scaling: batch 2) must
contain the N = 1 problem unit for unit -- the gathered per-unit checksums agree -- and the line
must report n_gpus = 2 and every unit."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "2", "--warmup", "3",
           "--no-dense", "--no-cpu-baseline", "--no-e2e", "--no-sustained", *args]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    if out.returncode != 0 and os.path.isdir(os.path.join(ROOT, "gpurun_out")):
        with open(os.path.join(ROOT, "gpurun_out", "multirank_failure.log"), "w") as f:
            f.write(out.stdout + "\n---- stderr ----\n" + out.stderr)
    assert out.returncode == 0, out.stderr[:3000] + "\n...\n" + out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_two_ranks_partition_the_global_problem():
    one = _bench()
    two = _bench("--gpus", "2")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert one["config"]["units"] == 2 and two["config"]["units"] == 4  # weak scaling: batch = world
    assert two["validation"]["units"] == 4
    assert two["validation"]["checksums"][:2] == one["validation"]["checksums"]
    assert two["gpu_launches_per_step"] == one["gpu_launches_per_step"]
