"""Race hunt at the benchmarked shape: the C3 fwd+bwd captured into a CUDA graph and replayed
REPS times (default 300); after every replay the outputs must equal the first replay's bit for bit.

    python profiles/stress_determinism.py [reps] [d] [phi]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24006_b200 import SlaConfig  # noqa: E402
from paper_2509_24006_b200.runner import CudaUnits, ShardedStep  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
phi = sys.argv[3] if len(sys.argv) > 3 else "softmax"
dev = torch.device("cuda", 0)
runner = ShardedStep(1, 12, d, 1, 0)
comp = CudaUnits(runner.shard, 12, 32768, d, 64, SlaConfig(k_h=5.0, k_l=10.0, phi=phi), dev)
runner.attach(comp)
torch.cuda.set_stream(torch.cuda.Stream(dev))
for _ in range(3):
    comp.step()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=torch.cuda.current_stream()):
    comp.step()
g.replay()
torch.cuda.synchronize()
names = ("o", "dq", "dk", "dv")
ref = {nm: t.clone() for nm, t in comp.outputs().items()}
ref["dw"] = comp.dw.clone()
bad = 0
for it in range(reps):
    g.replay()
    outs = dict(comp.outputs())
    outs["dw"] = comp.dw
    for nm, t in outs.items():
        if not torch.equal(t, ref[nm]):
            n = int((t != ref[nm]).sum())
            print(f"replay {it}: {nm} differs in {n} elements", flush=True)
            bad += 1
print(f"d={d} phi={phi}: {reps} replays, {bad} mismatching tensors", flush=True)
sys.exit(1 if bad else 0)
