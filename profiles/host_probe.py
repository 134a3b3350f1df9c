"""Host enqueue cost of one C3 fwd+bwd step against its GPU time, eager and as a CUDA graph.

    python profiles/host_probe.py [steps]

Prints, per mode: host microseconds to enqueue one step (no synchronisation inside the loop),
device ms per step (CUDA events), and for HostTrainStep (the e2e path, 12 chunks) the host time
per call.  A step whose host enqueue time exceeds its device time is launch-bound on that host.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24006_b200 import SlaConfig  # noqa: E402
from paper_2509_24006_b200.runner import CudaUnits, ShardedStep  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
cfg = SlaConfig(k_h=5.0, k_l=10.0, phi="softmax")
runner = ShardedStep(1, 12, 128, 1, 0)
comp = CudaUnits(runner.shard, 12, 32768, 128, 64, cfg, dev)
runner.attach(comp)
for _ in range(5):
    runner.step()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run(fn, label):
    torch.cuda.synchronize()
    e0.record(st)
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    t1 = time.perf_counter()
    e1.record(st)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label}: host enqueue {1e6 * (t1 - t0) / steps:.0f} us/step, device {e0.elapsed_time(e1) / steps:.3f} ms/step, "
          f"wall {1e3 * (t2 - t0) / steps:.3f} ms/step", flush=True)


# per-call pieces of the eager step
op = comp.op
t0 = time.perf_counter()
for _ in range(steps):
    stt = op.forward(comp.q, comp.k, comp.v, comp.w, state=comp.state, out=(comp.o, comp.o_s, comp.o_l, comp.lse))
t1 = time.perf_counter()
for _ in range(steps):
    op.backward(stt, comp.q, comp.k, comp.v, comp.w, comp.do, out=(comp.dq, comp.dk, comp.dv, comp.dw))
t2 = time.perf_counter()
torch.cuda.synchronize()
print(f"op.forward host {1e6 * (t1 - t0) / steps:.0f} us/call, op.backward host {1e6 * (t2 - t1) / steps:.0f} us/call")
t0 = time.perf_counter()
for _ in range(steps):
    runner.reduce_dw()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"reduce_dw host {1e6 * (t1 - t0) / steps:.0f} us/call")

run(runner.step, "eager")
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(st)
with torch.cuda.stream(side):
    runner.step()
torch.cuda.synchronize()
with torch.cuda.graph(g):
    runner.step()
torch.cuda.synchronize()
run(g.replay, "graph")
run(runner.step, "eager again")
