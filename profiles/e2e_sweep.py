"""Pipelined HostTrainStep per-step time (C3, 12 heads) over chunk and slot counts, 20 steps each,
against the bidirectional copy floor of the same bytes."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24006_b200 import SlaConfig, HostTrainStep
dev = torch.device("cuda:0"); H, N, d = 12, 32768, 128
shape = (1, H, N, d)
hs = [torch.randn(shape).bfloat16().pin_memory() for _ in range(4)]
hw = (torch.randn((H, d, d)) * 0.1).bfloat16().pin_memory()
ho = [torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
hdw = torch.empty((H, d, d), dtype=torch.float32).pin_memory()
cfg = SlaConfig(k_h=5, k_l=10, phi="softmax")
res = {}
for slots in (3, 4):
    for chunks in (2, 3, 4, 6, 12):
        hts = HostTrainStep(1, H, N, d, 64, 64, cfg, torch.bfloat16, dev, chunks=chunks, slots=slots, pipelined=True)
        step = lambda: hts(hs[0], hs[1], hs[2], hw, hs[3], ho[0], ho[1], ho[2], ho[3], hdw)
        for _ in range(3): step()
        hts.finish(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): step()
        hts.finish(); e1.record(); torch.cuda.synchronize()
        res[f"s{slots}_c{chunks}"] = round(e0.elapsed_time(e1) / 20, 3)
        del hts; torch.cuda.empty_cache()
dq = [torch.empty(shape, dtype=torch.bfloat16, device=dev) for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        for a, b in zip(dq, hs): a.copy_(b, non_blocking=True)
    with torch.cuda.stream(s2):
        for a, b in zip(ho, dq): a.copy_(b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for _ in range(2): both()
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): both()
e1.record(); torch.cuda.synchronize(); res["copy_floor_both"] = round(e0.elapsed_time(e1) / 10, 3)
print(json.dumps(res))
