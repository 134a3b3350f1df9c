"""Where the e2e step's time goes (HostTrainStep, C3 12 heads): full step vs the same copy
pattern without compute, per chunk count; per-chunk event timeline of one step."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24006_b200 import SlaConfig, HostTrainStep
dev = torch.device("cuda:0"); B, H, N, d = 1, 12, 32768, 128
shape = (1, H, N, d)
hs = [torch.randn(shape).bfloat16().pin_memory() for _ in range(4)]
hw = (torch.randn((H, d, d)) * 0.1).bfloat16().pin_memory()
ho = [torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
hdw = torch.empty((H, d, d), dtype=torch.float32).pin_memory()
cfg = SlaConfig(k_h=5, k_l=10, phi="softmax")
def timeit(fn, steps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps
res = {}
for chunks in (3, 4, 6, 12):
    for pipe in (False, True):
        hts = HostTrainStep(1, H, N, d, 64, 64, cfg, torch.bfloat16, dev, chunks=chunks, pipelined=pipe)
        def step():
            hts(hs[0], hs[1], hs[2], hw, hs[3], ho[0], ho[1], ho[2], ho[3], hdw)
        def steps10():
            for _ in range(10): step()
            hts.finish()
        res[f"{'pipe' if pipe else 'full'}_{chunks}"] = timeit(steps10, steps=1) / 10
        del hts; torch.cuda.empty_cache()
# one-direction and bidirectional floors on the whole tensors
dq = [torch.empty(shape, dtype=torch.bfloat16, device=dev) for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def h2d():
    for a, b in zip(dq, hs): a.copy_(b, non_blocking=True)
def d2h():
    for a, b in zip(ho, dq): a.copy_(b, non_blocking=True)
def both():
    cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): h2d()
    with torch.cuda.stream(s2): d2h()
    cur.wait_stream(s1); cur.wait_stream(s2)
res["h2d_only"] = timeit(h2d); res["d2h_only"] = timeit(d2h); res["both"] = timeit(both)
print(json.dumps({k: round(v, 3) for k, v in res.items()}))
