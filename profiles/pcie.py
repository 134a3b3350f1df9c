"""PCIe floor for the e2e number: pinned H2D and D2H of one step's bytes (4 x 100.7 MB each way),
alone and concurrently on two streams."""
import torch

n = 4 * 12 * 32768 * 128  # bf16 elements of Q,K,V,dO (and of O,dQ,dK,dV)
h_in = torch.empty(n, dtype=torch.bfloat16).pin_memory()
h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d_in = torch.empty(n, dtype=torch.bfloat16, device="cuda")
d_out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, it=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


gb = n * 2 / 1e9
t1 = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t2 = timed(lambda: h_out.copy_(d_out, non_blocking=True))
t3 = timed(both)
print(f"H2D {gb:.3f} GB: {t1:.2f} ms ({gb / t1 * 1e3:.1f} GB/s); D2H: {t2:.2f} ms ({gb / t2 * 1e3:.1f} GB/s); "
      f"both concurrently: {t3:.2f} ms")
