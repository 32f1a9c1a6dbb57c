"""PCIe copy rates on the box (dev tool): H2D alone, D2H alone, both at once (pinned)."""
import time
import torch

n = 100_000_000
h_in = torch.empty(n, dtype=torch.int64).pin_memory()
h_out = torch.empty(n, dtype=torch.int64).pin_memory()
d_a = torch.empty(n, dtype=torch.int64, device="cuda")
d_b = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
    t = timed(fn)
    print(f"{name}: {t*1e3:.2f} ms  {8*n/t/1e9:.1f} GB/s per direction")
