"""PCIe copy-engine probe: pinned H2D alone, D2H alone, and both concurrently (cfg3 byte counts)."""
import time

import torch

dev = torch.device("cuda:0")
h_in = torch.empty(2322432000 // 2, dtype=torch.bfloat16, pin_memory=True)
h_out = torch.empty(786240000 // 2, dtype=torch.bfloat16, pin_memory=True)
d_in = torch.empty_like(h_in, device=dev)
d_out = torch.empty_like(h_out, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


def h2d_chunked(n=40):
    with torch.cuda.stream(s1):
        for a, b in zip(d_in.chunk(n), h_in.chunk(n)):
            a.copy_(b, non_blocking=True)


a, b, c, e = timed(h2d), timed(d2h), timed(both), timed(h2d_chunked)
print(f"H2D {a:.2f} ms ({h_in.numel() * 2 / a / 1e6:.1f} GB/s)  D2H {b:.2f} ms "
      f"({h_out.numel() * 2 / b / 1e6:.1f} GB/s)  both {c:.2f} ms  H2D in 40 chunks {e:.2f} ms")
