"""Pinned host <-> device copy bandwidth: H2D alone, D2H alone, both at once."""
import torch

n = 1 << 30   # 8 GiB of fp64... use 1 GiB doubles = 8 GB? keep 2^28 doubles = 2 GiB
n = 1 << 28
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e-3


def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


B = n * 8
for name, fn, bytes_ in (("H2D", h2d, B), ("D2H", d2h, B), ("both", both, 2 * B)):
    fn()
    t = min(timed(fn) for _ in range(3))
    print(f"{name}: {bytes_ / t / 1e9:.1f} GB/s ({t * 1e3:.1f} ms for {bytes_ / 1e9:.2f} GB)")
