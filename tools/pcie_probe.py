"""Pinned host <-> device copy rates: one direction, both at once, and split over two streams."""
import torch

n = 1 << 28  # 512 MiB of bf16 pairs
h = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
d = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
ss = [torch.cuda.Stream() for _ in range(4)]


def timed(fn, reps=3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in ss:
        s.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        fn()
    for s in ss:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


B = n * 2
def h2d1():
    with torch.cuda.stream(ss[0]):
        d[0].copy_(h[0], non_blocking=True)
def d2h1():
    with torch.cuda.stream(ss[1]):
        h[1].copy_(d[1], non_blocking=True)
def both():
    h2d1(); d2h1()
def h2d2():
    with torch.cuda.stream(ss[0]):
        d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(ss[2]):
        d[2].copy_(h[2], non_blocking=True)
def both2():
    h2d2()
    with torch.cuda.stream(ss[1]):
        h[1].copy_(d[1], non_blocking=True)
    with torch.cuda.stream(ss[3]):
        h[3].copy_(d[3], non_blocking=True)
print("H2D GB/s", B / timed(h2d1) / 1e6)
print("D2H GB/s", B / timed(d2h1) / 1e6)
t = timed(both)
print("both: each GB/s", B / t / 1e6)
print("H2D on 2 streams GB/s", 2 * B / timed(h2d2) / 1e6)
t = timed(both2)
print("both on 2+2 streams: each GB/s", 2 * B / t / 1e6)
