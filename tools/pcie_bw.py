"""Pinned host <-> device copy bandwidth (the roofline of bench.py's e2e):
H2D alone, D2H alone, and both directions concurrently on two streams."""
import json
import torch

dev = torch.device("cuda:0")
n = 512 << 20
h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device=dev)
d_b = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_h2d = timed(lambda: d_a.copy_(h_src, non_blocking=True))
t_d2h = timed(lambda: h_dst.copy_(d_b, non_blocking=True))
t_both = timed(both)
print(json.dumps({"bytes": n, "h2d_GBps": n / t_h2d / 1e6, "d2h_GBps": n / t_d2h / 1e6,
                  "concurrent_each_GBps": n / t_both / 1e6}))
