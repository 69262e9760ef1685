"""Host<->device copy bandwidth on the GPU box (the bound of bench.py's e2e):
pinned H2D of 132 MB, D2H of 95 MB (C3's per-frame bytes), alone and
concurrently on two streams.  CUDA events; prints one JSON line."""
import json

import torch

h2d_b, d2h_b = 131976288, 95468376
hin = torch.empty(h2d_b, dtype=torch.uint8).pin_memory()
hout = torch.empty(d2h_b, dtype=torch.uint8).pin_memory()
din = torch.empty(h2d_b, dtype=torch.uint8, device="cuda")
dout = torch.empty(d2h_b, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    s1.synchronize()


def d2h():
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    s2.synchronize()


def both():
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_ms": t1, "h2d_GBs": h2d_b / t1 / 1e6, "d2h_ms": t2, "d2h_GBs": d2h_b / t2 / 1e6,
                  "concurrent_ms": t3, "concurrent_frames_per_s": 1e3 / t3}))
