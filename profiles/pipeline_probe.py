"""The e2e pipeline's copy pattern without libvdi: per frame 8 x (2 MB count,
8*S depth, 16*S rgba) pinned H2D copies on one stream, a 0.4 ms kernel on a
compute stream, a 95 MB D2H on a third stream; 24 frames, double-buffered.
Prints frames/s: the rate the copy engines allow for this pattern."""
import json
import time

import torch

P, S, F, OUT = 1920 * 1080, 600977, 24, 95468376
hin = [[torch.empty(n, dtype=torch.uint8).pin_memory() for n in (P, 8 * S, 16 * S)] for _ in range(8)]
din = [[[torch.empty(n, dtype=torch.uint8, device="cuda") for n in (P, 8 * S, 16 * S)] for _ in range(8)]
       for _ in range(2)]
dout = [torch.empty(OUT, dtype=torch.uint8, device="cuda") for _ in range(2)]
hout = [torch.empty(OUT, dtype=torch.uint8).pin_memory() for _ in range(2)]
sin, scomp, sout = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
tot_in = 8 * (P + 24 * S)
hflat = torch.empty(tot_in, dtype=torch.uint8).pin_memory()
dflat = [torch.empty(tot_in, dtype=torch.uint8, device="cuda") for _ in range(2)]
work = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def run(frames, one_copy=False):
    ev_in = [torch.cuda.Event() for _ in range(frames)]
    ev_c = [torch.cuda.Event() for _ in range(frames)]
    ev_o = [torch.cuda.Event() for _ in range(frames)]
    for f in range(frames):
        sl = f & 1
        with torch.cuda.stream(sin):
            if f >= 2:
                sin.wait_event(ev_c[f - 2])
            if one_copy:
                dflat[sl].copy_(hflat, non_blocking=True)
            else:
                for l in range(8):
                    for a in range(3):
                        din[sl][l][a].copy_(hin[l][a], non_blocking=True)
            ev_in[f].record(sin)
        with torch.cuda.stream(scomp):
            scomp.wait_event(ev_in[f])
            if f >= 2:
                scomp.wait_event(ev_o[f - 2])
            work.fill_(f & 255)  # ~0.2 ms of HBM writes, like the pass-through
            dout[sl].fill_(1)
            ev_c[f].record(scomp)
        with torch.cuda.stream(sout):
            sout.wait_event(ev_c[f])
            hout[sl].copy_(dout[sl], non_blocking=True)
            ev_o[f].record(sout)
    torch.cuda.synchronize()


res = {}
for one in (False, True, False, True):
    run(2, one)
    t0 = time.perf_counter()
    run(F, one)
    dt = time.perf_counter() - t0
    res.setdefault("one_h2d_copy" if one else "24_h2d_copies", []).append(F / dt)
print(json.dumps({"frames": F, "frames_per_s": res}))
