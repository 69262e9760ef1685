#!/usr/bin/env python
"""bench.py — composited VDIs/s of the sort-last VDI compositing hot path on
1..8 B200 (BASELINE.json metric), with the merge's HBM roofline fraction, the
search's ALU roofline, an end-to-end (host buffers) number and the CPU
oracle's baseline.

A step composites VDIs in the paper's strip mode: strip
bounds, the device-driven exchange of the strip slices (N > 1), receive-side
scan, per-list merge / gamma search / full-representation write, and the
gather to rank 0.  N = 1: one VDI per step.  N > 1: F VDIs per step enqueued
back to back (no host synchronisation inside a step: frame f+1's exchange
and merge overlap frame f's gather on the other ranks), all gathered to rank
0.  Inputs (untimed): the config's synthetic volume raycast into per-PE dense
sub-VDIs by vdi_generate_subvdi for the paper's timing protocol
(the camera rotates 10 degrees every 10th iteration; views V0
and V1), resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--pes n] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")
# stdout carries exactly one JSON line: everything else written to fd 1 (the
# NCCL banner, library chatter) is sent to stderr; emit() writes the line.
_JSON_FD = os.dup(1)
os.dup2(2, 1)


def emit(obj):
    os.write(_JSON_FD, (json.dumps(obj) + "\n").encode())


import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "composited VDIs/sec at 1080p k=20"
UNIT = "VDIs/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region: samples
    every 20 ms, line-buffered, selected by their own timestamps."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []  # (unix time, fields)
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        cmd = ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
               "-lms", "20"]
        try:
            try:
                self.proc = subprocess.Popen(["stdbuf", "-oL"] + cmd, stdout=subprocess.PIPE,
                                             stderr=subprocess.DEVNULL, text=True)
            except FileNotFoundError:
                self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:  # sampling is live before timing starts
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        import datetime
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = time.time()
            self.rows.append((ts, f))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        t = time.time()
        while self.proc and time.time() - t < 0.5 and not any(ts >= self.t1 for ts, _ in self.rows[-3:]):
            time.sleep(0.005)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.t0 is None or self.t1 is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = [f for ts, f in self.rows if self.t0 - 0.01 <= ts <= self.t1 + 0.01]
        if not rows:  # region shorter than the sampling period: the first sample after its start
            after = [f for ts, f in self.rows if ts >= self.t0]
            rows = after[:1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "diag": {"rows": len(self.rows), "t0": self.t0, "t1": self.t1,
                             "last": self.rows[-1][0] if self.rows else None}}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def workload_name(cfg, view):
    return (f"{cfg.name}: {cfg.n_pes} PEs, {cfg.W}x{cfg.H}, k_in={cfg.k_in}, k_out={cfg.k_out}, "
            f"{cfg.volume.upper()}-like {cfg.dims[0]}x{cfg.dims[1]}x{cfg.dims[2]}, {cfg.decomp} decomposition, "
            f"view V{view}")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def stats_ms(xs):
    xs = sorted(xs)
    if not xs:
        return {}
    p95 = xs[min(len(xs) - 1, int(round(0.95 * (len(xs) - 1))))]
    return {"mean": statistics.mean(xs), "median": statistics.median(xs), "p95": p95, "n": len(xs)}


# ---------------------------------------------------------------------------
# oracle helpers (cpu_baseline, parity_sample and --impl reference ONLY)
# ---------------------------------------------------------------------------
def oracle_band_inputs(cfg, vol_host, tf, cam, dec, rows, threads):
    import oracle
    sc = oracle.scene(vol_host, cfg.dims, tf, cam, dec)
    P = cfg.W * cfg.H
    r0 = cfg.H // 2 - rows // 2
    pix = np.arange(r0 * cfg.W, (r0 + rows) * cfg.W, dtype=np.int64)
    pes = []
    for pe in range(cfg.n_pes):
        g = oracle.generate_pixels(sc, pe, cfg.k_in, pix, n_threads=threads)
        pes.append(oracle.pixels_to_dense(g, P, pix))
    return pes, pix


_band_out = {}


def oracle_setup_seconds(cfg, pes, pix, threads, reps=3):
    """The oracle's per-call cost that does not scale with the band (its
    simulated all-to-all copies every record of the image):
    the time of a one-list band, min over reps."""
    import oracle
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.composite(pes, cfg.W, cfg.H, 1, cfg.k_out, pix_begin=int(pix[0]), pix_end=int(pix[0]) + 1,
                         n_threads=threads, with_stats=True, out=_band_out.get((cfg.W, cfg.H, cfg.k_out)))
        ts.append(time.perf_counter() - t0)
    return min(ts)


def vdi_seconds(t_band, t_setup, frac):
    """Whole-VDI oracle time extrapolated from a band: the setup once plus the
    band's own work scaled to the image."""
    return t_setup + max(t_band - t_setup, 0.0) / frac


def oracle_composite_band(cfg, pes, pix, threads):
    """The oracle on one band of lists; its whole-image output arrays are
    allocated once (outside the timing), so the time is the band's work."""
    import oracle
    key = (cfg.W, cfg.H, cfg.k_out)
    if key not in _band_out:
        _band_out[key] = oracle.composite(pes, cfg.W, cfg.H, 1, cfg.k_out, pix_begin=int(pix[0]),
                                          pix_end=int(pix[0]) + 1, n_threads=threads, with_stats=True)
    t0 = time.perf_counter()
    out = oracle.composite(pes, cfg.W, cfg.H, 1, cfg.k_out, pix_begin=int(pix[0]), pix_end=int(pix[-1]) + 1,
                           n_threads=threads, with_stats=True, out=_band_out[key])
    return out, time.perf_counter() - t0


def host_volume(vol_t):
    a = vol_t.detach().cpu().numpy()
    return np.ascontiguousarray(a.view(np.uint16) if a.dtype == np.int16 else a)


def get_config(args):
    cfg = synth.config_by_name(args.config)
    if args.pes:
        cfg = synth.config_by_name(args.config, n_pes=args.pes)
    return cfg


# ---------------------------------------------------------------------------
def run_reference(args, world, rank):
    """--impl reference: the CPU oracle as it stands, on the box's host cores,
    each step a bounded sample (a band of image rows) of the same workload;
    ms_per_step is the measured band time, value the VDIs/s it extrapolates to."""
    if rank != 0:
        return
    cfg = get_config(args)
    threads = os.cpu_count() or 1
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    vol = host_volume(synth.make_volume(cfg, device=dev))
    tf = synth.tf_table(cfg.tf, cfg.tf_scale)
    cam = synth.make_camera(cfg.W, cfg.H, view=args.view)
    dec = cfg.decomposition()
    pes, pix = oracle_band_inputs(cfg, vol, tf, cam, dec, args.cpu_rows, threads)
    frac = len(pix) / (cfg.W * cfg.H)
    for _ in range(args.warmup):
        oracle_composite_band(cfg, pes, pix, threads)
    ts = [oracle_composite_band(cfg, pes, pix, threads)[1] for _ in range(args.steps)]
    band_ms = statistics.mean(ts) * 1e3
    t_setup = oracle_setup_seconds(cfg, pes, pix, threads)
    v = 1.0 / vdi_seconds(statistics.mean(ts), t_setup, frac)
    sample = (f"rows [{pix[0] // cfg.W}, {pix[-1] // cfg.W + 1}) of {cfg.H} ({len(pix)} lists, {frac:.4f} of the "
              f"image); value = 1 / (setup + (band time - setup) / band fraction), setup = a one-list call "
              f"({t_setup * 1e3:.1f} ms: the oracle's simulated all-to-all copies every record)")
    emit({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": band_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.view), "sample": sample,
                   "ms_per_step_is": "measured time of one band (the bounded sample), not of a whole VDI"},
        "step_ms": stats_ms([t * 1e3 for t in ts]),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


def run_ours(args, world, rank, local):
    # clock sampling starts now, well before the timed region (nvidia-smi can
    # take seconds to deliver its first sample on a busy box)
    with ClockSampler(local) as clk:
        return _run_ours(args, world, rank, local, clk)


def _run_ours(args, world, rank, local, clk):
    import paper_2206_14503_b200 as vdi
    from paper_2206_14503_b200 import _lib as L

    cfg = get_config(args)
    G, n, W, H, k = world, cfg.n_pes, cfg.W, cfg.H, cfg.k_out
    # VDIs per step (frames in flight): 16, at least 4 per GPU -- within a call
    # the frames overlap (push, merge, search, gather send / inflate on their
    # own streams); every call ends with a join of its streams on the caller's
    # stream, which costs ~0.05 ms per call (C3, 1 GPU: F = 4 / 8 / 16 ->
    # 0.331 / 0.319 / 0.314 ms per VDI; profiles/r2_frames_probe_g*.json for G > 1)
    F = args.frames if args.frames > 0 else max(16, 4 * G)
    img_bytes = W * H * (1 + 24 * k)
    F = max(1, min(F, int((48 << 30) // img_bytes)))  # every frame has its own full image (<= 48 GB of them)
    stream = torch.cuda.current_stream()

    def new_uid():
        if G == 1:
            return None
        import torch.distributed as dist
        obj = [vdi.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    comp = vdi.Compositor(W, H, cfg.k_in, k, n, n_ranks=G, rank=rank, flags=L.VDI_FLAG_STAGE_TIMING,
                          unique_id=new_uid(), stream=stream)

    # ---- inputs (untimed): the timing protocol of PAPER.md:366 -- views V0,
    # V1, the camera rotating 10 degrees every 10th iteration
    # (5 rotations per view) -- raycast into dense sub-VDIs resident in HBM
    t0 = time.time()
    vol = synth.make_volume(cfg, device="cuda")
    tf = synth.tf_table(cfg.tf, cfg.tf_scale)
    tft = torch.from_numpy(tf).cuda()
    dec = cfg.decomposition()
    local_ids = [pe for pe in range(n) if vdi.pe_home(n, G, pe) == rank]
    rotations = [10.0 * r for r in range(args.rotations)]
    views = [0, 1] if not args.no_v1 else [0]
    sets = {}
    # bound the resident input sets (~32 GB of HBM): the first set's size decides
    cam_probe = synth.make_camera(W, H, view=0)
    probe = [comp.generate_subvdi(vol, tft, cam_probe, dec, pe) for pe in local_ids]
    set_bytes = sum(24 * p.total + 5 * W * H for p in probe)
    max_sets = max(1, int((32 << 30) // max(1, set_bytes)))
    while len(views) * len(rotations) > max_sets and len(rotations) > 1:
        rotations = rotations[:-1]
    if len(views) * len(rotations) > max_sets:
        views = [0]
    for v in views:
        for a in rotations:
            cam = synth.make_camera(W, H, view=v, angle_deg=a)
            ps = [comp.generate_subvdi(vol, tft, cam, dec, pe) for pe in local_ids]
            sets[(v, a)] = [vdi.DenseSubVDI(p.pe_id, p.total, p.count.clone(), p.offset.clone(), p.depth.clone(),
                                            p.rgba.clone()) for p in ps]
    torch.cuda.synchronize()
    t_gen = time.time() - t0
    base = sets[(0, 0.0)]
    S_local = sum(p.total for p in base)
    S_total = int(allreduce_sum(S_local, G))
    # Phase 1 as a measured stage (outside `value`)
    g_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    g_ms = []
    cam0 = synth.make_camera(W, H, view=0)
    for _ in range(2):
        g_ev[0].record(stream)
        p0 = comp.generate_subvdi(vol, tft, cam0, dec, local_ids[0])
        g_ev[1].record(stream)
        torch.cuda.synchronize()
        g_ms.append(g_ev[0].elapsed_time(g_ev[1]))
    assert p0.total == base[0].total
    phase1 = {"ms_per_subvdi": min(g_ms), "pe": local_ids[0], "supersegments": int(p0.total),
              "note": "vdi_generate_subvdi: gamma search + count pass, scan, write pass (PAPER.md:113-118, "
                      ":150-157); not part of the timed step"}

    if rank == 0:  # rank 0's strip aliases the first rows of the image (no copy in the gather)
        image = vdi.FullVDI.empty(W, 0, H, k)
        P0 = (comp.row_end - comp.row_begin) * W
        strip = vdi.FullVDI(comp.row_begin, comp.row_end, image.count[:P0], image.depth[:P0], image.rgba[:P0])
    else:
        image = vdi.FullVDI.empty(W, 0, H, k) if args.rotating else None
        strip = comp.empty_strip()
    own_image = image if image is not None else None
    # frames in flight write distinct images (frame f's search runs beside frame f+1's pass-through)
    frame_images = ([image] + [vdi.FullVDI.empty(W, 0, H, k) for _ in range(F - 1)]) if image is not None else None
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device="cuda")

    def frame(s, root):
        comp.composite(s, strip)
        comp.gather(strip, own_image if rank == root else None, root=root)

    def timed(K, view, rotating=False, frames=F):
        """K steps of `frames` VDIs; the protocol's rotation changes every 10th step."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        cnts, nl = [], 0
        torch.cuda.synchronize()
        barrier(G)
        for i in range(K):
            s = sets[(view, rotations[(i // 10) % len(rotations)])]
            flush.zero_()
            evs[i][0].record(stream)
            if frames == 1:
                frame(s, (i % G) if rotating else 0)
            else:  # frames in flight (vdi_composite_frames; strips over all GPUs when G > 1)
                roots = [(i * frames + f) % G if rotating else 0 for f in range(frames)]
                comp.composite_frames([s] * frames, [frame_images[f] if r == rank else None
                                                     for f, r in enumerate(roots)], roots=roots)
            evs[i][1].record(stream)
            x = comp.counters()  # syncs the stream; outside the events
            cnts.append(x)
            nl += x["kernel_launches"] * (frames if frames == 1 else 1)
        torch.cuda.synchronize()
        barrier(G)
        return [a_.elapsed_time(b_) for a_, b_ in evs], cnts, nl

    # warm-up: every protocol set, one VDI and F in flight (the second parity
    # of merge scratch and the pools are first touched here, not while timed)
    for _ in range(args.warmup):
        frame(base, 0)
    for _ in range(2):
        for s in sets.values():
            frame(s, 0)
            comp.composite_frames([s] * F, [frame_images[f] if rank == 0 else None for f in range(F)],
                                  roots=[0] * F)
            if args.rotating and G > 1:
                roots = [f % G for f in range(F)]
                comp.composite_frames([s] * F, [frame_images[f] if r == rank else None for f, r in enumerate(roots)],
                                      roots=roots)
    torch.cuda.synchronize()
    barrier(G)

    # ---- timed region: exactly K steps, L2 flushed between steps (untimed)
    clk.mark_start()
    step_ms, cnts, launches = timed(args.steps, 0)
    clk.mark_end()
    tot_ms = allreduce_max(sum(step_ms), G)
    ms_per_step = tot_ms / args.steps
    value = F * args.steps / (tot_ms / 1e3)
    per_vdi = [t / F for t in step_ms]
    protocol = {"V0": {"vdis_per_s": value, "ms_per_vdi": stats_ms(per_vdi)}}
    if 1 in views:
        v1_ms, _, _ = timed(args.steps, 1)
        v1_tot = allreduce_max(sum(v1_ms), G)
        protocol["V1"] = {"vdis_per_s": F * args.steps / (v1_tot / 1e3), "ms_per_vdi": stats_ms([t / F for t in v1_ms])}
    protocol["note"] = (f"PAPER.md:366 protocol: {args.steps} timed iterations, camera rotated 10 deg every 10th "
                        f"iteration ({len(rotations)} rotations), views V0 and V1 (PAPER.md:364); statistics per VDI")

    # ---- N > 1: secondary modes -- a rotating root (frame f gathered on
    # rank f mod G), latency mode (1 VDI per step, stage breakdown), and the
    # full-representation pipeline of Fig. 6
    latency = rotating = full_rep = replicas = None
    K1 = max(10, args.steps // 4)
    l_ms, lstage, _ = timed(K1, 0, frames=1)
    l_tot = allreduce_max(sum(l_ms), G)
    latency = {"ms_per_vdi": l_tot / K1, "value": 1e3 * K1 / l_tot, "steps": K1,
               "ms_per_vdi_stats": stats_ms(l_ms),
               "stages_ms": {s_: statistics.mean(c_[f"ms_{s_}"] for c_ in lstage)
                             for s_ in ("exchange", "merge", "gather")},
               "note": "one VDI per step (vdi_composite + vdi_gather, no overlap between VDIs)"}
    cnts = lstage  # per-stage numbers below come from the one-VDI steps
    if G > 1:
        if args.rotating:
            r_ms, _, _ = timed(args.steps, 0, rotating=True)
            r_tot = allreduce_max(sum(r_ms), G)
            rotating = {"vdis_per_s": F * args.steps / (r_tot / 1e3), "ms_per_vdi": stats_ms([t / F for t in r_ms]),
                        "note": "frame f gathered on rank f mod G (vdi_gather_root): the root's inflate is shared"}
        compx = vdi.Compositor(W, H, cfg.k_in, k, n, n_ranks=G, rank=rank, unique_id=new_uid(), stream=stream,
                               flags=L.VDI_FLAG_STAGE_TIMING)
        fulls = [compx.dense_to_full(p) for p in base]
        ids = [p.pe_id for p in base]
        stx = compx.empty_strip()
        imx = vdi.FullVDI.empty(W, 0, H, k) if rank == 0 else None

        def full_step():
            compx.composite_fullrep(fulls, ids, stx)
            compx.gather(stx, imx)
        for _ in range(3):
            full_step()
        Kx = max(5, args.steps // 10)
        xs = []
        torch.cuda.synchronize()
        barrier(G)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(Kx):
            e0.record(stream)
            full_step()
            e1.record(stream)
            xs.append(compx.counters())
            torch.cuda.synchronize()
            xs[-1]["ms"] = e0.elapsed_time(e1)
        xm = allreduce_max(statistics.mean(x["ms"] for x in xs), G)
        full_rep = {"ms_per_vdi": xm, "value": 1e3 / xm, "steps": Kx,
                    "stages_ms": {s_: statistics.mean(c_[f"ms_{s_}"] for c_ in xs) for s_ in ("exchange", "merge", "gather")},
                    "exchange_bytes_sent_rank0": xs[-1]["bytes_sent"],
                    "note": "sub-VDIs in the full representation: fixed-size exchange, compositing from full slices "
                            "(Fig. 6 'full'); one VDI per step"}
        compx.close()
        del fulls
    # secondary: replicas -- every GPU composites whole VDIs of its own (all
    # n sub-VDIs resident on each GPU, no strips, no exchange, no gather);
    # skipped for 4K images (a second context's scratch beside the strip
    # context's would not fit next to the frame images)
    if G > 1 and img_bytes <= (2 << 30):
        comp1 = vdi.Compositor(W, H, cfg.k_in, k, n, stream=stream)
        allpes = [comp1.generate_subvdi(vol, tft, synth.make_camera(W, H, view=0), dec, pe) for pe in range(n)]
        F1 = max(1, min(F, 8, int((24 << 30) // img_bytes)))  # the root reuses its frame images; the others allocate F1
        ims1 = frame_images[:F1] if frame_images is not None else [vdi.FullVDI.empty(W, 0, H, k) for _ in range(F1)]
        for _ in range(3):
            comp1.composite_frames([allpes] * F1, ims1)
        K2 = max(10, args.steps // 4)
        r_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K2)]
        torch.cuda.synchronize()
        barrier(G)
        for i in range(K2):
            flush.zero_()
            r_evs[i][0].record(stream)
            comp1.composite_frames([allpes] * F1, ims1)
            r_evs[i][1].record(stream)
        torch.cuda.synchronize()
        barrier(G)
        rep_tot = allreduce_max(sum(a_.elapsed_time(b_) for a_, b_ in r_evs), G)
        replicas = {"vdis_per_s": G * F1 * K2 / (rep_tot / 1e3), "ms_per_vdi_per_gpu": rep_tot / (K2 * F1), "steps": K2,
                    "frames_per_step": F1,
                    "note": "secondary (not the paper's split): every GPU composites whole VDIs of its own, all n "
                            "sub-VDIs resident on each GPU, no exchange or gather; view V0"}
        del comp1, allpes, ims1

    # ---- rooflines.  Headline: the whole merge stage (every
    # merge kernel, one stream) against HBM; beside it the pass-through kernel
    # alone and the search's ALU bound.
    P_g = strip.count.numel()
    ng = (P_g + 31) // 32
    rec = cnts[-1]["records_in"]
    rec_s = cnts[-1]["records_search"]
    B_merge = 24 * rec + n * P_g + P_g * (24 * k + 1)  # SURVEY §8(d) algorithmic bytes of the merge stage
    B_fast = n * P_g + 4 * n * ng + 24 * (rec - rec_s) + P_g * (24 * k + 1)
    ms_merge = statistics.mean(c["ms_merge"] for c in cnts)
    ms_vdi_pipe = ms_per_step / F  # per VDI in the timed (frames-in-flight) steps, max over ranks
    ms_fast = statistics.mean(c["ms_fast"] for c in cnts)
    ms_search = statistics.mean(c["ms_search"] for c in cnts)
    peak, peak_src = _peaks()
    traffic = traffic_fast = None
    tp = os.path.join(ROOT, "profiles", "merge_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp)).get(cfg.name if not args.pes else f"{cfg.name}-{cfg.n_pes}")
            if isinstance(tj, dict) and G == 1:  # captured on one GPU (whole image)
                traffic, traffic_fast = tj.get("merge_stage"), tj.get("merge_fast")
        except Exception:
            pass
    # ALU roofline of the gamma search: the plain procedure's sample-steps
    # (counted on the GPU by the margin replay, VDI_FLAG_PIXEL_STATS, untimed)
    # x 20 FP32 operations / the search kernels' time
    alu = None
    if G == 1:
        cs = vdi.Compositor(W, H, cfg.k_in, k, n, flags=L.VDI_FLAG_PIXEL_STATS, stream=stream)
        sst = cs.empty_strip()
        cs.composite(base, sst)
        steps_alg = cs.counters()["sweep_steps"]
        cs.close()
        del sst
        clk_mhz = clk.summary().get("sm_mhz") or 1965.0
        fp32_peak = 148 * 128 * 2 * clk_mhz * 1e6 / 1e12  # TFLOP/s: SMs x FP32 lanes x FMA at the measured clock
        ach = 20.0 * steps_alg / (ms_search * 1e-3) / 1e12 if ms_search > 0 else 0.0
        alu = {"bound": "alu", "kernel": "search kernels (short + long gather / bisection sweeps)",
               "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": ach / fp32_peak if fp32_peak else None,
               "sweep_steps": int(steps_alg), "flop_per_step": 20, "ms": ms_search,
               "flop_per_byte": 20.0 * steps_alg / max(1, 24 * rec_s),
               "peak_source": f"148 SMs x 128 FP32 lanes x 2 (FMA) x {clk_mhz:.0f} MHz (median SM clock under load)"}
    ms_ex = statistics.mean(c["ms_exchange"] for c in cnts)
    ms_ga = statistics.mean(c["ms_gather"] for c in cnts)
    bytes_sent = cnts[-1]["bytes_sent"]
    bytes_recv = cnts[-1]["bytes_received"]
    ing_max = allreduce_max(bytes_recv, G)
    eg_max = allreduce_max(bytes_sent, G)
    ms_ex_max = allreduce_max(ms_ex, G)
    ms_push = statistics.mean(c.get("ms_push", 0.0) for c in cnts)
    push_rate_min = -allreduce_max(-(bytes_sent / max(ms_push, 1e-6) / 1e6), G) if G > 1 else 0.0

    # ---- Phase 1 + Phase 2 of one VDI
    v2r = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        torch.cuda.synchronize()
        barrier(G)
        ev0.record(stream)
        regen = [comp.generate_subvdi(vol, tft, cam0, dec, pe) for pe in local_ids]
        frame(regen, 0)
        ev1.record(stream)
        torch.cuda.synchronize()
        v2r.append(ev0.elapsed_time(ev1))
    ms_v2r = allreduce_max(min(v2r), G)
    volume_to_root = {"ms": ms_v2r, "vdis_per_s": 1e3 / ms_v2r, "pes_generated_per_rank": len(local_ids),
                      "note": "Phase 1 (vdi_generate_subvdi of every local PE) + exchange, merge and gather of one "
                              "VDI, one stream, max over ranks"}

    # ---- end to end through the C ABI with host buffers (pinned): per frame
    # the host sub-VDIs in, the composited strip back in the dense
    # representation (vdi_composite_host_dense_frames); the
    # frames cycle over the protocol's input sets (distinct inputs)
    e2e = None
    if not args.no_e2e:
        compe = vdi.Compositor(W, H, cfg.k_in, k, n, n_ranks=G, rank=rank, flags=L.VDI_FLAG_HOST_SPAN,
                               unique_id=new_uid(), stream=stream)
        keys = list(sets.keys())[: args.e2e_sets]
        host_sets, arenas = [], []
        for key in keys:
            parts = [[p.count, p.depth, p.rgba] for p in sets[key]]
            sizes = [[(t.numel() * t.element_size() + 255) // 256 * 256 for t in ts] for ts in parts]
            arena = torch.empty(max(1, sum(map(sum, sizes))), dtype=torch.uint8).pin_memory()
            hp, off = [], 0
            for p, ts, ss in zip(sets[key], parts, sizes):
                hv = []
                for t, sz in zip(ts, ss):
                    nb = t.numel() * t.element_size()
                    h = arena[off:off + nb].view(t.dtype).view(t.shape)
                    h.copy_(t)
                    hv.append(h)
                    off += sz
                hp.append(vdi.DenseSubVDI(p.pe_id, p.total, hv[0], None, hv[1], hv[2]))
            host_sets.append(hp)
            arenas.append(arena)
        P_g = strip.count.numel()
        cap = max(1, min(P_g * k, S_total))  # a list never gains supersegments: output <= input records
        outs = [(torch.empty(P_g, dtype=torch.uint8).pin_memory(), torch.empty((cap, 2), dtype=torch.float32).pin_memory(),
                 torch.empty((cap, 4), dtype=torch.float32).pin_memory()) for _ in range(2)]
        want = [compe.composite_host_dense(hs, *outs[0]) for hs in host_sets]
        compe.composite_host_dense_frames([host_sets[0]] * 2, outs)
        barrier(G)
        fr = [host_sets[f % len(host_sets)] for f in range(args.e2e_steps)]
        t0 = time.perf_counter()
        Ts = compe.composite_host_dense_frames(fr, [outs[f & 1] for f in range(args.e2e_steps)])
        dt = allreduce_max(time.perf_counter() - t0, G)
        assert all(Ts[f] == want[f % len(host_sets)] for f in range(args.e2e_steps)), (Ts, want)
        h2d = statistics.mean(sum(P_full + 24 * p.total for p in hs) for hs in host_sets for P_full in [W * H])
        d2h = statistics.mean(P_g + 24 * t for t in want)
        e2e = {"value": args.e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(allreduce_sum(h2d, G)),
               "d2h_bytes_per_step": int(allreduce_sum(d2h, G)), "frames": args.e2e_steps,
               "input_sets": len(host_sets),
               "host_link_GBs": (h2d + d2h) * args.e2e_steps / dt / 1e9,
               "note": "vdi_composite_host_dense_frames: per frame, pinned host sub-VDIs (one arena per frame, "
                       "VDI_FLAG_HOST_SPAN) -> H2D -> composite -> on-device compaction -> counts + packed "
                       "supersegments D2H, every rank; frame f's H2D overlaps frame f-1's compositing and frame "
                       "f-2's D2H; frames cycle over the protocol's input sets"}
        compe.close()

    # ---- SURVEY §8(f) f4 (N = 1): the limit case (one S~ per sub-domain
    # intersection composited to a plain image) timed like a
    # step, and the rendering quality of the composited VDI from novel
    # viewpoints (SSIM / PSNR vs DVR)
    f4 = None
    if G == 1 and not args.no_f4:
        from evaluation import psnr, ssim, to_rgb
        cl = vdi.Compositor(W, H, 32, 1, n, stream=stream)
        lim = [cl.generate_subvdi(vol, tft, cam0, dec, pe, limit=True) for pe in range(n)]
        lim = [vdi.DenseSubVDI(p.pe_id, p.total, p.count.clone(), p.offset.clone(), p.depth.clone(), p.rgba.clone())
               for p in lim]
        img = cl.composite_image(lim)
        dv = cl.render_dvr(vol, tft, cam0, W, H)
        torch.cuda.synchronize()
        err = (img - dv).abs().max().item()
        lm, dm = [], []
        for _ in range(10):
            flush.zero_()
            ev0.record(stream)
            cl.composite_image(lim, img)
            ev1.record(stream)
            torch.cuda.synchronize()
            lm.append(ev0.elapsed_time(ev1))
            ev0.record(stream)
            cl.render_dvr(vol, tft, cam0, W, H)
            ev1.record(stream)
            torch.cuda.synchronize()
            dm.append(ev0.elapsed_time(ev1))
        recs = sum(p.total for p in lim)
        frame(base, 0)
        torch.cuda.synchronize()
        qual = {}
        for ang in (5.0, 20.0):
            vc = synth.make_camera(W, H, view=0, angle_deg=ang)
            gt = to_rgb(comp.render_dvr(vol, tft, vc, W, H), W, H)
            nv = to_rgb(comp.render_novel_view(image, cam0, vc, cfg.dims, W, H), W, H)
            qual[f"{ang:g}deg"] = {"ssim": ssim(nv, gt), "psnr_db": psnr(nv, gt)}
        f4 = {"limit_case": {"ms_per_image": statistics.median(lm), "images_per_s": 1e3 / statistics.median(lm),
                             "records": int(recs), "max_abs_err_vs_dvr": err,
                             "dvr_ms_same_view": statistics.median(dm),
                             "note": "vdi_composite_image over limit sub-VDIs (vdi_generate_limit, one S~ per "
                                     "sub-domain intersection, PAPER.md:198) vs vdi_render_dvr of the whole volume"},
              "novel_view_quality_vs_dvr": qual,
              "quality_note": "the composited VDI of V0 rendered at V0 rotated by 5 / 20 degrees "
                              "(vdi_render_novel_view) vs DVR at that view (vdi_render_dvr); SSIM 11x11 Gaussian, "
                              "PSNR peak 1, RGB over black (PAPER.md:213, :364)"}
        cl.close()
        del lim

    # ---- CPU oracle baseline (rank 0, N = 1 only) + a parity band
    cpu = parity = None
    if rank == 0 and G == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        volh = host_volume(vol)
        t0 = time.perf_counter()
        pes_o, pix = oracle_band_inputs(cfg, volh, tf, cam0, dec, args.cpu_rows, threads)
        t_gen_o = time.perf_counter() - t0
        out, t = oracle_composite_band(cfg, pes_o, pix, threads)
        out, t = oracle_composite_band(cfg, pes_o, pix, threads)  # timed with its outputs allocated
        frac = len(pix) / (W * H)
        t_setup = oracle_setup_seconds(cfg, pes_o, pix, threads)
        sample = (f"rows [{pix[0] // W}, {pix[-1] // W + 1}) of {H} ({len(pix)} lists, {frac:.4f} of the image), "
                  f"oracle-generated inputs; value = 1 / (setup + (band time - setup) / band fraction), setup = a "
                  f"one-list call ({t_setup * 1e3:.1f} ms: the oracle's simulated all-to-all copies every record)")
        cpu = {"value": 1.0 / vdi_seconds(t, t_setup, frac), "unit": UNIT, "cores": threads, "cpu_model": cpu_model(),
               "kind": "oracle", "sample": sample, "seconds": t, "setup_seconds": t_setup,
               "oracle_generation_seconds": t_gen_o}
        frame(base, 0)  # the image of V0, rotation 0
        torch.cuda.synchronize()
        gc = strip.count[pix].cpu().numpy()
        gd = strip.depth[pix].cpu().numpy()
        gr = strip.rgba[pix].cpu().numpy()
        oc, od, orr = out["count"][pix], out["depth"][pix], out["rgba"][pix]
        tie = out["stats"]["margin"][pix] < 1e-6
        parity = {"lists": int(len(pix)), "ties_listed": int(tie.sum()),
                  "count_mismatch": int((gc != oc).sum()),
                  "count_mismatch_on_ties": int(((gc != oc) & tie).sum()),
                  "max_rgba_err": float(np.abs(gr - orr).max()),
                  "max_depth_rel_err": float((np.abs(gd - od) / np.maximum(np.abs(od), 1e-30)).max()),
                  "note": "every list of the band compared, ties included"}

    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg, 0), "n_pes": n, "image": f"{W}x{H}",
                       "k_in": cfg.k_in, "k_out": k, "supersegments_total": S_total,
                       "parallelism": ((f"one GPU: every PE homed on it; {F} VDIs per step in flight "
                                        f"(vdi_composite_frames: VDI f's gamma search beside VDI f+1's pass-through)")
                                       if G == 1 else
                                       f"strip mode (PAPER.md:164): each VDI split in {G} row strips, PEs block-"
                                       f"mapped to ranks, device-driven all-to-all exchange, dense gather to rank 0; "
                                       f"{F} VDIs per step in flight (vdi_composite_frames)"),
                       "frames_per_step": F,
                       "l2": f"flushed between steps ({args.flush_mb} MiB memset, untimed)",
                       "inputs": (f"sub-VDIs raycast by vdi_generate_subvdi (untimed), resident in HBM; "
                                  f"{len(sets)} input sets (views x rotations, PAPER.md:364-366)"),
                       "gen_seconds": round(t_gen, 2)},
            "roofline": {"kernel": ("merge stage per VDI with VDIs in flight (all merge kernels: receive scan, "
                                    "pass-through, gamma search, general path; VDI f's search beside VDI f+1's "
                                    "pass-through)" + ("" if G == 1 else "; per rank, exchange and gather included")),
                         "bound": "hbm", "achieved": B_merge / (ms_vdi_pipe * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": B_merge / (ms_vdi_pipe * 1e-3) / 1e9 / peak, "traffic": traffic,
                         "peak_source": peak_src, "algorithmic_bytes": int(B_merge), "ms": ms_vdi_pipe,
                         "single_vdi_merge_stage": {"ms": ms_merge, "achieved": B_merge / (ms_merge * 1e-3) / 1e9,
                                                    "frac": B_merge / (ms_merge * 1e-3) / 1e9 / peak,
                                                    "note": "one VDI, the merge kernels back to back on one stream"},
                         "merge_fast": {"kernel": "merge_fast (pass-through lists + full-representation write, "
                                                  "TMA bulk stores)", "algorithmic_bytes": int(B_fast), "ms": ms_fast,
                                        "achieved": B_fast / (ms_fast * 1e-3) / 1e9,
                                        "frac": B_fast / (ms_fast * 1e-3) / 1e9 / peak, "traffic": traffic_fast},
                         "search_alu": alu},
            "timing_protocol": protocol,
            "stages_ms": {"exchange": ms_ex, "merge": ms_merge, "gather": ms_ga,
                          "merge_scan": statistics.mean(c["ms_scan"] for c in cnts),
                          "merge_fast": ms_fast, "merge_search": ms_search},
            "phase1_generate": phase1,
            "volume_to_root_vdi": volume_to_root,
            "latency_mode": latency,
            "rotating_root": rotating,
            "replicas_whole_frames": replicas,
            "full_representation_mode": full_rep,
            "f4": f4,
            "supersegments_merged_per_s": S_total * value,
            "searched_lists": cnts[-1]["searched_lists"],
            "search_buckets": cnts[-1]["bucket_lists"], "fast_fallback_groups": cnts[-1]["fallback_groups"],
            "exchange_bytes_sent_rank0": bytes_sent, "exchange_bytes_received_rank0": bytes_recv,
            "gather_bytes_into_root": cnts[-1]["bytes_gather"],
            "nvlink_roofline": None if G == 1 else {
                "peak_GBs_per_direction": 900.0, "peak_source": "NVLink 5 nominal per GPU per direction",
                "exchange_GBs": max(ing_max, eg_max) / max(ms_ex_max, 1e-6) / 1e6,
                "exchange_frac": max(ing_max, eg_max) / max(ms_ex_max, 1e-6) / 1e6 / 900.0,
                "exchange_note": "max over ranks of max(egress, ingress) bytes / the exchange stage time (strip "
                                 "bounds + push + ready wait), one-VDI steps",
                "push_kernel_GBs": push_rate_min, "push_kernel_frac": push_rate_min / 900.0,
                "push_kernel_note": "min over ranks of the rank's pushed bytes / its push kernel's CUDA-event time "
                                    "(the NVLink egress rate of the exchange kernel itself), one-VDI steps",
                "gather_into_root_GBs": cnts[-1]["bytes_gather"] / max(ms_ga, 1e-6) / 1e6,
                "gather_into_root_frac": cnts[-1]["bytes_gather"] / max(ms_ga, 1e-6) / 1e6 / 900.0,
                "gather_note": "dense bytes into the root / gather stage time (includes the root's wait and its "
                               "inflate of the full representation)",
                # measured ceilings of peer stores on this pool's B200 pairs (profiles/nvlink_probe.cu,
                # profiles/r2_nvlink_probe.txt): the push kernel's copy loop, one direction, 1 GiB / 32 MiB
                "sm_store_ceiling_GBs": {"1GiB": 713.7, "32MiB": 603.0,
                                         "source": "profiles/r2_nvlink_probe.txt (SM peer stores; copy engines "
                                                   "778.6 / 632.8)"},
                "push_kernel_frac_of_sm_ceiling_32MiB": push_rate_min / 603.0},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity_sample": parity,
        }
        emit(res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--pes", type=int, default=0, help="override the config's PE count (C5 sweep: 2/4/8/16)")
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--rotations", type=int, default=5, help="protocol rotations of 10 degrees per view")
    ap.add_argument("--no-v1", action="store_true")
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--e2e-steps", type=int, default=24)
    ap.add_argument("--e2e-sets", type=int, default=3)
    ap.add_argument("--cpu-rows", type=int, default=64)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-f4", action="store_true", help="skip the limit-case / rendering-quality measurements")
    ap.add_argument("--rotating", action="store_true", help="N > 1: also time a root rotating over the frames")
    ap.add_argument("--frames", type=int, default=0, help="VDIs per step (frames in flight; default max(16, 4 per GPU))")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world, rank, local = dist_setup()
    if args.impl == "reference":
        # the reference arm's bounded sample per step: the cpu_baseline's band
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
