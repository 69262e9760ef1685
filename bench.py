#!/usr/bin/env python
"""bench.py — composited VDIs/s of the sort-last VDI compositing hot path on
1..8 B200 (BASELINE.json metric), with the merge's HBM roofline fraction,
an end-to-end (host buffers) number and the CPU oracle's baseline.

A step = one pass of the whole hot path over one VDI:
strip totals, size exchange + all-to-allv (NCCL, G > 1), receive-side scan,
per-list merge / gamma search / full-representation write, gather to rank 0.
Inputs (untimed): the config's synthetic volume raycast into per-PE dense
sub-VDIs by vdi_generate_subvdi, resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]
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


# ---------------------------------------------------------------------------
# oracle helpers (cpu_baseline and --impl reference ONLY)
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


def oracle_composite_band(cfg, pes, pix, threads):
    import oracle
    t0 = time.perf_counter()
    out = oracle.composite(pes, cfg.W, cfg.H, 1, cfg.k_out, pix_begin=int(pix[0]), pix_end=int(pix[-1]) + 1,
                           n_threads=threads, with_stats=True)
    return out, time.perf_counter() - t0


def host_volume(vol_t):
    a = vol_t.detach().cpu().numpy()
    return np.ascontiguousarray(a.view(np.uint16) if a.dtype == np.int16 else a)


# ---------------------------------------------------------------------------
def run_reference(args, world, rank):
    """--impl reference: the CPU oracle as it stands, on the box's host cores,
    each step a bounded sample (a band of image rows) of the same workload."""
    if rank != 0:
        return
    cfg = synth.config_by_name(args.config)
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
    per_vdi = statistics.mean(ts) / frac
    v = 1.0 / per_vdi
    sample = f"rows [{pix[0] // cfg.W}, {pix[-1] // cfg.W + 1}) of {cfg.H} ({len(pix)} lists, {frac:.4f} of the image)"
    emit({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_vdi * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.view), "sample": sample},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
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

    cfg = synth.config_by_name(args.config)
    G, n, W, H, k = world, cfg.n_pes, cfg.W, cfg.H, cfg.k_out
    F = args.frames if args.frames > 0 else 4 * G if G > 1 else 1  # VDIs per step (4 per rank: G=2 4160 vs 3772 VDIs/s at 2)
    flags = (L.VDI_FLAG_STAGE_TIMING | (L.VDI_FLAG_FULL_GATHER if args.full_gather else 0)
             | (L.VDI_FLAG_NCCL_EXCHANGE if args.nccl_exchange else 0)
             | (L.VDI_FLAG_PEER_READS if args.peer_reads else 0) | (L.VDI_FLAG_CE_COPIES if args.ce_copies else 0))
    stream = torch.cuda.current_stream()

    def new_uid():
        if G == 1:
            return None
        import torch.distributed as dist
        obj = [vdi.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    # strip mode (the paper's direct send: strips of one VDI on every GPU, gather to rank 0)
    comp = vdi.Compositor(W, H, cfg.k_in, k, n, n_ranks=G, rank=rank, flags=flags, unique_id=new_uid(),
                          stream=stream)
    # frames mode (G > 1): F VDIs per step, frame f composited whole by rank f mod G
    compf = (vdi.Compositor(W, H, cfg.k_in, k, n, n_ranks=G, rank=rank,
                            flags=L.VDI_FLAG_STAGE_TIMING | (L.VDI_FLAG_PEER_READS if args.peer_reads else 0)
                            | (L.VDI_FLAG_CE_COPIES if args.ce_copies else 0),
                            unique_id=new_uid(), stream=stream) if G > 1 else None)

    # ---- inputs (untimed): synthetic volume -> per-PE dense sub-VDIs in HBM;
    # frames mode gets one private copy per frame (every frame is this VDI)
    t0 = time.time()
    vol = synth.make_volume(cfg, device="cuda")
    tf = synth.tf_table(cfg.tf, cfg.tf_scale)
    tft = torch.from_numpy(tf).cuda()
    cam = synth.make_camera(W, H, view=args.view)
    dec = cfg.decomposition()
    local_ids = [pe for pe in range(n) if vdi.pe_home(n, G, pe) == rank]
    local = [comp.generate_subvdi(vol, tft, cam, dec, pe) for pe in local_ids]
    torch.cuda.synchronize()
    t_gen = time.time() - t0
    S_local = sum(p.total for p in local)
    S_total = int(allreduce_sum(S_local, G))
    # Phase 1 as a measured stage (untimed w.r.t. `value`):
    # vdi_generate_subvdi of one local PE (two-pass raycast, device scan, write)
    # timed with CUDA events; deterministic, so the regenerated output is the same
    g_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    g_ms = []
    for _ in range(2):
        g_ev[0].record(stream)
        p0 = comp.generate_subvdi(vol, tft, cam, dec, local_ids[0])
        g_ev[1].record(stream)
        torch.cuda.synchronize()
        g_ms.append(g_ev[0].elapsed_time(g_ev[1]))
    assert p0.total == local[0].total
    phase1 = {"ms_per_subvdi": min(g_ms), "pe": local_ids[0], "supersegments": int(p0.total),
              "note": "vdi_generate_subvdi: gamma search + count pass, scan, write pass (PAPER.md:113-118, "
                      ":150-157); not part of the timed step"}
    frames_local, frames_img = None, None
    if compf is not None:
        frames_local = [[vdi.DenseSubVDI(p.pe_id, p.total, p.count.clone(), p.offset.clone(), p.depth.clone(),
                                         p.rgba.clone()) for p in local] for _ in range(F)]
        frames_img = [vdi.FullVDI.empty(W, 0, H, k) if f % G == rank else None for f in range(F)]

    if G > 1 and rank == 0:  # rank 0's strip aliases the first rows of the image (no copy in the gather)
        image = vdi.FullVDI.empty(W, 0, H, k)
        P0 = (comp.row_end - comp.row_begin) * W
        strip = vdi.FullVDI(comp.row_begin, comp.row_end, image.count[:P0], image.depth[:P0], image.rgba[:P0])
    else:
        strip = comp.empty_strip()
        image = strip if G == 1 else None
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device="cuda")

    def strip_step():
        comp.composite(local, strip)
        comp.gather(strip, image)

    def frames_step():
        compf.composite_frames(frames_local, frames_img, chunks=args.chunks)

    def timed_steps(K, fn, c):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        stats, nl = [], 0
        torch.cuda.synchronize()
        barrier(G)
        for i in range(K):
            flush.zero_()
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
            x = c.counters()  # syncs the stream; outside the events
            stats.append(x)
            nl += x["kernel_launches"]
        torch.cuda.synchronize()
        barrier(G)
        return [a_.elapsed_time(b_) for a_, b_ in evs], stats, nl

    step, step_comp = (frames_step, compf) if compf is not None else (strip_step, comp)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(G)

    # ---- timed region: exactly K steps, L2 flushed between steps (untimed)
    clk.mark_start()
    step_ms, fstage, launches = timed_steps(args.steps, step, step_comp)
    clk.mark_end()
    tot_ms = allreduce_max(sum(step_ms), G)
    ms_per_step = tot_ms / args.steps
    value = F * args.steps / (tot_ms / 1e3)  # whole VDIs composited by all ranks per second

    # ---- strip (latency) mode: one VDI per step, strips on every GPU, gather
    # to rank 0 (timed paper-style per stage).
    # At G = 1 this is the timed run itself.
    latency = None
    if compf is not None:
        for _ in range(3):
            strip_step()
        K1 = max(10, args.steps // 4)
        lat_ms, stage, _ = timed_steps(K1, strip_step, comp)
        l_ms = allreduce_max(sum(lat_ms), G) / K1
        latency = {"ms_per_vdi": l_ms, "value": 1e3 / l_ms, "steps": K1,
                   "stages_ms": {s_: statistics.mean(c_[f"ms_{s_}"] for c_ in stage)
                                 for s_ in ("exchange", "merge", "gather")},
                   "note": "one VDI per step in strips over all GPUs, dense gather to rank 0"}
        frames_info = {"frames_per_step": F, "chunks": args.chunks,
                       "ms_size_exchange_and_first_copy": statistics.mean(c_["ms_exchange"] for c_ in fstage),
                       "ms_size_exchange": statistics.mean(c_["ms_sizes"] for c_ in fstage),
                       "ms_first_pull": statistics.mean(c_["ms_pull"] for c_ in fstage),
                       "first_pull_GBs": (fstage[-1]["bytes_received"] / max(1, F // G)) / 1e6
                                         / max(1e-6, statistics.mean(c_["ms_pull"] for c_ in fstage)),
                       "ms_merge_incl_overlapped_copies": statistics.mean(c_["ms_merge"] for c_ in fstage),
                       "bytes_pulled_per_step_rank0": fstage[-1]["bytes_received"]}
        # the full-representation pipeline of Fig. 6: sub-VDIs in
        # the full representation (converted untimed), fixed-size exchange,
        # full-representation gather -- same image, the paper's A/B
        compx = vdi.Compositor(W, H, cfg.k_in, k, n, n_ranks=G, rank=rank, unique_id=new_uid(), stream=stream,
                               flags=L.VDI_FLAG_STAGE_TIMING | L.VDI_FLAG_FULL_GATHER)
        fulls = [compx.dense_to_full(p) for p in local]
        ids = [p.pe_id for p in local]

        def full_step():
            compx.composite_fullrep(fulls, ids, strip)
            compx.gather(strip, image)
        for _ in range(3):
            full_step()
        Kx = max(5, args.steps // 10)
        x_ms, x_stage, _ = timed_steps(Kx, full_step, compx)
        xm = allreduce_max(sum(x_ms), G) / Kx
        full_rep = {"ms_per_vdi": xm, "value": 1e3 / xm, "steps": Kx,
                    "stages_ms": {s_: statistics.mean(c_[f"ms_{s_}"] for c_ in x_stage)
                                  for s_ in ("exchange", "merge", "gather")},
                    "exchange_bytes_sent_rank0": x_stage[-1]["bytes_sent"],
                    "note": "sub-VDIs in the full representation: fixed-size exchange, compositing from full "
                            "slices, full-representation gather (Fig. 6 'full'); latency mode"}
        compx.close()
        del fulls
    else:
        stage = fstage
        frames_info = None
        full_rep = None

    # ---- rooflines, per rank.  The dominant HBM-bound kernel is
    # merge_fast: it reads the counts, the group bases and the records of the
    # pass-through lists and writes the whole full representation.
    P_g = strip.count.numel()
    ng = (P_g + 31) // 32
    rec = stage[-1]["records_in"]
    rec_s = stage[-1]["records_search"]
    B_merge = 24 * rec + n * P_g + P_g * (24 * k + 1)  # SURVEY §8(d) algorithmic bytes of the merge stage
    B_fast = n * P_g + 4 * n * ng + 24 * (rec - rec_s) + P_g * (24 * k + 1)
    ms_merge = statistics.mean(c["ms_merge"] for c in stage)
    ms_fast = statistics.mean(c["ms_fast"] for c in stage)
    ms_merge_max = allreduce_max(ms_merge, G)
    achieved = B_fast / (ms_fast * 1e-3) / 1e9
    peak, peak_src = _peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "merge_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(cfg.name)
        except Exception:
            traffic = None
    ms_ex = statistics.mean(c["ms_exchange"] for c in stage)
    ms_ga = statistics.mean(c["ms_gather"] for c in stage)
    bytes_sent = stage[-1]["bytes_sent"]
    bytes_recv = stage[-1]["bytes_received"]

    # ---- Phase 1 + Phase 2 of one VDI: every local PE's
    # sub-VDI raycast from the resident volume (vdi_generate_subvdi), then the
    # strip-mode exchange + merge + gather; CUDA events on the stream, min over
    # 3 repetitions, max over ranks; deterministic, so `local` is regenerated
    # in place with identical contents
    v2r = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        torch.cuda.synchronize()
        barrier(G)
        ev0.record(stream)
        regen = [comp.generate_subvdi(vol, tft, cam, dec, pe) for pe in local_ids]
        strip_step()
        ev1.record(stream)
        torch.cuda.synchronize()
        v2r.append(ev0.elapsed_time(ev1))
    assert [p.total for p in regen] == [p.total for p in local]
    ms_v2r = allreduce_max(min(v2r), G)
    volume_to_root = {"ms": ms_v2r, "vdis_per_s": 1e3 / ms_v2r, "pes_generated_per_rank": len(local_ids),
                      "note": "Phase 1 (vdi_generate_subvdi of every local PE: gamma search + count pass, scan, "
                              "write pass; PAPER.md:113-118, :150-157) + strip-mode exchange, merge and gather of "
                              "one VDI (PAPER.md:164-185), one stream, max over ranks"}

    # ---- end to end through the C ABI with host buffers (pinned): host
    # sub-VDIs in, the composited strip back in the dense representation
    # (vdi_composite_host_dense)
    e2e = None
    if not args.no_e2e:
        # the local sub-VDIs packed in one pinned host arena (256-B aligned
        # arrays): libvdi then moves a frame's inputs with one H2D copy
        parts = [[p.count] + ([p.offset] if G > 1 else []) + [p.depth, p.rgba] for p in local]
        sizes = [[(t.numel() * t.element_size() + 255) // 256 * 256 for t in ts] for ts in parts]
        arena = torch.empty(sum(map(sum, sizes)), dtype=torch.uint8).pin_memory()
        host_pes, off = [], 0
        for p, ts, ss in zip(local, parts, sizes):
            hv = []
            for t, sz in zip(ts, ss):
                nb = t.numel() * t.element_size()
                h = arena[off:off + nb].view(t.dtype).view(t.shape)
                h.copy_(t)
                hv.append(h)
                off += sz
            host_pes.append(vdi.DenseSubVDI(p.pe_id, p.total, hv[0], hv[1] if G > 1 else None, hv[-2], hv[-1]))
        P_g = strip.count.numel()
        cap = max(1, min(P_g * k, S_total))  # a list never gains supersegments: output <= input records
        outs = [(torch.empty(P_g, dtype=torch.uint8).pin_memory(), torch.empty((cap, 2), dtype=torch.float32).pin_memory(),
                 torch.empty((cap, 4), dtype=torch.float32).pin_memory()) for _ in range(2)]
        # warm-up: the single-frame call once, then the pipelined call (its
        # first call allocates the second input slot and the output slots)
        T_one = comp.composite_host_dense(host_pes, *outs[0])
        comp.composite_host_dense_frames([host_pes] * 2, outs)
        barrier(G)
        t0 = time.perf_counter()
        # every step = one frame: its sub-VDIs host->device, compositing, its
        # dense result device->host; consecutive frames overlap (copy engines
        # in both directions beside the SMs)
        Ts = comp.composite_host_dense_frames([host_pes] * args.e2e_steps, [outs[f & 1] for f in range(args.e2e_steps)])
        dt = allreduce_max(time.perf_counter() - t0, G)
        assert all(t == T_one for t in Ts), (Ts, T_one)
        T_out = T_one
        P_full = W * H
        h2d = sum(P_full + 24 * p.total + (4 * (P_full + 1) if G > 1 else 0) for p in host_pes)
        d2h = P_g + 24 * T_out
        e2e = {"value": args.e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(allreduce_sum(h2d, G)),
               "d2h_bytes_per_step": int(allreduce_sum(d2h, G)),
               "frames": args.e2e_steps,
               "host_link_GBs": (h2d + d2h) * args.e2e_steps / dt / 1e9,  # this rank's H2D + D2H bytes / time
               "note": "vdi_composite_host_dense_frames: per frame, pinned host sub-VDIs -> H2D -> composite "
                       "(strip mode) -> on-device compaction -> counts + packed supersegments D2H, every rank; "
                       "frame f's H2D overlaps frame f-1's compositing and frame f-2's D2H"}

    # ---- CPU oracle baseline (rank 0, N = 1 only) + a parity spot check
    cpu = None
    parity = None
    if rank == 0 and G == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        volh = host_volume(vol)
        pes_o, pix = oracle_band_inputs(cfg, volh, tf, cam, dec, args.cpu_rows, threads)
        out, t = oracle_composite_band(cfg, pes_o, pix, threads)
        frac = len(pix) / (W * H)
        sample = (f"rows [{pix[0] // W}, {pix[-1] // W + 1}) of {H} ({len(pix)} lists, {frac:.4f} of the image), "
                  f"oracle-generated inputs")
        cpu = {"value": frac / t, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
               "seconds": t}
        gc = strip.count[pix].cpu().numpy()
        gd = strip.depth[pix].cpu().numpy()
        gr = strip.rgba[pix].cpu().numpy()
        oc, od, orr = out["count"][pix], out["depth"][pix], out["rgba"][pix]
        tie = out["stats"]["margin"][pix] < 1e-6
        ok = ~tie
        parity = {"lists": int(len(pix)), "ties": int(tie.sum()),
                  "count_mismatch": int((gc[ok] != oc[ok]).sum()),
                  "max_rgba_err": float(np.abs(gr[ok] - orr[ok]).max()),
                  "max_depth_rel_err": float((np.abs(gd[ok] - od[ok]) / np.maximum(np.abs(od[ok]), 1e-30)).max())}

    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg, args.view), "n_pes": n, "image": f"{W}x{H}",
                       "k_in": cfg.k_in, "k_out": k, "supersegments_total": S_total,
                       "parallelism": (f"{F} VDIs per step, frame f composited whole on rank f mod {G} from all "
                                       f"ranks' PEs (frames mode)" if G > 1 else
                                       "one GPU: every PE homed on it, one VDI per step"),
                       "frames_per_step": F,
                       "l2": f"flushed between steps ({args.flush_mb} MiB memset, untimed)",
                       "inputs": "sub-VDIs raycast by vdi_generate_subvdi (untimed), resident in HBM",
                       "gen_seconds": round(t_gen, 2)},
            "roofline": {"kernel": "merge_fast (pass-through lists + full-representation write, TMA bulk stores)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes": int(B_fast), "ms": ms_fast,
                         "merge_stage": {"algorithmic_bytes": int(B_merge), "ms": ms_merge,
                                         "achieved_GBs": B_merge / (ms_merge * 1e-3) / 1e9,
                                         "frac": B_merge / (ms_merge * 1e-3) / 1e9 / peak,
                                         "ms_max_over_ranks": ms_merge_max}},
            "stages_ms": {"exchange": ms_ex, "merge": ms_merge, "gather": ms_ga,
                          "merge_scan": statistics.mean(c["ms_scan"] for c in stage),
                          "merge_fast": statistics.mean(c["ms_fast"] for c in stage),
                          "merge_search": statistics.mean(c["ms_search"] for c in stage)},
            "phase1_generate": phase1,
            "volume_to_root_vdi": volume_to_root,
            "latency_mode": latency,
            "frames_mode": frames_info,
            "full_representation_mode": full_rep,
            "supersegments_merged_per_s": S_total * F / (ms_per_step * 1e-3),
            "searched_lists": stage[-1]["searched_lists"],
            "search_buckets": stage[-1]["bucket_lists"], "fast_fallback_groups": stage[-1]["fallback_groups"],
            "exchange_bytes_sent_rank0": bytes_sent, "exchange_bytes_received_rank0": bytes_recv,
            "gather": "full representation (PAPER.md:185)" if args.full_gather else "dense + root inflate (f1)",
            "exchange": ("NCCL send/recv" if args.nccl_exchange else
                         "peer reads: merge kernels load peers' sub-VDIs over NVLink (CUDA IPC)" if args.peer_reads else
                         "peer copies: copy engines pull peers' strip slices over NVLink (CUDA IPC)" if args.ce_copies else
                         "peer copies: one SM kernel pulls peers' strip slices over NVLink (CUDA IPC)"),
            "gather_bytes_into_root": stage[-1]["bytes_gather"],
            "nvlink_roofline": None if G == 1 else {
                "peak_GBs_per_direction": 900.0, "peak_source": "NVLink 5 nominal per GPU per direction",
                "strip_exchange_GBs_rank0": bytes_recv / max(ms_ex, 1e-6) / 1e6,
                "strip_exchange_frac": bytes_recv / max(ms_ex, 1e-6) / 1e6 / 900.0,
                "strip_exchange_note": "peer slices pulled into rank 0 / (size exchange + host sync + pull) time",
                "gather_into_root_GBs": stage[-1]["bytes_gather"] / max(ms_ga, 1e-6) / 1e6,
                "gather_into_root_frac": stage[-1]["bytes_gather"] / max(ms_ga, 1e-6) / 1e6 / 900.0,
                "gather_note": "dense bytes into the root / gather stage time (includes compaction, host sync and "
                               "the root's 1 GB inflate)",
                "frames_first_pull_GBs": frames_info["first_pull_GBs"] if frames_info else None,
                "frames_first_pull_frac": frames_info["first_pull_GBs"] / 900.0 if frames_info else None},
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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--e2e-steps", type=int, default=24)
    ap.add_argument("--cpu-rows", type=int, default=12)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--full-gather", action="store_true", help="gather the full representation (PAPER.md:185)")
    ap.add_argument("--nccl-exchange", action="store_true", help="NCCL send/recv exchange instead of peer copies")
    ap.add_argument("--peer-reads", action="store_true", help="merge kernels read peers' slices over NVLink")
    ap.add_argument("--frames", type=int, default=0,
                    help="G > 1: VDIs per step in frames mode (default 4G; frame f composited whole on rank f mod G)")
    ap.add_argument("--ce-copies", action="store_true", help="exchange copies on the copy engines, not the SM copy kernel")
    ap.add_argument("--chunks", type=int, default=1, help="frames mode: row chunks per frame (copy/merge overlap)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
