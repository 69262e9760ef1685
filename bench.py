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
    F = args.frames if args.frames > 0 else G  # frames in flight per step
    flags = (L.VDI_FLAG_STAGE_TIMING | (L.VDI_FLAG_FULL_GATHER if args.full_gather else 0)
             | (L.VDI_FLAG_NCCL_EXCHANGE if args.nccl_exchange else 0)
             | (L.VDI_FLAG_PEER_READS if args.peer_reads else 0))
    main_stream = torch.cuda.current_stream()
    # one libvdi context per frame in flight, each on its own stream with its
    # own communicator; frame f is gathered onto rank f mod G (Q14)
    comps = []
    for f in range(F):
        uid = None
        if G > 1:
            import torch.distributed as dist
            obj = [vdi.get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        st = main_stream if F == 1 else torch.cuda.Stream()
        comps.append(vdi.Compositor(W, H, cfg.k_in, k, n, n_ranks=G, rank=rank, flags=flags, unique_id=uid,
                                    stream=st, root=f % G))
    comp = comps[0]
    stream = comp.stream

    # ---- inputs (untimed): synthetic volume -> per-PE dense sub-VDIs in HBM,
    # one private copy per frame context (same view: every frame is the C3 VDI)
    t0 = time.time()
    vol = synth.make_volume(cfg, device="cuda")
    tf = synth.tf_table(cfg.tf, cfg.tf_scale)
    tft = torch.from_numpy(tf).cuda()
    cam = synth.make_camera(W, H, view=args.view)
    dec = cfg.decomposition()
    torch.cuda.synchronize()  # the frame streams read the volume
    local_ids = [pe for pe in range(n) if vdi.pe_home(n, G, pe) == rank]
    locals_ = []
    for c in comps:
        with torch.cuda.stream(c.stream):
            locals_.append([c.generate_subvdi(vol, tft, cam, dec, pe) for pe in local_ids])
    torch.cuda.synchronize()
    local = locals_[0]
    t_gen = time.time() - t0
    S_local = sum(p.total for p in local)
    S_total = int(allreduce_sum(S_local, G))

    strips, images = [], []
    for c in comps:
        if G > 1 and rank == c.root:  # the root's strip aliases its rows of the image (no copy in the gather)
            image = vdi.FullVDI.empty(W, 0, H, k)
            a0, a1 = c.row_begin * W, c.row_end * W
            strip = vdi.FullVDI(c.row_begin, c.row_end, image.count[a0:a1], image.depth[a0:a1], image.rgba[a0:a1])
        else:
            strip = c.empty_strip()
            image = strip if G == 1 else None
        strips.append(strip)
        images.append(image)
    strip = strips[0]
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device="cuda")

    def step():
        # every composite first (host syncs only on its own frame's size
        # exchange), then every gather: frame f+1's exchange and merge overlap
        # frame f's merge and gather
        for c, lp, sp in zip(comps, locals_, strips):
            c.composite(lp, sp)
        for c, sp, im in zip(comps, strips, images):
            c.gather(sp, im)

    def timed_steps(K, fn, frames):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        done = [torch.cuda.Event() for _ in frames]
        stats, nl = [], 0
        torch.cuda.synchronize()
        barrier(G)
        for i in range(K):
            flush.zero_()
            evs[i][0].record(main_stream)
            for c in frames:
                if c.stream != main_stream:
                    c.stream.wait_event(evs[i][0])
            fn()
            for c, d in zip(frames, done):
                if c.stream != main_stream:
                    d.record(c.stream)
                    main_stream.wait_event(d)
            evs[i][1].record(main_stream)
            cs = [c.counters() for c in frames]  # syncs the frame streams; outside the events
            stats.append(cs[0])
            nl += sum(x["kernel_launches"] for x in cs)
        torch.cuda.synchronize()
        barrier(G)
        return [a.elapsed_time(b) for a, b in evs], stats, nl

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(G)

    # ---- timed region: exactly K steps of F frames, L2 flushed between steps (untimed)
    clk.mark_start()
    step_ms, stage, launches = timed_steps(args.steps, step, comps)
    clk.mark_end()
    tot_ms = allreduce_max(sum(step_ms), G)
    ms_per_step = tot_ms / args.steps
    value = F * args.steps / (tot_ms / 1e3)  # whole VDIs composited by all ranks per second

    # ---- latency mode (paper-style): one VDI per step onto rank 0
    latency = None
    if F > 1:
        def one():
            comps[0].composite(locals_[0], strips[0])
            comps[0].gather(strips[0], images[0])
        for _ in range(3):
            one()
        K1 = max(10, args.steps // 4)
        lat_ms, lat_stage, _ = timed_steps(K1, one, comps[:1])
        l_ms = allreduce_max(sum(lat_ms), G) / K1
        latency = {"ms_per_vdi": l_ms, "value": 1e3 / l_ms, "steps": K1,
                   "stages_ms": {s_: statistics.mean(c[f"ms_{s_}"] for c in lat_stage)
                                 for s_ in ("exchange", "merge", "gather")}}

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

    # ---- end to end through the C ABI with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        host_pes = [vdi.DenseSubVDI(p.pe_id, p.total, p.count.cpu().pin_memory(),
                                    p.offset.cpu().pin_memory() if G > 1 else None,
                                    p.depth.cpu().pin_memory(), p.rgba.cpu().pin_memory()) for p in local]
        hstrip = comp.empty_strip(device="cpu", pin=True)
        for _ in range(2):
            comp.composite_host(host_pes, hstrip)
        barrier(G)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            comp.composite_host(host_pes, hstrip)
        dt = allreduce_max(time.perf_counter() - t0, G)
        P_full = W * H
        h2d = sum(P_full + 24 * p.total + (4 * (P_full + 1) if G > 1 else 0) for p in host_pes)
        d2h = P_g * (1 + 24 * k)
        e2e = {"value": args.e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(allreduce_sum(h2d, G)),
               "d2h_bytes_per_step": int(allreduce_sum(d2h, G)),
               "note": "vdi_composite_host: pinned host sub-VDIs -> H2D -> composite -> strip D2H on every rank"}

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
            "scaling": "weak" if F == G else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg, args.view), "n_pes": n, "image": f"{W}x{H}",
                       "k_in": cfg.k_in, "k_out": k, "supersegments_total": S_total,
                       "parallelism": (f"image-space strips x{G} (direct send); {F} frame(s) in flight per step, "
                                       f"frame f gathered onto rank f mod {G}"),
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
            "latency_mode": latency,
            "supersegments_merged_per_s": S_total * F / (ms_per_step * 1e-3),
            "searched_lists": stage[-1]["searched_lists"],
            "search_buckets": stage[-1]["bucket_lists"], "fast_fallback_groups": stage[-1]["fallback_groups"],
            "exchange_bytes_sent_rank0": bytes_sent, "exchange_bytes_received_rank0": bytes_recv,
            "gather": "full representation (PAPER.md:185)" if args.full_gather else "dense + root inflate (f1)",
            "exchange": ("NCCL send/recv" if args.nccl_exchange else
                         "peer reads: merge kernels load peers' sub-VDIs over NVLink (CUDA IPC)" if args.peer_reads else
                         "peer copies: copy engines pull peers' strip slices over NVLink (CUDA IPC)"),
            "gather_bytes_into_root": stage[-1]["bytes_gather"],
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
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-rows", type=int, default=12)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--full-gather", action="store_true", help="gather the full representation (PAPER.md:185)")
    ap.add_argument("--nccl-exchange", action="store_true", help="NCCL send/recv exchange instead of peer copies")
    ap.add_argument("--peer-reads", action="store_true", help="merge kernels read peers' slices over NVLink")
    ap.add_argument("--frames", type=int, default=0,
                    help="frames in flight per step (default: one per GPU, frame f gathered onto rank f mod G)")
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
