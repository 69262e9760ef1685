"""Multi-GPU parity check, run under torchrun (one process per GPU):

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_check.py [--config synthetic|C1|C3]

Every rank builds the same seeded inputs (neutral synth/ generators), keeps
the PEs homed on it (PAPER.md:218 block placement), composites its strip
through vdi_composite (device-driven push of the strip slices into the
owners' windows over NVLink) and gathers to the root
(vdi_gather / vdi_gather_root).  Rank 0 checks every gathered
image bit-for-bit against a 1-GPU composite of the same inputs (the result
must not depend on G) and against the CPU oracle on sampled lists; exchange
bytes are checked for conservation (sum sent == sum received).  Also: the
full-representation exchange (vdi_composite_fullrep), a pipelined sequence
of frames with a rotating root (no host synchronisation between frames), and
the host entry point vdi_composite_host_dense_frames at n_ranks > 1 over
three distinct input sets (both input slots reused; per-array and one-span
uploads).  Prints one JSON line on rank 0; exit code 0 iff all checks pass."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2206_14503_b200 as vdi  # noqa: E402
import synth  # noqa: E402
from parity import compare, dense_to_device  # noqa: E402


def uid(rank):
    u = [vdi.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(u, src=0)
    return u[0]


def to_rank0(im, R, rank):
    """The root's image, shipped to rank 0 for the comparison (torch.distributed; test only)."""
    if R == 0:
        return im
    if rank == 0:
        W_, k_ = im_shape
        im = vdi.FullVDI.empty(W_, 0, H_, k_)
    if rank in (0, R):
        for t in (im.count, im.depth, im.rgba):
            (dist.send if rank == R else dist.recv)(t, R if rank == 0 else 0)
    return im if rank == 0 else None


def equal(a, b):
    return all(torch.equal(x, y) for x, y in ((a.count, b.count), (a.depth, b.depth), (a.rgba, b.rgba)))


def main():
    global im_shape, H_
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="synthetic")
    ap.add_argument("--W", type=int, default=640)
    ap.add_argument("--H", type=int, default=360)
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--k", type=int, default=12)
    ap.add_argument("--lam", type=float, default=9.0)
    args = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = vdi._lib
    flags = L.VDI_FLAG_STAGE_TIMING

    if args.config == "synthetic":
        W, H, n, k_in, k_out = args.W, args.H, args.n, args.k, args.k
        sets_np = [synth.random_subvdis(n, W, H, k_in, lam=args.lam + s, seed=31 + s) for s in range(3)]
        comp = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=uid(rank), flags=flags)
        sets = [[dense_to_device(p[pe], pe) for pe in range(n)] for p in sets_np]
    else:
        cfg = synth.config_by_name(args.config)
        W, H, n, k_in, k_out = cfg.W, cfg.H, cfg.n_pes, cfg.k_in, cfg.k_out
        comp = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=uid(rank), flags=flags)
        vol = synth.make_volume(cfg, device="cuda")
        tf = torch.from_numpy(synth.tf_table(cfg.tf, cfg.tf_scale)).cuda()
        dec = cfg.decomposition()
        gen = vdi.Compositor(W, H, k_in, k_out, n)
        sets, sets_np = [], None
        for v in range(2):  # views V0 / V1
            cam = synth.make_camera(W, H, view=v)
            ps = [gen.generate_subvdi(vol, tf, cam, dec, pe) for pe in range(n)]
            sets.append([vdi.DenseSubVDI(p.pe_id, p.total, p.count.clone(), p.offset.clone(), p.depth.clone(),
                                         p.rgba.clone()) for p in ps])
    im_shape, H_ = (W, k_out), H
    mine = lambda s: [p for p in s if vdi.pe_home(n, world, p.pe_id) == rank]

    # 1-GPU references (every rank computes them; rank 0 compares)
    one = vdi.Compositor(W, H, k_in, k_out, n)
    refs = []
    for s in sets:
        r_ = one.empty_strip()
        one.composite(s, r_)
        refs.append(r_)
    torch.cuda.synchronize()
    res = {"world": world, "W": W, "H": H, "n": n, "k": k_out}
    ok = True

    # (1) strips + dense gather to rank 0, twice
    strip = comp.empty_strip()
    image = vdi.FullVDI.empty(W, 0, H, k_out) if rank == 0 else None
    for _ in range(2):
        comp.composite(mine(sets[0]), strip)
        comp.gather(strip, image)
    cnt = comp.counters()
    torch.cuda.synchronize()
    t = torch.tensor([cnt["bytes_sent"], cnt["bytes_received"]], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    res["bytes_sent"], res["bytes_received"] = int(t[0]), int(t[1])
    ok &= res["bytes_sent"] == res["bytes_received"] and res["bytes_sent"] > 0
    if rank == 0:
        res["strip_gather_equal"] = equal(image, refs[0])
        ok &= res["strip_gather_equal"]

    # (2) full-representation exchange (Fig. 6 "full")
    c2 = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=uid(rank))
    fulls = [c2.dense_to_full(p) for p in mine(sets[0])]
    st2 = c2.empty_strip()
    im2 = vdi.FullVDI.empty(W, 0, H, k_out) if rank == 0 else None
    c2.composite_fullrep(fulls, [p.pe_id for p in mine(sets[0])], st2)
    c2.gather(st2, im2)
    torch.cuda.synchronize()
    if rank == 0:
        res["fullrep_equal"] = equal(im2, refs[0])
        ok &= res["fullrep_equal"]
    c2.close()
    del fulls

    # (3) pipelined frames with a rotating root: vdi_gather_root calls
    # enqueued back to back, then vdi_composite_frames (frames in flight, one
    # root and a rotating root)
    F = 2 * world + 1
    roots = [f % world for f in range(F)]
    for mode in ("calls", "frames_root0", "frames_rotating"):
        rts = [0] * F if mode == "frames_root0" else roots
        ims = [vdi.FullVDI.empty(W, 0, H, k_out) if rank == rts[f] else None for f in range(F)]
        if mode == "calls":
            strips = [comp.empty_strip() for _ in range(F)]
            for f in range(F):
                comp.composite(mine(sets[f % len(sets)]), strips[f])
                comp.gather(strips[f], ims[f], root=rts[f])
        else:
            comp.composite_frames([mine(sets[f % len(sets)]) for f in range(F)], ims, roots=rts)
        torch.cuda.synchronize()
        eq = []
        for f in range(F):
            im0 = to_rank0(ims[f], rts[f], rank)
            torch.cuda.synchronize()
            if rank == 0:
                eq.append(equal(im0, refs[f % len(sets)]))
        if rank == 0:
            res[f"{mode}_equal"] = eq
            ok &= all(eq)

    # (4) host entry points at n_ranks > 1: 3 distinct input sets (2 for C*),
    # order reusing both slots, per-array and one-span uploads
    order = [0, 1, len(sets) - 1, 1, 0]
    for span in (False, True):
        c3 = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=uid(rank),
                            flags=L.VDI_FLAG_HOST_SPAN if span else 0)
        frames, keep = [], []
        for i in order:
            hs = [p.to("cpu") for p in mine(sets[i])]
            if span:
                parts = [[h.count, h.depth, h.rgba] for h in hs]
                sizes = [[(x.numel() * x.element_size() + 255) // 256 * 256 for x in ts] for ts in parts]
                arena = torch.empty(max(1, sum(map(sum, sizes))), dtype=torch.uint8).pin_memory()
                pk, off = [], 0
                for h, ts, ss in zip(hs, parts, sizes):
                    hv = []
                    for x, sz in zip(ts, ss):
                        nb = x.numel() * x.element_size()
                        v = arena[off:off + nb].view(x.dtype).view(x.shape)
                        v.copy_(x)
                        hv.append(v)
                        off += sz
                    pk.append(vdi.DenseSubVDI(h.pe_id, h.total, hv[0], None, hv[1], hv[2]))
                frames.append(pk)
                keep.append(arena)
            else:
                frames.append([h.to("cpu", pin=True) for h in hs])
        P = (c3.row_end - c3.row_begin) * W
        outs = [(torch.empty(P, dtype=torch.uint8), torch.empty((P * k_out, 2), dtype=torch.float32),
                 torch.empty((P * k_out, 4), dtype=torch.float32)) for _ in order]
        Ts = c3.composite_host_dense_frames(frames, outs)
        good = True
        a, b = c3.row_begin * W, c3.row_end * W
        for f, i in enumerate(order):
            fc = refs[i].count[a:b].cpu().numpy()
            sel = np.arange(k_out)[None, :] < fc[:, None].astype(np.int64)
            good &= Ts[f] == int(sel.sum()) and np.array_equal(outs[f][0].numpy(), fc)
            good &= np.array_equal(outs[f][1].numpy()[:Ts[f]], refs[i].depth[a:b].cpu().numpy()[sel])
            good &= np.array_equal(outs[f][2].numpy()[:Ts[f]], refs[i].rgba[a:b].cpu().numpy()[sel])
        g = torch.tensor([1 if good else 0], device="cuda")
        dist.all_reduce(g, op=dist.ReduceOp.MIN)
        res[f"host_dense_frames_{'span' if span else 'arrays'}_equal"] = bool(g.item())
        ok &= bool(g.item())
        c3.close()

    # (5) oracle on sampled lists (synthetic inputs only: the oracle needs host inputs)
    if rank == 0 and sets_np is not None:
        import oracle
        rng = np.random.default_rng(3)
        pix = np.unique(rng.choice(W * H, 3000, replace=False))
        o = oracle.composite_pixels(sets_np[0], pix, k_out)
        nl, ties = compare(image.count.cpu().numpy()[pix], image.depth.cpu().numpy()[pix],
                           image.rgba.cpu().numpy()[pix], o["count"], o["depth"], o["rgba"],
                           o["stats"]["margin"], "mgpu")
        res["oracle_lists"] = nl
        res["oracle_ties"] = len(ties)
    res["ms_exchange"], res["ms_merge"], res["ms_gather"] = cnt["ms_exchange"], cnt["ms_merge"], cnt["ms_gather"]
    res["ok"] = bool(ok)
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps(res), flush=True)
    comp.close()
    dist.destroy_process_group()
    sys.exit(0 if okt.item() == 1 else 1)


if __name__ == "__main__":
    main()
