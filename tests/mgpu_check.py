"""Multi-GPU parity check, run under torchrun (one process per GPU):

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_check.py [--config synthetic|C1|C3]

Every rank builds the same seeded inputs (neutral synth/ generators), keeps
the PEs homed on it (PAPER.md:218 block placement), composites its strip
through vdi_composite (NCCL size exchange + all-to-allv) and
gathers to rank 0 (vdi_gather).  Rank 0 checks the gathered
image bit-for-bit against a 1-GPU composite of the same inputs (the result
must not depend on G) and against the CPU oracle on sampled lists.
Prints one JSON line on rank 0; exit code 0 iff all checks pass."""
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


def main():
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
    obj = [vdi.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)

    if args.config == "synthetic":
        W, H, n, k_in, k_out = args.W, args.H, args.n, args.k, args.k
        pes_np = synth.random_subvdis(n, W, H, k_in, lam=args.lam, seed=31)
        comp = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=obj[0])
        local_pes = [dense_to_device(pes_np[pe], pe) for pe in range(n) if vdi.pe_home(n, world, pe) == rank]
    else:
        cfg = synth.config_by_name(args.config)
        W, H, n, k_in, k_out = cfg.W, cfg.H, cfg.n_pes, cfg.k_in, cfg.k_out
        comp = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=obj[0])
        vol = synth.make_volume(cfg, device="cuda")
        tf = torch.from_numpy(synth.tf_table(cfg.tf, cfg.tf_scale)).cuda()
        cam = synth.make_camera(W, H)
        dec = cfg.decomposition()
        local_pes = [comp.generate_subvdi(vol, tf, cam, dec, pe) for pe in range(n)
                     if vdi.pe_home(n, world, pe) == rank]
        pes_np = None

    strip = comp.empty_strip()
    image = vdi.FullVDI.empty(W, 0, H, k_out) if rank == 0 else None
    comp.composite(local_pes, strip)   # default: peer (NVLink, CUDA IPC) exchange + dense gather
    comp.gather(strip, image)
    comp.composite(local_pes, strip)   # twice: the IPC mappings are cached
    comp.gather(strip, image)
    cnt = comp.counters()
    # the NCCL exchange and the paper's full-representation gather
    # must give the same image
    variants = {}
    for name, fl in (("full_gather", vdi._lib.VDI_FLAG_FULL_GATHER),
                     ("nccl_exchange", vdi._lib.VDI_FLAG_NCCL_EXCHANGE),
                     ("peer_reads", vdi._lib.VDI_FLAG_PEER_READS),
                     ("ce_copies", vdi._lib.VDI_FLAG_CE_COPIES)):
        u = [vdi.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(u, src=0)
        c2 = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=u[0], flags=fl)
        im2 = vdi.FullVDI.empty(W, 0, H, k_out) if rank == 0 else None
        st2 = c2.empty_strip()
        c2.composite(local_pes, st2)
        c2.gather(st2, im2)
        torch.cuda.synchronize()
        variants[name] = im2
        c2.close()
    # compositing in the full representation (Fig. 6 "full"):
    # fixed-size exchange of full-representation slices + full gather
    u = [vdi.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(u, src=0)
    c2 = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=u[0],
                        flags=vdi._lib.VDI_FLAG_FULL_GATHER)
    fulls = [c2.dense_to_full(p) for p in local_pes]
    st2 = c2.empty_strip()
    im2 = vdi.FullVDI.empty(W, 0, H, k_out) if rank == 0 else None
    c2.composite_fullrep(fulls, [p.pe_id for p in local_pes], st2)
    c2.gather(st2, im2)
    torch.cuda.synchronize()
    variants["fullrep_exchange"] = im2
    c2.close()
    # the gather onto another root (frames in flight are gathered round-robin,
    # Q14): dense and full-representation gathers onto the last and a middle
    # rank; the root ships its image to rank 0 for the comparison
    for R in sorted({world - 1, world // 2}):
        for name, fl in (("dense", 0), ("full", vdi._lib.VDI_FLAG_FULL_GATHER)):
            u = [vdi.get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(u, src=0)
            c2 = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=u[0], flags=fl, root=R)
            st2 = c2.empty_strip()
            im2 = vdi.FullVDI.empty(W, 0, H, k_out) if rank in (R, 0) else None
            c2.composite(local_pes, st2)
            c2.gather(st2, im2 if rank == R else None)
            torch.cuda.synchronize()
            if R != 0:
                for t_ in (im2.count, im2.depth, im2.rgba) if rank in (R, 0) else ():
                    (dist.send if rank == R else dist.recv)(t_, R if rank == 0 else 0)
            torch.cuda.synchronize()
            variants[f"root{R}_{name}"] = im2
            c2.close()
    # frames in flight (vdi_composite_frames): frame f composited whole on rank
    # f mod G from every rank's PEs; each owner checks its frames bit for bit
    # against a 1-GPU composite of the same frame (synthetic inputs only: every
    # rank can rebuild every frame from its seed)
    frames_ok = None
    if args.config == "synthetic":
        F = 2 * world
        fr_np = [synth.random_subvdis(n, W, H, k_in, lam=args.lam + f, seed=700 + f) for f in range(F)]
        u = [vdi.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(u, src=0)
        cf = vdi.Compositor(W, H, k_in, k_out, n, n_ranks=world, rank=rank, unique_id=u[0])
        fl = [[dense_to_device(fr_np[f][pe], pe) for pe in range(n) if vdi.pe_home(n, world, pe) == rank]
              for f in range(F)]
        ims = [vdi.FullVDI.empty(W, 0, H, k_out) if f % world == rank else None for f in range(F)]
        for chunks in (1, 3):
            cf.composite_frames(fl, ims, chunks=chunks)
            torch.cuda.synchronize()
            one = vdi.Compositor(W, H, k_in, k_out, n)
            for f in range(rank, F, world):
                ref1 = one.empty_strip()
                one.composite([dense_to_device(p, i) for i, p in enumerate(fr_np[f])], ref1)
                torch.cuda.synchronize()
                same = all(torch.equal(a, b) for a, b in ((ims[f].count, ref1.count), (ims[f].depth, ref1.depth),
                                                          (ims[f].rgba, ref1.rgba)))
                frames_ok = same if frames_ok is None else (frames_ok and same)
            one.close()
        fc = cf.counters()
        t2 = torch.tensor([fc["bytes_sent"], fc["bytes_received"], 0 if frames_ok else 1], dtype=torch.float64,
                          device="cuda")
        dist.all_reduce(t2)
        frames_ok = int(t2[2]) == 0 and int(t2[0]) == int(t2[1])
        cf.close()
    torch.cuda.synchronize()
    ok = True
    if frames_ok is not None:
        ok &= frames_ok
    res = {"world": world, "frames_identical_to_1gpu": frames_ok, "config": args.config, "bytes_sent_rank": cnt["bytes_sent"],
           "bytes_received_rank": cnt["bytes_received"]}
    # byte conservation over ranks
    t = torch.tensor([cnt["bytes_sent"], cnt["bytes_received"]], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    res["sent_total"], res["received_total"] = int(t[0]), int(t[1])
    ok &= int(t[0]) == int(t[1])

    # single-GPU reference composite on rank 0 (all PEs, G = 1)
    if args.config != "synthetic":
        # every rank regenerates all PEs so rank 0 can run the G = 1 composite
        allp = [comp.generate_subvdi(vol, tf, cam, dec, pe) for pe in range(n)] if rank == 0 else []
    dist.barrier()
    if rank == 0:
        one = vdi.Compositor(W, H, k_in, k_out, n)
        if args.config == "synthetic":
            allp = [dense_to_device(p, i) for i, p in enumerate(pes_np)]
        ref = one.empty_strip()
        one.composite(allp, ref)
        torch.cuda.synchronize()
        same = all(torch.equal(a, b) for a, b in ((image.count, ref.count), (image.depth, ref.depth),
                                                     (image.rgba, ref.rgba)))
        res["bit_identical_to_1gpu"] = bool(same)
        ok &= same
        for name, im2 in variants.items():
            s2 = all(torch.equal(a, b) for a, b in ((im2.count, ref.count), (im2.depth, ref.depth),
                                                      (im2.rgba, ref.rgba)))
            res[name + "_identical"] = bool(s2)
            ok &= s2
        res["gather_bytes_dense"] = cnt["bytes_gather"]
        if pes_np is not None:
            import oracle
            rng = np.random.default_rng(3)
            pix = np.unique(rng.choice(W * H, min(6000, W * H), replace=False))
            o = oracle.composite_pixels(pes_np, pix, k_out)
            gc, gd, gr = image.count.cpu().numpy(), image.depth.cpu().numpy(), image.rgba.cpu().numpy()
            nl, ties = compare(gc[pix], gd[pix], gr[pix], o["count"], o["depth"], o["rgba"], o["stats"]["margin"],
                               "mgpu")
            res["oracle_lists_checked"] = nl
            res["oracle_ties"] = len(ties)
        print(json.dumps(res), flush=True)
    dist.barrier()
    comp.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
