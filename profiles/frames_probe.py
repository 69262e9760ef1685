"""Probe of the frames-in-flight strip pipeline (vdi_composite_frames) at G > 1:
ms per VDI for F = 1, 2, 4, 8, 16 frames per call, single root and rotating
root, plus each rank's one-VDI stage times.  torchrun --nproc-per-node G."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2206_14503_b200 as vdi  # noqa: E402
import synth  # noqa: E402


def main():
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.config_by_name(os.environ.get("CFG", "C3"))
    W, H, n, k = cfg.W, cfg.H, cfg.n_pes, cfg.k_out
    u = [vdi.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(u, src=0)
    L = vdi._lib
    comp = vdi.Compositor(W, H, cfg.k_in, k, n, n_ranks=world, rank=rank, unique_id=u[0], flags=L.VDI_FLAG_STAGE_TIMING)
    vol = synth.make_volume(cfg, device="cuda")
    tf = torch.from_numpy(synth.tf_table(cfg.tf, cfg.tf_scale)).cuda()
    dec = cfg.decomposition()
    cam = synth.make_camera(W, H)
    ids = [pe for pe in range(n) if vdi.pe_home(n, world, pe) == rank]
    ps = [comp.generate_subvdi(vol, tf, cam, dec, pe) for pe in ids]
    pes = [vdi.DenseSubVDI(p.pe_id, p.total, p.count.clone(), p.offset.clone(), p.depth.clone(), p.rgba.clone())
           for p in ps]
    image = vdi.FullVDI.empty(W, 0, H, k)
    st = torch.cuda.current_stream()
    res = {}
    for rot in (False, True):
        for F in (1, 2, 4, 8, 16):
            roots = [f % world if rot else 0 for f in range(F)]
            ims = [image if r == rank else None for r in roots]
            for _ in range(3):
                comp.composite_frames([pes] * F, ims, roots=roots)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 10
            e0.record(st)
            for _ in range(K):
                comp.composite_frames([pes] * F, ims, roots=roots)
            e1.record(st)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / (K * F)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[f"{'rot' if rot else 'root0'}_F{F}_ms_per_vdi"] = round(float(t), 4)
    # one VDI: stage times on every rank
    strip = comp.empty_strip()
    for _ in range(3):
        comp.composite(pes, strip)
        comp.gather(strip, image if rank == 0 else None)
    c = comp.counters()
    stages = {k_: round(c[k_], 4) for k_ in ("ms_exchange", "ms_merge", "ms_scan", "ms_fast", "ms_search", "ms_gather")}
    allst = [None] * world
    dist.all_gather_object(allst, stages)
    res["stages_per_rank"] = allst
    if rank == 0:
        print(json.dumps(res))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
