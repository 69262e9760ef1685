"""Multi-GPU timeline of vdi_composite_frames (VDI_TRACE events per rank:
push, receive wait, merge kernels, gather send / receive + inflate).
torchrun --nproc-per-node G profiles/trace_probe_mgpu.py [C3] [F] [rot]"""
import os
import sys

os.environ["VDI_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2206_14503_b200 as vdi  # noqa: E402
import synth  # noqa: E402

world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = synth.config_by_name(sys.argv[1] if len(sys.argv) > 1 else "C3")
F = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rot = len(sys.argv) > 3 and sys.argv[3] == "rot"
u = [vdi.get_unique_id() if rank == 0 else None]
dist.broadcast_object_list(u, src=0)
comp = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes, n_ranks=world, rank=rank, unique_id=u[0])
vol = synth.make_volume(cfg, device="cuda")
tf = torch.from_numpy(synth.tf_table(cfg.tf, cfg.tf_scale)).cuda()
cam = synth.make_camera(cfg.W, cfg.H)
ids = [pe for pe in range(cfg.n_pes) if vdi.pe_home(cfg.n_pes, world, pe) == rank]
ps = [comp.generate_subvdi(vol, tf, cam, cfg.decomposition(), pe) for pe in ids]
pes = [vdi.DenseSubVDI(p.pe_id, p.total, p.count.clone(), p.offset.clone(), p.depth.clone(), p.rgba.clone()) for p in ps]
roots = [f % world if rot else 0 for f in range(F)]
image = vdi.FullVDI.empty(cfg.W, 0, cfg.H, cfg.k_out)
ims = [image if r == rank else None for r in roots]
torch.cuda.synchronize()
for it in range(4):
    dist.barrier()
    print(f"--- rank {rank} call {it}", file=sys.stderr, flush=True)
    comp.composite_frames([pes] * F, ims, roots=roots)
    torch.cuda.synchronize()
dist.barrier()
dist.destroy_process_group()
