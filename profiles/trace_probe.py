"""Timeline of the merge kernels of vdi_composite_frames on one GPU (VDI_TRACE
events around the pass-through and the search kernels of each VDI): shows how
far VDI f's search overlaps VDI f+1's pass-through.  python profiles/trace_probe.py [C3] [F]"""
import os
import sys

os.environ["VDI_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2206_14503_b200 as vdi  # noqa: E402
import synth  # noqa: E402

cfg = synth.config_by_name(sys.argv[1] if len(sys.argv) > 1 else "C3")
F = int(sys.argv[2]) if len(sys.argv) > 2 else 4
comp = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes)
vol = synth.make_volume(cfg, device="cuda")
tf = torch.from_numpy(synth.tf_table(cfg.tf, cfg.tf_scale)).cuda()
cam = synth.make_camera(cfg.W, cfg.H)
pes = [comp.generate_subvdi(vol, tf, cam, cfg.decomposition(), pe) for pe in range(cfg.n_pes)]
ims = [vdi.FullVDI.empty(cfg.W, 0, cfg.H, cfg.k_out) for _ in range(F)]
torch.cuda.synchronize()
for it in range(4):
    print(f"--- call {it}", file=sys.stderr, flush=True)
    comp.composite_frames([pes] * F, ims)
    torch.cuda.synchronize()
