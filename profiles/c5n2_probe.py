import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2206_14503_b200 as vdi, synth
cfg = synth.config_by_name("C5", n_pes=2)
comp = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes, flags=vdi._lib.VDI_FLAG_STAGE_TIMING)
vol = synth.make_volume(cfg, device="cuda")
tf = torch.from_numpy(synth.tf_table(cfg.tf, cfg.tf_scale)).cuda()
cam = synth.make_camera(cfg.W, cfg.H)
dec = cfg.decomposition()
pes = [comp.generate_subvdi(vol, tf, cam, dec, pe) for pe in range(cfg.n_pes)]
torch.cuda.synchronize(); print("generated", [p.total for p in pes], flush=True)
strip = comp.empty_strip()
comp.composite(pes, strip); torch.cuda.synchronize(); print("composite ok", comp.counters()["bucket_lists"], comp.counters()["general_lists"], flush=True)
ims = [vdi.FullVDI.empty(cfg.W, 0, cfg.H, cfg.k_out) for _ in range(2)]
comp.composite_frames([pes] * 2, ims); torch.cuda.synchronize(); print("frames 2 ok", flush=True)
