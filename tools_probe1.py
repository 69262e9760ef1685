import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch, synth, paper_2206_14503_b200 as vdi
cfg = synth.config_by_name("C3")
vol = synth.make_volume(cfg, device="cuda")
tf = torch.from_numpy(synth.tf_table(cfg.tf)).cuda()
cam = synth.make_camera(cfg.W, cfg.H); dec = cfg.decomposition()
gen = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes)
pes = [gen.generate_subvdi(vol, tf, cam, dec, pe) for pe in range(cfg.n_pes)]
comp = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes, max_iters=int(sys.argv[1]))
strip = comp.empty_strip()
for _ in range(3): comp.composite(pes, strip)
torch.cuda.synchronize()
