import sys, os, json, statistics
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch, numpy as np
import synth, paper_2206_14503_b200 as vdi
from paper_2206_14503_b200 import _lib as L
cfg = synth.config_by_name("C3")
vol = synth.make_volume(cfg, device="cuda")
tf = torch.from_numpy(synth.tf_table(cfg.tf)).cuda()
cam = synth.make_camera(cfg.W, cfg.H)
dec = cfg.decomposition()
gen = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes)
pes = [gen.generate_subvdi(vol, tf, cam, dec, pe) for pe in range(cfg.n_pes)]
out = {}
for iters in (16, 4, 1):
    comp = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes, max_iters=iters,
                          flags=L.VDI_FLAG_STAGE_TIMING | L.VDI_FLAG_PIXEL_STATS)
    strip = comp.empty_strip()
    ts = []
    for r in range(8):
        comp.composite(pes, strip)
        c = comp.counters()
        ts.append((c["ms_fast"], c["ms_search"]))
    out[iters] = [statistics.median(x) for x in zip(*ts)]
    if iters == 16:
        g, m = comp.pixel_stats()
        m = m.cpu().numpy().astype(np.int64)
        srch = m[m > cfg.k_out]
        out["m_hist"] = np.bincount(np.minimum(srch, 100), minlength=101)[20:].tolist()
        out["m_mean"] = float(srch.mean()); out["n_search"] = int(len(srch))
out.pop("m_hist", None); print(json.dumps(out))
