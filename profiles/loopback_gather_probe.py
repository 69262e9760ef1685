import os, sys, threading, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2206_14503_b200 as vdi, synth
cfg = synth.config_by_name("C3"); W,H,n,k = cfg.W,cfg.H,cfg.n_pes,cfg.k_out
G = 2
key = os.urandom(128)
comps = [vdi.Compositor(W,H,cfg.k_in,k,n,n_ranks=G,rank=r,unique_id=key,flags=vdi._lib.VDI_FLAG_LOOPBACK,stream=torch.cuda.Stream()) for r in range(G)]
vol = synth.make_volume(cfg, device="cuda"); tf = torch.from_numpy(synth.tf_table(cfg.tf, cfg.tf_scale)).cuda()
gen = vdi.Compositor(W,H,cfg.k_in,k,n)
cam = synth.make_camera(W,H)
pes=[]
for pe in range(n):
    p = gen.generate_subvdi(vol, tf, cam, cfg.decomposition(), pe)
    pes.append(vdi.DenseSubVDI(p.pe_id,p.total,p.count.clone(),p.offset.clone(),p.depth.clone(),p.rgba.clone()))
strips=[c.empty_strip() for c in comps]; image=vdi.FullVDI.empty(W,0,H,k)
torch.cuda.synchronize()
def rank(r):
    mine=[p for p in pes if vdi.pe_home(n,G,p.pe_id)==r]
    for _ in range(4):
        comps[r].composite(mine, strips[r]); comps[r].gather(strips[r], image if r==0 else None)
th=[threading.Thread(target=rank,args=(r,)) for r in range(G)]
[t.start() for t in th]; [t.join() for t in th]
torch.cuda.synchronize(); print("done")
