"""End-to-end parity at the full sizes of the BASELINE.json configurations,
in the bench's launch configuration: the GPU raycaster (vdi_generate_subvdi)
and the GPU composite (vdi_composite) against the oracle generator and the
oracle composite on sampled lists (the oracle computes them one by one).
Every input is the seeded synthetic scene of synth/ (DESIGN.md §4); no oracle
input comes from the CUDA path: the oracle regenerates the sampled rays from
the same volume itself."""
import os

import numpy as np
import pytest
import torch

import synth
from parity import compare

pytestmark = pytest.mark.gpu

CONFIGS = [("C2", 0), ("C3", 0), ("C4", 0), ("C5", 0), ("C5", 16), ("C5", 2)]  # C5 strong-scaling sweep: 2 to 16 PEs (m <= 64 ... 512)


@pytest.fixture(scope="module")
def vdi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2206_14503_b200 as vdi
    vdi._lib.lib()
    return vdi


def _lists_at(pe, pix, k):
    """GPU dense sub-VDI -> (count, depth [n,k,2], rgba [n,k,4]) at pixels pix."""
    cnt = pe.count.cpu().numpy()[pix].astype(np.int64)
    off = pe.offset.cpu().numpy().view(np.uint32)[pix].astype(np.int64)
    dep = pe.depth.cpu().numpy()
    rgb = pe.rgba.cpu().numpy()
    d = np.zeros((len(pix), k, 2), np.float32)
    c = np.zeros((len(pix), k, 4), np.float32)
    for i in range(len(pix)):
        d[i, :cnt[i]] = dep[off[i]:off[i] + cnt[i]]
        c[i, :cnt[i]] = rgb[off[i]:off[i] + cnt[i]]
    return cnt, d, c


@pytest.mark.parametrize("name,pes", CONFIGS, ids=[f"{c}-{p or 'default'}" for c, p in CONFIGS])
def test_end_to_end_sampled(vdi, orc, name, pes):
    cfg = synth.config_by_name(name, n_pes=pes) if pes else synth.config_by_name(name)
    W, H, n = cfg.W, cfg.H, cfg.n_pes
    vol = synth.make_volume(cfg, device="cuda")
    tf = synth.tf_table(cfg.tf, cfg.tf_scale)
    cam = synth.make_camera(W, H)
    dec = cfg.decomposition()
    comp = vdi.Compositor(W, H, cfg.k_in, cfg.k_out, n, flags=vdi._lib.VDI_FLAG_PIXEL_STATS)
    tft = torch.from_numpy(tf).cuda()
    pes = [comp.generate_subvdi(vol, tft, cam, dec, pe) for pe in range(n)]
    strip = comp.empty_strip()
    comp.composite(pes, strip)
    torch.cuda.synchronize()
    _, m = comp.pixel_stats()
    m = m.cpu().numpy().astype(np.int64)
    rng = np.random.default_rng(17)
    srch = np.nonzero(m > cfg.k_out)[0]
    busy = np.nonzero(m > 0)[0]
    pix = np.unique(np.concatenate([
        rng.choice(W * H, 1000, replace=False),
        rng.choice(busy, min(1000, len(busy)), replace=False) if len(busy) else [],
        rng.choice(srch, min(1000, len(srch)), replace=False) if len(srch) else [],
        np.argsort(m)[-20:],  # the longest lists
    ]).astype(np.int64))
    # the oracle regenerates the sampled rays itself
    sc = orc.scene(orc.volume_numpy(vol), cfg.dims, tf, cam, dec)
    threads = os.cpu_count() or 1
    dense = []
    for pe in range(n):
        g = orc.generate_pixels(sc, pe, cfg.k_in, pix, n_threads=threads)
        assert not g["capacity_exceeded"]
        gc, gd, gr = _lists_at(pes[pe], pix, cfg.k_in)
        np.testing.assert_array_equal(gc, g["count"].astype(np.int64), err_msg=f"{name} PE {pe} generator counts")
        np.testing.assert_allclose(gd, g["depth"], rtol=1e-5, err_msg=f"{name} PE {pe} generator depth")
        np.testing.assert_allclose(gr, g["rgba"], atol=1e-4, err_msg=f"{name} PE {pe} generator rgba")
        dense.append(orc.pixels_to_dense(g, W * H, pix))
    ref = orc.composite_pixels(dense, pix, cfg.k_out)
    oc, od, orgba = (strip.count.cpu().numpy()[pix], strip.depth.cpu().numpy()[pix],
                     strip.rgba.cpu().numpy()[pix])
    nl, ties = compare(oc, od, orgba, ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], name)
    print(f"{name}: {len(pix)} sampled lists ({len(srch)} searched in the image), {nl} bit-checked, ties {len(ties)}")
