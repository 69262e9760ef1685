"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Inputs come from synth/ (neutral generators) or from
the oracle itself -- never from the CUDA path."""
import numpy as np
import pytest
import torch

import synth
from parity import compare, dense_to_device, full_to_numpy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vdi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2206_14503_b200 as vdi
    vdi._lib.lib()  # fail loudly if libvdi.so is missing
    return vdi


def _gpu_composite(vdi, pes_np, W, H, k_in, k_out, flags=0, host=False, margin=False):
    n = len(pes_np)
    comp = vdi.Compositor(W, H, k_in, k_out, n, flags=flags | vdi._lib.VDI_FLAG_PIXEL_STATS)
    if host:
        dev = [dense_to_device(p, i, device="cpu") for i, p in enumerate(pes_np)]
        strip = comp.empty_strip(device="cpu")
        comp.composite_host(dev, strip)
    else:
        dev = [dense_to_device(p, i) for i, p in enumerate(pes_np)]
        strip = comp.empty_strip()
        comp.composite(dev, strip)
    torch.cuda.synchronize()
    g, m, mg = comp.pixel_stats(with_margin=True)
    cnt = comp.counters()
    if margin:
        return strip, g.cpu().numpy(), m.cpu().numpy(), cnt, mg.cpu().numpy()
    return strip, g.cpu().numpy(), m.cpu().numpy(), cnt


CASES = [
    # n, W, H, k_in, k_out, lam, overlap
    (2, 64, 48, 4, 4, 3.0, False),
    (8, 203, 97, 20, 20, 3.0, False),     # ragged: P = 19691 (not a multiple of 32)
    (8, 203, 97, 20, 20, 20.0, False),    # search-heavy, m up to 160
    (4, 100, 37, 8, 3, 4.0, False),       # k_out < k_in
    (3, 64, 33, 4, 4, 6.0, True),         # overlapping records -> subdivision
    (1, 77, 41, 20, 20, 10.0, False),     # single PE: identity
    (16, 96, 64, 32, 32, 16.0, False),    # n = 16, k = 32 (C5-like)
    (5, 50, 50, 6, 1, 4.0, False),        # k_out = 1
    (12, 40, 40, 10, 20, 8.0, False),     # non-power-of-two n, k_out > k_in
    (33, 32, 8, 4, 8, 3.0, False),        # n > 16 (generic path)
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_{c[1]}x{c[2]}_k{c[3]}-{c[4]}_lam{c[5]}{'_ov' if c[6] else ''}"
                                             for c in CASES])
def test_merge_parity_random(vdi, orc, case):
    n, W, H, k_in, k_out, lam, overlap = case
    pes = synth.random_subvdis(n, W, H, k_in, lam=lam, seed=100 + n, overlap=overlap)
    ref = orc.composite(pes, W, H, 1, k_out)
    strip, gam, m, cnt, mg = _gpu_composite(vdi, pes, W, H, k_in, k_out, margin=True)
    gc, gd, gr = full_to_numpy(strip)
    nl, ties = compare(gc, gd, gr, ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], str(case))
    st = ref["stats"]
    # the per-list gamma*, m and tie margin are reproduced on every list (ties included)
    assert np.array_equal(gam, st["gamma"])
    assert np.array_equal(m.astype(np.int64), st["m"].astype(np.int64))
    om = st["margin"].astype(np.float32)
    fin = np.isfinite(om)
    assert np.array_equal(np.isfinite(mg), fin)
    if overlap:  # subdivided samples carry powf results (ulp-level host/device differences)
        np.testing.assert_allclose(mg[fin], om[fin], rtol=0, atol=1e-6)
    else:        # identical comparisons: identical margins, identical tie lists
        assert np.array_equal(mg[fin], om[fin])
        assert np.nonzero(mg < 1e-6)[0].tolist() == ties
    assert cnt["records_in"] == sum(int(p["count"].sum()) for p in pes)
    print(f"{case}: {nl} lists bit-checked, ties listed: {ties[:20]} ({len(ties)}); searched {cnt['searched_lists']}")


def test_empty_and_transparent(vdi, orc):
    W, H = 70, 30
    empty = [{"count": np.zeros(W * H, np.uint8), "depth": np.zeros((0, 2), np.float32),
              "rgba": np.zeros((0, 4), np.float32)} for _ in range(3)]
    strip, _, _, _ = _gpu_composite(vdi, empty, W, H, 4, 4)
    gc, gd, gr = full_to_numpy(strip)
    assert not gc.any() and not gd.any() and not gr.any()
    # alpha == 0 records are dropped (Q23)
    pes = synth.random_subvdis(4, W, H, 6, lam=5.0, seed=5)
    rng = np.random.default_rng(0)
    for p in pes:
        z = rng.random(len(p["rgba"])) < 0.2
        p["rgba"][z] = 0.0
    ref = orc.composite(pes, W, H, 1, 6)
    strip, _, _, _ = _gpu_composite(vdi, pes, W, H, 6, 6)
    compare(*full_to_numpy(strip), ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], "alpha0")


def test_host_entry_and_determinism(vdi, orc):
    W, H, n, k = 128, 72, 6, 12
    pes = synth.random_subvdis(n, W, H, k, lam=9.0, seed=21)
    a, *_ = _gpu_composite(vdi, pes, W, H, k, k)
    b, *_ = _gpu_composite(vdi, pes, W, H, k, k)
    c, *_ = _gpu_composite(vdi, pes, W, H, k, k, host=True)
    for x, y in ((a, b), (a, c)):
        for u, v in zip(full_to_numpy(x), full_to_numpy(y)):
            assert np.array_equal(u, v)


def _c1_scene(orc, view=0, angle=0.0, decomp=None, n_pes=None, k=None):
    cfg = synth.config_by_name("C1")
    vol_t = synth.make_volume(cfg)
    tf = synth.tf_table(cfg.tf)
    cam = synth.make_camera(cfg.W, cfg.H, view=view, angle_deg=angle)
    dec = decomp if decomp is not None else cfg.decomposition()
    sc = orc.scene(orc.volume_numpy(vol_t), cfg.dims, tf, cam, dec)
    return cfg, vol_t, tf, cam, dec, sc


@pytest.mark.parametrize("variant", ["slab", "interleaved_v1"])
def test_generator_parity_c1(vdi, orc, variant):
    """vdi_generate_subvdi vs the oracle generator (SUPPORT path)."""
    if variant == "slab":
        cfg, vol_t, tf, cam, dec, sc = _c1_scene(orc)
        n, k = cfg.n_pes, cfg.k_in
    else:
        dec = synth.interleaved_decomposition((64, 64, 64), 4, (4, 4, 4), seed=3)
        cfg, vol_t, tf, cam, dec, sc = _c1_scene(orc, view=1, angle=20.0, decomp=dec)
        n, k = 4, 8
    comp = vdi.Compositor(cfg.W, cfg.H, k, k, n)
    tft = torch.from_numpy(tf).cuda()
    volc = vol_t.cuda()
    for pe in range(n):
        g = comp.generate_subvdi(volc, tft, cam, dec, pe)
        o = orc.generate_dense(sc, pe, k)
        assert np.array_equal(g.count.cpu().numpy(), o["count"]), f"pe {pe} counts"
        assert g.total == len(o["depth"])
        np.testing.assert_allclose(g.depth.cpu().numpy(), o["depth"], rtol=1e-5)
        np.testing.assert_allclose(g.rgba.cpu().numpy(), o["rgba"], atol=1e-4)


def test_composite_parity_c1_oracle_inputs(vdi, orc):
    cfg, vol_t, tf, cam, dec, sc = _c1_scene(orc)
    pes = [orc.generate_dense(sc, pe, cfg.k_in) for pe in range(cfg.n_pes)]
    ref = orc.composite(pes, cfg.W, cfg.H, 1, cfg.k_out)
    strip, gam, m, _ = _gpu_composite(vdi, pes, cfg.W, cfg.H, cfg.k_in, cfg.k_out)
    compare(*full_to_numpy(strip), ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], "C1")
    # end-to-end on the GPU (GPU generator + GPU composite) rendered at the
    # generation view equals the oracle's whole-volume DVR
    comp = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes)
    tft = torch.from_numpy(tf).cuda()
    volc = vol_t.cuda()
    g = [comp.generate_subvdi(volc, tft, cam, dec, pe) for pe in range(cfg.n_pes)]
    s2 = comp.empty_strip()
    comp.composite(g, s2)
    c2, d2, r2 = full_to_numpy(s2)
    img = orc.render_full(c2, r2)
    assert np.abs(img - orc.dvr(sc)).max() <= 1e-3


def test_full_size_synthetic_whole_image(vdi, orc):
    """1920x1080, 8 PEs, k=20 merge-only inputs (synth only) in the bench's
    launch configuration: ALL 2,073,600 lists against orc.composite (OpenMP
    over the host cores), ties included; the GPU's own tie list equals the
    oracle's."""
    import os
    W, H, n, k = 1920, 1080, 8, 20
    pes = synth.random_subvdis(n, W, H, k, lam=10.0, seed=7)
    strip, gam, m, cnt, mg = _gpu_composite(vdi, pes, W, H, k, k, margin=True)
    ref = orc.composite(pes, W, H, 1, k, n_threads=os.cpu_count() or 1)
    gc, gd, gr = full_to_numpy(strip)
    nl, ties = compare(gc, gd, gr, ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], "1080p")
    assert nl == W * H
    assert np.array_equal(gam, ref["stats"]["gamma"])
    assert np.nonzero(mg < 1e-6)[0].tolist() == ties
    assert cnt["records_in"] == sum(int(p["count"].sum()) for p in pes)
    print(f"1080p whole image: {nl} lists, {int((m > k).sum())} searched, ties {len(ties)}")


def test_dense_to_full_and_fullrep_composite(vdi, orc):
    """vdi_dense_to_full gives the full representation of a sub-VDI (records in
    the first count slots, zeros elsewhere); compositing from the
    full representation (vdi_composite_fullrep, Fig. 6 "full") gives the same
    image as the dense path."""
    n, W, H, k_in, k_out = 5, 120, 70, 10, 8
    pes = synth.random_subvdis(n, W, H, k_in, lam=8.0, seed=611)
    comp = vdi.Compositor(W, H, k_in, k_out, n)
    dev = [dense_to_device(p, i) for i, p in enumerate(pes)]
    fulls = [comp.dense_to_full(d) for d in dev]
    torch.cuda.synchronize()
    for p, f in zip(pes, fulls):  # layout law, checked on the host from the seeded inputs
        c = np.asarray(p["count"], np.int64)
        off = np.concatenate([[0], np.cumsum(c)])
        fc, fd, fr = full_to_numpy(f)
        assert np.array_equal(fc, p["count"])
        slot = np.arange(k_in)[None, :] < c[:, None]
        idx = (off[:-1, None] + np.arange(k_in)[None, :])[slot]
        assert np.array_equal(fd[slot], p["depth"][idx]) and np.array_equal(fr[slot], p["rgba"][idx])
        assert not fd[~slot].any() and not fr[~slot].any()
    a = comp.empty_strip()
    comp.composite(dev, a)
    b = comp.empty_strip()
    comp.composite_fullrep(fulls, list(range(n)), b)
    torch.cuda.synchronize()
    for x, y in ((a.count, b.count), (a.depth, b.depth), (a.rgba, b.rgba)):
        assert torch.equal(x, y)
    ref = orc.composite(pes, W, H, 1, k_out)
    gc, gd, gr = full_to_numpy(b)
    compare(gc, gd, gr, ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], "fullrep")


def test_offsets_or_receive_scan_same_image(vdi):
    """One GPU: with every source's offset array the merge reads the group
    bases from it; without, it scans the counts (receive-side scan,
    PAPER.md:166).  Same image."""
    n, W, H, k = 7, 131, 53, 9
    pes = synth.random_subvdis(n, W, H, k, lam=7.0, seed=77)
    comp = vdi.Compositor(W, H, k, k, n)
    dev = [dense_to_device(p, i) for i, p in enumerate(pes)]
    a = comp.empty_strip()
    comp.composite(dev, a)
    no_off = [vdi.DenseSubVDI(d.pe_id, d.total, d.count, None, d.depth, d.rgba) for d in dev]
    b = comp.empty_strip()
    comp.composite(no_off, b)
    torch.cuda.synchronize()
    for x, y in ((a.count, b.count), (a.depth, b.depth), (a.rgba, b.rgba)):
        assert torch.equal(x, y)


def test_host_dense_output(vdi):
    """vdi_composite_host_dense: host sub-VDIs in, the composited strip back
    in the dense representation -- the counts of the device composite and its
    non-empty slots packed in list order."""
    n, W, H, k = 5, 97, 61, 10
    pes = synth.random_subvdis(n, W, H, k, lam=8.0, seed=91)
    comp = vdi.Compositor(W, H, k, k, n)
    dev = [dense_to_device(p, i) for i, p in enumerate(pes)]
    full = comp.empty_strip()
    comp.composite(dev, full)
    torch.cuda.synchronize()
    host = [dense_to_device(p, i, device="cpu") for i, p in enumerate(pes)]
    cap = W * H * k
    hc = torch.empty(W * H, dtype=torch.uint8)
    hd = torch.empty((cap, 2), dtype=torch.float32)
    hr = torch.empty((cap, 4), dtype=torch.float32)
    T = comp.composite_host_dense(host, hc, hd, hr)
    fc, fd, fr = full_to_numpy(full)
    assert np.array_equal(hc.numpy(), fc)
    sel = np.arange(k)[None, :] < fc[:, None].astype(np.int64)
    assert T == int(sel.sum())
    assert np.array_equal(hd.numpy()[:T], fd[sel]) and np.array_equal(hr.numpy()[:T], fr[sel])
    small = torch.empty((max(T - 1, 1), 2), dtype=torch.float32), torch.empty((max(T - 1, 1), 4), dtype=torch.float32)
    with pytest.raises(Exception):
        comp.composite_host_dense(host, hc, small[0], small[1])  # VDI_ERR_CAPACITY


def test_host_dense_frames_pipeline(vdi):
    """vdi_composite_host_dense_frames: each frame of the pipelined call (H2D /
    compositing / D2H of consecutive frames overlapped, double-buffered slots)
    equals vdi_composite_host_dense on that frame's inputs, bit for bit; frames
    differ (three input sets, five frames: every slot is reused)."""
    n, W, H, k = 4, 83, 47, 8
    sets = [synth.random_subvdis(n, W, H, k, lam=7.0 + s, seed=300 + s) for s in range(3)]
    comp = vdi.Compositor(W, H, k, k, n)
    host = [[dense_to_device(p, i, device="cpu") for i, p in enumerate(pes)] for pes in sets]
    cap = W * H * k
    mk = lambda c: (torch.empty(W * H, dtype=torch.uint8), torch.empty((c, 2), dtype=torch.float32),
                    torch.empty((c, 4), dtype=torch.float32))
    want = []
    for hs in host:
        o = mk(cap)
        T = comp.composite_host_dense(hs, *o)
        want.append((T, o))
    order = [0, 1, 2, 1, 0]
    outs = [mk(cap) for _ in order]
    Ts = comp.composite_host_dense_frames([host[i] for i in order], outs)
    for f, i in enumerate(order):
        T, (wc, wd, wr) = want[i]
        assert Ts[f] == T
        assert torch.equal(outs[f][0], wc)
        assert torch.equal(outs[f][1][:T], wd[:T]) and torch.equal(outs[f][2][:T], wr[:T])
    # the same inputs packed in one pinned arena (libvdi's one-copy span path)
    # give the same bits, single-frame and pipelined
    packed = []
    for hs in host:
        parts = [[p.count, p.depth, p.rgba] for p in hs]
        sizes = [[(t.numel() * t.element_size() + 255) // 256 * 256 for t in ts] for ts in parts]
        arena = torch.empty(sum(map(sum, sizes)), dtype=torch.uint8).pin_memory()
        pk, off = [], 0
        for p, ts, ss in zip(hs, parts, sizes):
            hv = []
            for t, sz in zip(ts, ss):
                nb = t.numel() * t.element_size()
                h = arena[off:off + nb].view(t.dtype).view(t.shape)
                h.copy_(t)
                hv.append(h)
                off += sz
            pk.append(vdi.DenseSubVDI(p.pe_id, p.total, hv[0], None, hv[1], hv[2]))
        packed.append((arena, pk))
    o = mk(cap)
    assert comp.composite_host_dense(packed[1][1], *o) == want[1][0]
    assert torch.equal(o[0], want[1][1][0]) and torch.equal(o[2][:want[1][0]], want[1][1][2][:want[1][0]])
    outs = [mk(cap) for _ in order]
    Ts = comp.composite_host_dense_frames([packed[i][1] for i in order], outs)
    for f, i in enumerate(order):
        T, (wc, wd, wr) = want[i]
        assert Ts[f] == T and torch.equal(outs[f][0], wc)
        assert torch.equal(outs[f][1][:T], wd[:T]) and torch.equal(outs[f][2][:T], wr[:T])
    # capacity error is reported after every frame ran; totals are still set
    small = [mk(max(want[i][0] - 1, 1)) for i in order[:2]]
    with pytest.raises(Exception):
        comp.composite_host_dense_frames([host[i] for i in order[:2]], small)


def test_multi_gpu_strip_invariance(vdi):
    """G = 2 (or all visible GPUs): NCCL exchange + gather give the 1-GPU result
    bit-for-bit and match the oracle (tests/mgpu_check.py under torchrun)."""
    import os
    import subprocess
    import sys
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 4)}",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "tests", "mgpu_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("stats", [False, True])
def test_composite_frames_one_gpu(vdi, stats):
    """vdi_composite_frames on one GPU (frames in flight: frame f's search
    kernels beside frame f+1's pass-through, two parities of merge scratch;
    PIXEL_STATS turns the overlap off): every frame equals its own
    vdi_composite bit for bit."""
    n, W, H, k = 6, 200, 90, 12
    frames = [[dense_to_device(p, i) for i, p in enumerate(synth.random_subvdis(n, W, H, k, lam=9.0 + f, seed=700 + f))]
              for f in range(5)]
    comp = vdi.Compositor(W, H, k, k, n, flags=vdi._lib.VDI_FLAG_PIXEL_STATS if stats else 0)
    ones = []
    for fr in frames:
        o = comp.empty_strip()
        comp.composite(fr, o)
        ones.append(o)
    images = [vdi.FullVDI.empty(W, 0, H, k) for _ in frames]
    torch.cuda.synchronize()
    comp.composite_frames(frames, images)
    torch.cuda.synchronize()
    for f in range(len(frames)):
        for a, b in ((images[f].count, ones[f].count), (images[f].depth, ones[f].depth), (images[f].rgba, ones[f].rgba)):
            assert torch.equal(a, b), f


def test_composite_frames_long_schedule(vdi):
    """vdi_composite_frames over frames whose long search fills the GPU
    (> 600 000 lists with m > 40): from the second frame
    on, the long-search kernel's mapped-host hint makes each pass-through wait
    for the previous VDI's search instead of running beside it.  The schedule
    never changes a result: every frame equals its own vdi_composite bit for
    bit (two input sets: the PEs in order and reversed, which changes the
    sources' tie order, Q11)."""
    n, W, H, k = 8, 1200, 900, 32
    base = synth.random_subvdis(n, W, H, k, lam=30.0, seed=900)
    fwd = [dense_to_device(p, i) for i, p in enumerate(base)]
    rev = [dense_to_device(p, i) for i, p in enumerate(base[::-1])]
    frames = [fwd, rev, fwd, rev]
    comp = vdi.Compositor(W, H, k, k, n)
    ones = []
    for fr in frames[:2]:
        o = comp.empty_strip()
        comp.composite(fr, o)
        ones.append(o)
    torch.cuda.synchronize()
    b = comp.counters()["bucket_lists"]
    assert b[2] + b[3] > 600000, b  # the long buckets exceed the schedule's threshold
    images = [vdi.FullVDI.empty(W, 0, H, k) for _ in frames]
    comp.composite_frames(frames, images)
    torch.cuda.synchronize()
    for f in range(len(frames)):
        ref = ones[f % 2]
        for a, c in ((images[f].count, ref.count), (images[f].depth, ref.depth), (images[f].rgba, ref.rgba)):
            assert torch.equal(a, c), f
