"""The multi-GPU path (§8(e)) on ONE device.

G contexts of one process form a VDI_FLAG_LOOPBACK group, each rank driven by
its own host thread with its own stream: the same device code as G processes
on G GPUs -- strip bounds found on the device, the push of every (PE, strip)
slice into the owner's window, block-counted ready flags, the receive-side
scan and merge, the compaction of each strip into the root's window and the
root's inflate -- with the window pointers exchanged in-process instead of by
NCCL + CUDA IPC.  Kernels that spin on each other must not share a device
(B200_PROFILING.md), so a loopback rank waits for its peers on the host
(events) and only checks the flag words on the device (shortfalls fail
vdi_get_counters).  Results are compared with the oracle's direct-send
composite (orc.composite(..., G): strips, simulated exchange, gather) element
by element and with the one-context image bit for bit; exchange bytes are
checked for conservation against the seeded inputs."""
import os
import threading

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
    vdi._lib.lib()
    return vdi


def _group(vdi, G, W, H, k_in, k_out, n, flags=0, root=0, stats=True):
    key = os.urandom(128)
    L = vdi._lib
    extra = L.VDI_FLAG_PIXEL_STATS if stats else 0
    return [vdi.Compositor(W, H, k_in, k_out, n, n_ranks=G, rank=r, root=root, unique_id=key,
                           flags=flags | L.VDI_FLAG_LOOPBACK | extra | L.VDI_FLAG_STAGE_TIMING,
                           stream=torch.cuda.Stream()) for r in range(G)]


def _one_gpu(vdi, pes_dev, W, H, k_in, k_out):
    c = vdi.Compositor(W, H, k_in, k_out, len(pes_dev), flags=vdi._lib.VDI_FLAG_PIXEL_STATS)
    s = c.empty_strip()
    c.composite(pes_dev, s)
    torch.cuda.synchronize()
    g, m, mg = c.pixel_stats(with_margin=True)
    return s, g.cpu().numpy(), m.cpu().numpy(), mg.cpu().numpy()


def _local(vdi, comps, pes_dev, r):
    n = len(pes_dev)
    return [pes_dev[s] for s in range(n) if vdi.pe_home(n, len(comps), s) == r]


def _threads(fns):
    """Run fns[r] (rank r's calls) in one host thread per rank; re-raise errors."""
    errors = []

    def wrap(f):
        try:
            f()
        except Exception as e:  # noqa: BLE001 -- surfaced below
            errors.append(e)
    th = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not any(t.is_alive() for t in th), "a loopback rank did not finish"
    assert not errors, errors


def _run(vdi, comps, pes_dev, root, images, strips):
    """Every rank (thread): composite of its strip, then the gather to root."""
    def rank(r, c):
        def f():
            c.composite(_local(vdi, comps, pes_dev, r), strips[r])
            c.gather(strips[r], images if r == root else None, root=root)
        return f
    _threads([rank(r, c) for r, c in enumerate(comps)])


def _assert_equal_full(a, b, what):
    for x, y, nm in ((a.count, b.count, "count"), (a.depth, b.depth, "depth"), (a.rgba, b.rgba, "rgba")):
        assert torch.equal(x, y), f"{what}: {nm} differs"


CASES = [
    # G, n, W, H, k_in, k_out, lam  (W = 203: strips not 32-list aligned -> per-rank inflates)
    (2, 8, 203, 97, 20, 20, 12.0),
    (3, 5, 128, 90, 12, 8, 9.0),
    (4, 8, 256, 64, 20, 20, 14.0),
    (4, 3, 96, 41, 6, 6, 5.0),      # fewer PEs than ranks: rank 3 homes none
    (8, 8, 256, 64, 20, 20, 14.0),  # the north-star rank count (one PE per rank)
    (8, 16, 160, 40, 8, 8, 10.0),   # 8 ranks, two PEs each, unaligned strips
]


@pytest.mark.parametrize("case", CASES, ids=[f"G{c[0]}_n{c[1]}_{c[2]}x{c[3]}_k{c[4]}-{c[5]}" for c in CASES])
def test_loopback_strips_match_oracle(vdi, orc, case):
    G, n, W, H, k_in, k_out, lam = case
    pes = synth.random_subvdis(n, W, H, k_in, lam=lam, seed=900 + G + n)
    ref = orc.composite(pes, W, H, G, k_out)
    dev = [dense_to_device(p, i) for i, p in enumerate(pes)]
    # half the PEs without offset arrays: their strip bounds come from a scan of the counts
    dev = [d if d.pe_id % 2 == 0 else vdi.DenseSubVDI(d.pe_id, d.total, d.count, None, d.depth, d.rgba) for d in dev]
    one, g1, m1, mg1 = _one_gpu(vdi, dev, W, H, k_in, k_out)
    comps = _group(vdi, G, W, H, k_in, k_out, n)
    strips = [c.empty_strip() for c in comps]
    image = vdi.FullVDI.empty(W, 0, H, k_out)
    _run(vdi, comps, dev, 0, image, strips)
    torch.cuda.synchronize()
    _assert_equal_full(image, one, f"G={G} image vs 1 GPU")
    nl, ties = compare(*full_to_numpy(image), ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"],
                       f"G={G}")
    # per-strip statistics (gamma*, m, tie margin) equal the one-context ones
    P_img = W * H
    for r, c in enumerate(comps):
        g, m, mg = (t.cpu().numpy() for t in c.pixel_stats(with_margin=True))
        a, b = c.row_begin * W, c.row_end * W
        assert np.array_equal(g, g1[a:b]) and np.array_equal(m, m1[a:b]) and np.array_equal(mg, mg1[a:b])
    # exchange bytes: what rank r sent = sum over its PEs and strips g != r of
    # (count slice + 24 B per record); what g received = what the others sent it
    rows = [vdi.strip_rows(H, G, g) for g in range(G)]
    sent = np.zeros(G, np.int64)
    recv = np.zeros(G, np.int64)
    for s, p in enumerate(pes):
        h = vdi.pe_home(n, G, s)
        off = np.concatenate([[0], np.cumsum(p["count"].astype(np.int64))])
        for g, (a, b) in enumerate(rows):
            if g == h:
                continue
            nb = (b - a) * W + 24 * int(off[b * W] - off[a * W])
            sent[h] += nb
            recv[g] += nb
    for r, c in enumerate(comps):
        cnt = c.counters()
        assert cnt["bytes_sent"] == sent[r], (r, cnt["bytes_sent"], sent[r])
        assert cnt["bytes_received"] == recv[r], (r, cnt["bytes_received"], recv[r])
    print(f"G={G}: {nl} lists checked vs oracle, ties {len(ties)}, bytes sent {sent.tolist()}")
    for c in comps:
        c.close()


def test_loopback_frames_rotating_root(vdi, orc):
    """Five consecutive frames (different inputs) through one loopback group,
    gathered to roots 0, 1, 2, 0, 1: every window parity and flag epoch is
    reused; each frame's image equals its one-context image bit for bit."""
    G, n, W, H, k = 3, 6, 160, 75, 12
    comps = _group(vdi, G, W, H, k, k, n)
    strips = [c.empty_strip() for c in comps]
    frames, images, ones = [], [], []
    for f in range(5):
        pes = synth.random_subvdis(n, W, H, k, lam=8.0 + f, seed=1200 + f)
        dev = [dense_to_device(p, i) for i, p in enumerate(pes)]
        frames.append((pes, dev))
        ones.append(_one_gpu(vdi, dev, W, H, k, k)[0])
    images = [vdi.FullVDI.empty(W, 0, H, k) for _ in frames]
    torch.cuda.synchronize()

    def rank(r, c):
        def f():  # all five frames back to back, no host synchronisation between them
            for fi, (pes, dev) in enumerate(frames):
                c.composite(_local(vdi, comps, dev, r), strips[r])
                c.gather(strips[r], images[fi] if r == fi % G else None, root=fi % G)
        return f
    _threads([rank(r, c) for r, c in enumerate(comps)])
    torch.cuda.synchronize()
    for f in range(5):
        _assert_equal_full(images[f], ones[f], f"frame {f}")
    pes = frames[-1][0]
    ref = orc.composite(pes, W, H, G, k)
    compare(*full_to_numpy(images[-1]), ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], "rot")
    for c in comps:
        c.close()


def test_loopback_fullrep(vdi, orc):
    """vdi_composite_fullrep across a loopback group (fixed-size slices of the
    full representation pushed into the same windows, Fig. 6 "full"): the same
    image as the dense path."""
    G, n, W, H, k_in, k_out = 2, 4, 100, 60, 8, 6
    pes = synth.random_subvdis(n, W, H, k_in, lam=7.0, seed=1300)
    dev = [dense_to_device(p, i) for i, p in enumerate(pes)]
    one = _one_gpu(vdi, dev, W, H, k_in, k_out)[0]
    comps = _group(vdi, G, W, H, k_in, k_out, n)
    fulls = [comps[0].dense_to_full(d) for d in dev]
    torch.cuda.synchronize()
    strips = [c.empty_strip() for c in comps]
    image = vdi.FullVDI.empty(W, 0, H, k_out)
    def rank(r):
        def f():
            ids = [s for s in range(n) if vdi.pe_home(n, G, s) == r]
            comps[r].composite_fullrep([fulls[s] for s in ids], ids, strips[r])
            comps[r].gather(strips[r], image if r == 0 else None)
        return f
    _threads([rank(r) for r in range(G)])
    torch.cuda.synchronize()
    _assert_equal_full(image, one, "fullrep G=2")
    for c in comps:
        c.close()


@pytest.mark.parametrize("span", [False, True])
def test_loopback_host_entries(vdi, span):
    """The host entry points at n_ranks > 1: every rank runs
    vdi_composite_host_dense_frames in its own thread over 3 distinct input
    sets in an order that reuses both input slots; each frame's dense strip
    equals the rows of the one-context composite of that frame, bit for bit.
    span: the inputs of a frame packed in one pinned arena (VDI_FLAG_HOST_SPAN)."""
    G, n, W, H, k = 2, 4, 96, 50, 8
    L = vdi._lib
    comps = _group(vdi, G, W, H, k, k, n, flags=L.VDI_FLAG_HOST_SPAN if span else 0)
    sets = [synth.random_subvdis(n, W, H, k, lam=7.0 + s, seed=1400 + s) for s in range(3)]
    order = [0, 1, 2, 1, 0]
    ones = [_one_gpu(vdi, [dense_to_device(p, i) for i, p in enumerate(pes)], W, H, k, k)[0] for pes in sets]

    def host_pes(pes, ids):
        hs = [dense_to_device(pes[s], s, device="cpu") for s in ids]
        if not span:
            return [h.to("cpu", pin=True) for h in hs], None
        parts = [[h.count, h.depth, h.rgba] for h in hs]
        sizes = [[(t.numel() * t.element_size() + 255) // 256 * 256 for t in ts] for ts in parts]
        arena = torch.empty(sum(map(sum, sizes)), dtype=torch.uint8).pin_memory()
        out, off = [], 0
        for h, ts, ss in zip(hs, parts, sizes):
            hv = []
            for t, sz in zip(ts, ss):
                nb = t.numel() * t.element_size()
                v = arena[off:off + nb].view(t.dtype).view(t.shape)
                v.copy_(t)
                hv.append(v)
                off += sz
            out.append(vdi.DenseSubVDI(h.pe_id, h.total, hv[0], None, hv[1], hv[2]))
        return out, arena

    results = [None] * G
    errors = []

    def rank(r):
        try:
            ids = [s for s in range(n) if vdi.pe_home(n, G, s) == r]
            frames, keep = [], []
            for i in order:
                hp, arena = host_pes(sets[i], ids)
                frames.append(hp)
                keep.append(arena)
            P = (comps[r].row_end - comps[r].row_begin) * W
            outs = [(torch.empty(P, dtype=torch.uint8), torch.empty((P * k, 2), dtype=torch.float32),
                     torch.empty((P * k, 4), dtype=torch.float32)) for _ in order]
            Ts = comps[r].composite_host_dense_frames(frames, outs)
            results[r] = (Ts, outs)
        except Exception as e:  # surfaced below
            errors.append(e)

    _threads([(lambda r=r: rank(r)) for r in range(G)])
    assert not errors, errors
    for r, c in enumerate(comps):
        Ts, outs = results[r]
        a, b = c.row_begin * W, c.row_end * W
        for f, i in enumerate(order):
            fc, fd, fr = (x[a:b].cpu().numpy() for x in (ones[i].count, ones[i].depth, ones[i].rgba))
            sel = np.arange(k)[None, :] < fc[:, None].astype(np.int64)
            assert Ts[f] == int(sel.sum()), (r, f)
            assert np.array_equal(outs[f][0].numpy(), fc), (r, f)
            assert np.array_equal(outs[f][1].numpy()[:Ts[f]], fd[sel]) and \
                np.array_equal(outs[f][2].numpy()[:Ts[f]], fr[sel]), (r, f)
    for c in comps:
        c.close()


@pytest.mark.parametrize("rotate,overlap,G", [(False, True, 3), (True, True, 3), (True, False, 3), (True, True, 8)])
def test_loopback_composite_frames(vdi, rotate, overlap, G):
    """vdi_composite_frames (frames in flight through strip mode): the root
    merges into its image rows and inflates the others on a second stream;
    six frames, one root or a rotating one -- each image equals the
    one-context composite of its frame bit for bit."""
    n, W, H, k = 6, 128, 72, 10
    F = 6
    comps = _group(vdi, G, W, H, k, k, n, stats=not overlap)  # PIXEL_STATS turns the search overlap off
    frames = []
    for f in range(F):
        pes = synth.random_subvdis(n, W, H, k, lam=7.0 + f, seed=1500 + f)
        frames.append([dense_to_device(p, i) for i, p in enumerate(pes)])
    ones = [_one_gpu(vdi, fr, W, H, k, k)[0] for fr in frames]
    roots = [f % G if rotate else 0 for f in range(F)]
    images = {r: [vdi.FullVDI.empty(W, 0, H, k) if roots[f] == r else None for f in range(F)] for r in range(G)}
    torch.cuda.synchronize()
    _threads([(lambda r=r, c=c: c.composite_frames([_local(vdi, comps, fr, r) for fr in frames], images[r],
                                                   roots=roots)) for r, c in enumerate(comps)])
    torch.cuda.synchronize()
    for f in range(F):
        _assert_equal_full(images[roots[f]][f], ones[f], f"frame {f} (root {roots[f]})")
    for c in comps:
        c.close()
