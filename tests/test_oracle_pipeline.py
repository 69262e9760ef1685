"""Oracle pins for the whole direct-send composite and the sub-VDI generator:
north-star checks 1-4 on config C1, the hand-checked 4x4 image, strip-count
(G) invariance, and the generator's domain-exit / dense-layout invariants."""
import numpy as np
import pytest

import synth
from conftest import golden


@pytest.fixture(scope="module")
def c1(orc):
    cfg = synth.config_by_name("C1")
    vol = orc.volume_numpy(synth.make_volume(cfg))
    tf = synth.tf_table(cfg.tf)
    cam = synth.make_camera(cfg.W, cfg.H)
    dec = cfg.decomposition()
    sc = orc.scene(vol, cfg.dims, tf, cam, dec)
    pes = [orc.generate_dense(sc, pe, cfg.k_in) for pe in range(cfg.n_pes)]
    return dict(cfg=cfg, vol=vol, tf=tf, cam=cam, dec=dec, sc=sc, pes=pes)


def test_dense_layout(c1):
    """offsets = exclusive scan of counts, payload = sum."""
    for p in c1["pes"]:
        off = p["offset"].astype(np.int64)
        assert off[0] == 0 and np.array_equal(np.diff(off), p["count"].astype(np.int64))
        assert off[-1] == len(p["depth"]) == len(p["rgba"])
        assert p["count"].max() <= c1["cfg"].k_in


def test_composite_matches_dvr(orc, c1):
    """North-star check 2: the composited VDI rendered from the generating
    viewpoint equals direct raycasting of the whole volume within 1e-3
    (PAPER.md:77 exactness by associativity of over)."""
    cfg = c1["cfg"]
    out = orc.composite(c1["pes"], cfg.W, cfg.H, 1, cfg.k_out)
    img = orc.render_full(out["count"], out["rgba"])
    ref = orc.dvr(c1["sc"])
    assert ref[:, 3].max() > 0.5  # the scene is not empty
    assert np.abs(img - ref).max() <= 1e-3
    assert (out["stats"]["m"] > cfg.k_out).sum() > 100  # the search path is exercised


def test_single_pe_identity(orc, c1):
    """North-star check 1: compositing a single PE's VDI is the identity."""
    cfg = c1["cfg"]
    dec1 = synth.slab_decomposition(cfg.dims, 1)
    sc1 = orc.scene(c1["vol"], cfg.dims, c1["tf"], c1["cam"], dec1)
    v = orc.generate_dense(sc1, 0, cfg.k_in)
    out = orc.composite([v], cfg.W, cfg.H, 1, cfg.k_out)
    assert np.array_equal(out["count"], v["count"])
    idx = np.repeat(np.arange(cfg.W * cfg.H), v["count"]) * cfg.k_out + \
        (np.arange(len(v["depth"])) - np.repeat(v["offset"][:-1].astype(np.int64), v["count"]))
    assert np.array_equal(out["depth"].reshape(-1, 2)[idx], v["depth"])
    assert np.array_equal(out["rgba"].reshape(-1, 4)[idx], v["rgba"])
    # whole-volume VDI is also exact vs DVR
    img = orc.render_full(out["count"], out["rgba"])
    assert np.abs(img - orc.dvr(sc1)).max() <= 1e-3


def test_invariants_c1(orc, c1):
    """North-star check 4 on every pixel of C1."""
    cfg = c1["cfg"]
    out = orc.composite(c1["pes"], cfg.W, cfg.H, 1, cfg.k_out)
    n = out["count"].astype(int)
    assert n.max() <= cfg.k_out
    slot = np.arange(cfg.k_out)[None, :]
    used = slot < n[:, None]
    d, c = out["depth"], out["rgba"]
    assert np.all(d[..., 0][used] < d[..., 1][used])
    nxt = used[:, 1:]
    assert np.all(d[:, 1:, 0][nxt] >= d[:, :-1, 1][nxt])
    assert np.all((c[..., 3][used] > 0) & (c[..., 3][used] <= 1))
    assert np.all(c[..., :3][used] <= c[..., 3:][used] + 1e-6)
    assert np.all(d[~used] == 0) and np.all(c[~used] == 0)


def test_strip_count_invariance(orc, c1):
    """The composite depends only on inputs, not on the number of strips G
    (direct-send partition): bit-identical for G = 1, 2, 4, 8."""
    cfg = c1["cfg"]
    ref = orc.composite(c1["pes"], cfg.W, cfg.H, 1, cfg.k_out, with_stats=False)
    for G in (2, 4, 8):
        o = orc.composite(c1["pes"], cfg.W, cfg.H, G, cfg.k_out, with_stats=False)
        for key in ("count", "depth", "rgba"):
            assert np.array_equal(o[key], ref[key])


def test_hand_checked_4x4(orc):
    """North-star check 3: brute force on a 4x4 image with hand-checked lists."""
    g = golden("image4x4.json")
    W, H, k, G = g["W"], g["H"], g["k"], g["G"]
    pes = []
    for pe in g["pes"]:
        cnt = np.zeros(W * H, np.uint8)
        recs = []
        for p in range(W * H):
            l = pe["lists"].get(str(p), [])
            cnt[p] = len(l)
            recs += l
        r = np.array(recs, np.float32).reshape(-1, 6)
        pes.append({"count": cnt, "depth": r[:, :2].copy(), "rgba": r[:, 2:].copy()})
    out = orc.composite(pes, W, H, G, k)
    for p in range(W * H):
        exp = np.array(g["expected"].get(str(p), []), np.float32).reshape(-1, 6)
        n = out["count"][p]
        assert n == len(exp), p
        got = np.concatenate([out["depth"][p], out["rgba"][p]], axis=1)
        np.testing.assert_array_equal(got[:n], exp)
        assert np.all(got[n:] == 0)


def test_generator_domain_exit(orc, c1):
    """a sub-supersegment terminates when the ray leaves the PE's
    domain -- every record covers only samples owned by its PE."""
    cfg, sc = c1["cfg"], c1["sc"]
    for p in np.random.default_rng(5).choice(cfg.W * cfg.H, 60, replace=False):
        own, tlo, thi, _ = orc.ray_owners(sc, p % cfg.W, p // cfg.W)
        for pe, v in enumerate(c1["pes"]):
            o = v["offset"][p]
            for q in range(int(o), int(o) + int(v["count"][p])):
                tf, tb = v["depth"][q]
                inside = (tlo >= tf) & (thi <= tb)
                assert inside.any() and np.all(own[inside] == pe)


def test_nonconvex_interleaved(orc):
    """with a non-convex (interleaved-brick) decomposition the
    depth-ordered composite is still exact vs DVR (Eq. 3 handled by ordering)."""
    cfg = synth.config_by_name("C1")
    vol = orc.volume_numpy(synth.make_volume(cfg))
    tf = synth.tf_table(cfg.tf)
    cam = synth.make_camera(cfg.W, cfg.H, view=1, angle_deg=20)
    dec = synth.interleaved_decomposition(cfg.dims, 4, (4, 4, 4), seed=3)
    sc = orc.scene(vol, cfg.dims, tf, cam, dec)
    pes = [orc.generate_dense(sc, pe, 8) for pe in range(4)]
    out = orc.composite(pes, cfg.W, cfg.H, 2, 8)
    img = orc.render_full(out["count"], out["rgba"])
    assert np.abs(img - orc.dvr(sc)).max() <= 1e-3
    # the limit case: k_out large enough -> over-compositing only
    big = orc.composite(pes, cfg.W, cfg.H, 1, 32)
    assert np.abs(orc.render_full(big["count"], big["rgba"]) - orc.dvr(sc)).max() <= 1e-3


def test_overlapping_inputs_subdivided(orc):
    """Overlapping sub-supersegments (not produced by disjoint domains) are
    subdivided (step 2); exactness of the transmittance still holds."""
    pes = synth.random_subvdis(3, 16, 16, 4, lam=6.0, seed=9, overlap=True)
    out = orc.composite(pes, 16, 16, 1, 4)
    assert out["stats"]["overlap"].sum() > 0
    n = out["count"].astype(int)
    d = out["depth"]
    for p in range(256):
        assert np.all(d[p, 1:n[p], 0] >= d[p, :max(n[p] - 1, 0), 1])
