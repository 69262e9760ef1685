"""Oracle pins for the primitives: over, scan, depth sort, subdivision, tau.

Each pin is something other than the oracle itself: a value printed in the
paper / SPEC worked examples (tests/golden/*.json, cited), a closed form, an
algebraic invariant, or brute force on tiny inputs."""
import heapq

import numpy as np
import pytest

from conftest import golden


def test_over_worked_example(orc):
    g = golden("primitives.json")["over"]
    np.testing.assert_allclose(orc.over(g["front"], g["back"]), g["out"], atol=1e-6)


def test_over_associative_not_commutative(orc):
    # PAPER.md:77 (associativity -> exact image at the generation view),
    # Eq. 3 PAPER.md:191-193 (a over b != b over a)
    rng = np.random.default_rng(0)
    for _ in range(2000):
        a, b, c = [np.append(rng.random(3) * x, x) for x in rng.random(3)]
        l = orc.over(orc.over(a, b), c)
        r = orc.over(a, orc.over(b, c))
        np.testing.assert_allclose(l, r, atol=1e-6)
    a = np.array([0.5, 0, 0, 0.5], np.float32)
    b = np.array([0, 0.5, 0, 0.5], np.float32)
    assert not np.allclose(orc.over(a, b), orc.over(b, a))
    # opaque front hides everything (saturation)
    np.testing.assert_allclose(orc.over([1, 0, 0, 1], [0, 1, 1, 1]), [1, 0, 0, 1])


def test_scan_fig2(orc):
    g = golden("primitives.json")["scan"]
    o = orc.exclusive_scan(g["counts"])
    assert o[:-1].tolist() == g["offsets"] and int(o[-1]) == g["total"]
    assert len(g["counts"]) * 3 == g["slots"]  # N_s = 3 lists of Fig. 1
    rng = np.random.default_rng(1)
    c = rng.integers(0, 21, 10000)
    o = orc.exclusive_scan(c)
    assert o[0] == 0 and np.array_equal(np.diff(o.astype(np.int64)), c)


def _brute_kway(lists):
    """PAPER.md:168 literally: repeatedly pop the lowest-starting head among the
    per-PE sorted runs (ties -> lower PE id, Q11); alpha==0 dropped (Q23)."""
    heads = [0] * len(lists)
    out = []
    while True:
        best = None
        for s, l in enumerate(lists):
            if heads[s] < len(l) and (best is None or l[heads[s]][0] < lists[best][heads[best]][0]):
                best = s
        if best is None:
            return np.array([r for r in out if r[5] != 0], np.float32).reshape(-1, 6)
        out.append(lists[best][heads[best]])
        heads[best] += 1


def test_sort_equals_kway_merge_bruteforce(orc):
    rng = np.random.default_rng(2)
    for case in range(10000):
        n = rng.integers(1, 5)
        lists = []
        for s in range(n):
            c = rng.integers(0, 5)
            tf = np.sort(rng.integers(0, 6, c).astype(np.float32))  # small ints -> many ties
            l = np.zeros((c, 6), np.float32)
            l[:, 0] = tf
            l[:, 1] = tf + 0.5
            l[:, 2] = s
            l[:, 3] = np.arange(c)
            l[:, 5] = rng.choice([0.0, 0.25, 0.5], c)
            lists.append(l)
        got = orc.sort_samples(lists)
        exp = _brute_kway(lists)
        assert np.array_equal(got, exp), case


def test_adjusted_opacity_example(orc):
    # SPEC.md:358 via the subdivision of a record into two halves.
    g = golden("primitives.json")["adjusted_opacity"]
    a = g["alpha"]
    rec = [0.0, g["l_stored"], a, 0, 0, a]
    cut = [g["l_covered"], g["l_covered"] + 0.25, 0, 0, 0, 1e-30]  # negligible record forcing a cut at l=1
    out = orc.subdivide(np.array([rec, cut], np.float32))
    assert out.shape[0] == 3
    np.testing.assert_allclose(out[0, 5], g["out"], atol=1e-6)


def test_subdivision_closed_form(orc):
    g = golden("subdivision.json")
    srt = orc.sort_samples([np.array(l, np.float32) for l in g["lists"]])
    out = orc.subdivide(srt)
    np.testing.assert_allclose(out, np.array(g["out"], np.float32), atol=g["tol"])


def test_subdivision_preserves_composite(orc):
    """Splitting records and re-compositing the pieces reproduces them:
    prod (1-alpha)^(l_i/l) = 1-alpha and the colours telescope (Eq. 2)."""
    rng = np.random.default_rng(3)
    for _ in range(500):
        n = rng.integers(2, 6)
        recs = []
        for _ in range(n):
            tf = rng.uniform(0, 2)
            a = rng.uniform(0.05, 0.9)
            recs.append([tf, tf + rng.uniform(0.1, 1.0), a * rng.random(), a * rng.random(), a * rng.random(), a])
        recs = np.array(recs, np.float32)
        srt = orc.sort_samples([recs])
        out = orc.subdivide(srt)
        # output is sorted and non-overlapping
        assert np.all(out[1:, 0] >= out[:-1, 1])
        # total transmittance equals the product over records (order-free)
        np.testing.assert_allclose(np.prod(1 - out[:, 5].astype(np.float64)),
                                   np.prod(1 - recs[:, 5].astype(np.float64)), atol=1e-5)
        # a single record is untouched; disjoint inputs are untouched
    disj = np.array([[0, 1, .1, .1, .1, .3], [1, 2, .2, 0, 0, .4], [3, 4, 0, 0, .1, .2]], np.float32)
    assert np.array_equal(orc.subdivide(disj), disj)


def test_tau_direction(orc):
    """SPEC.md:244-245 under Q1 (split iff D > gamma, merge on equality)."""
    g = golden("primitives.json")["tau"]
    a = np.array(g["a"], np.float32)
    b = a + np.array(g["b_offset"], np.float32)  # distance 0.3 from a (one component)
    samples = np.array([[0, 1, *a], [1, 2, *b]], np.float32)
    for gamma, split in zip(g["gammas"], g["splits"]):
        n = orc.sweep(samples, gamma, 8, write=False)
        assert n == (2 if split else 1)
    # merge on equality: identical samples never split, even at gamma = 0
    same = np.array([[0, 1, .2, .2, .2, .4], [1, 2, .2, .2, .2, .4]], np.float32)
    assert orc.sweep(same, 0.0, 8, write=False) == 1


def test_full_rep_size_matches_paper():
    g = golden("primitives.json")["full_rep_size"]
    mib = g["W"] * g["H"] * g["k"] * g["bytes_per_slot"] / 2 ** 20
    assert abs(mib - g["MiB"]) < 1e-9 and abs(mib - 950) < 1.0
