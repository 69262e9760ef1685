"""Oracle pins for the re-segmentation (steps 3-6): hand fixtures F1-F3
(tests/golden/appendixA.json), the k_out = 1 closed form, the bisection
bracket property, pass-through identity, output invariants and generation-
view exactness (associativity of over)."""
import numpy as np
import pytest

from conftest import golden

FIX = golden("appendixA.json")


@pytest.mark.parametrize("name", ["F1", "F2_k2", "F2_k3", "F3"])
def test_appendix_fixture(orc, name):
    f = FIX[name]
    lists = [np.array(l, np.float32) for l in f["lists"]]
    n, out, st = orc.recomposite(lists, f["k_out"])
    exp = np.array(f["out"], np.float32)
    assert n == len(exp)
    np.testing.assert_array_equal(out[:n], exp)  # dyadic inputs: exact
    assert np.all(out[n:] == 0)
    if "gamma" in f:
        assert st["gamma"] == np.float32(f["gamma"])
    if "trace" in f:
        srt = orc.sort_samples(lists)
        g, trace = orc.gamma_search(srt, f["k_out"])
        assert [list(t) for t in trace] == f["trace"]


def _fold_over(samples):
    acc = np.zeros(4, np.float64)
    for s in samples:
        acc = acc + (1 - acc[3]) * s[2:6].astype(np.float64)
    return acc


def _random_ray(rng, m, gap_p=0.3, equal_p=0.0):
    t = 0.0
    out = []
    for _ in range(m):
        if rng.random() < gap_p:
            t += rng.uniform(0.1, 1.0)
        l = rng.uniform(0.1, 1.0)
        a = rng.uniform(0.01, 0.9)
        if out and rng.random() < equal_p:
            rgba = out[-1][2:]
        else:
            rgba = [a * rng.random(), a * rng.random(), a * rng.random(), a]
        out.append([t, t + l, *rgba])
        t += l
    return np.array(out, np.float32)


def test_k_out_1_closed_form(orc):
    """k_out = 1: a single segment = over of all samples, extent [first.tf, last.tb]."""
    rng = np.random.default_rng(10)
    for _ in range(300):
        S = _random_ray(rng, int(rng.integers(2, 30)))
        n, out, st = orc.recomposite([S], 1)
        assert n == 1
        assert out[0, 0] == S[0, 0] and out[0, 1] == S[-1, 1]
        np.testing.assert_allclose(out[0, 2:], _fold_over(S), atol=1e-5)


def test_bisection_bracket_property(orc):
    """Procedure pin (Q5/Q6): midpoints are the dyadic bisection of [0, 2];
    every mid with count <= k_out becomes the new upper bound (and `best`),
    every infeasible mid the new lower bound; stop at count == k_out or after
    I = 16 iterations; the final count is <= k_out."""
    rng = np.random.default_rng(11)
    for _ in range(400):
        m = int(rng.integers(3, 60))
        S = _random_ray(rng, m, gap_p=rng.random(), equal_p=0.2)
        k = int(rng.integers(1, m))
        g, trace = orc.gamma_search(S, k)
        lo, hi, best = 0.0, 2.0, 2.0
        for i, (mid, c) in enumerate(trace):
            assert mid == np.float32(0.5) * (np.float32(lo) + np.float32(hi))
            assert c == orc.sweep(S, mid, k, write=False)
            if c <= k:
                best = hi = mid
                if c == k:
                    assert i == len(trace) - 1
            else:
                lo = mid
        assert len(trace) <= 16 and g == best
        n, out, st = orc.recomposite([S], k)
        assert n <= k and st["gamma"] == g
        assert n == orc.sweep(S, g, k, write=True)[0]


def test_gamma_max_always_feasible(orc):
    """D <= 2 for premultiplied RGBA in [0,1]^4 and ||acc|| <= 2, so sweep(2)
    never splits: count <= 1 (Q8 keeps gamma_max feasible)."""
    rng = np.random.default_rng(12)
    for _ in range(300):
        S = _random_ray(rng, int(rng.integers(1, 40)), gap_p=0.7)
        assert orc.sweep(S, 2.0, 1, write=False) == 1


def _check_invariants(out, n, k):
    assert 0 <= n <= k
    seg = out[:n]
    assert np.all(seg[:, 0] < seg[:, 1])
    assert np.all(seg[1:, 0] >= seg[:-1, 1])           # depth-ordered, non-overlapping
    assert np.all((seg[:, 5] >= 0) & (seg[:, 5] <= 1))  # opacity in [0,1]
    assert np.all(seg[:, 2:5] <= seg[:, 5:6] + 1e-6)   # premultiplied bound
    assert np.all(out[n:] == 0)                        # zero slots


def test_invariants_and_exactness_random(orc):
    """North-star oracle check 4 (invariants) and PAPER.md:77 exactness: the
    over of the outputs equals the over of the inputs (gaps are empty)."""
    rng = np.random.default_rng(13)
    for _ in range(500):
        n_src = int(rng.integers(1, 6))
        lists = []
        t0 = 0.0
        # disjoint per-source runs interleaved along the ray (non-convex domains)
        pieces = _random_ray(rng, int(rng.integers(1, 40)), gap_p=0.4)
        owner = rng.integers(0, n_src, len(pieces))
        lists = [pieces[owner == s] for s in range(n_src)]
        k = int(rng.integers(1, 25))
        n, out, st = orc.recomposite(lists, k)
        _check_invariants(out, n, k)
        np.testing.assert_allclose(_fold_over(out[:n]), _fold_over(pieces), atol=1e-5)


def test_pass_through_identity(orc):
    """Q9 / north-star check 1: m <= k_out -> the samples verbatim."""
    rng = np.random.default_rng(14)
    for _ in range(200):
        S = _random_ray(rng, int(rng.integers(1, 20)), gap_p=0.5, equal_p=0.3)
        k = int(rng.integers(len(S), 25))
        n, out, st = orc.recomposite([S], k)
        assert n == len(S) and np.array_equal(out[:n], S) and st["gamma"] == 0


def test_empty_and_transparent(orc):
    n, out, st = orc.recomposite([np.zeros((0, 6), np.float32)], 4)
    assert n == 0 and np.all(out == 0)
    z = np.array([[0, 1, 0, 0, 0, 0]], np.float32)  # alpha == 0 dropped (Q23)
    n, out, st = orc.recomposite([z, z], 4)
    assert n == 0
