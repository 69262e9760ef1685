"""Independent pin of the oracle's re-segmentation:
a float32 replica of the greedy sweep and the gamma bisection, written from
the paper (PAPER.md:93-101 Eq. 1 + the per-ray gamma search, :168 depth
order, :176 gaps as transparent samples, :185 full representation) under the
readings Q1-Q9, Q11, Q23 of DESIGN.md §2 -- NOT from oracle/oracle.cpp.

It is a different program: every ray of a batch advances in lock step as a
row of numpy arrays (masks instead of branches), fused multiply-adds are
emulated exactly (float64 product, TwoSum, round-to-nearest-even to float32
with the midpoint decided by the sign of the TwoSum error), and the depth
order is a lexicographic sort by (t_front, PE id, index).  It is compared
BIT FOR BIT with orc.recomposite -- count, gamma*, every output slot -- on
>= 10^4 random rays: contiguous runs, gaps, gap-then-split chains, repeated
samples (D = 0), dyadic values that put D exactly on a bisection midpoint
(merge-on-equality ties, Q1), transparent records (Q23), several PEs whose
runs interleave along the ray, and every k_out from 1 to m - 1."""
import numpy as np
import pytest

F32 = np.float32


# ---------------------------------------------------------------------------
# exact single-rounding fma on float32 arrays
# ---------------------------------------------------------------------------
def fma32(a, b, c):
    a64 = np.asarray(a, F32).astype(np.float64)
    b64 = np.asarray(b, F32).astype(np.float64)
    c64 = np.asarray(c, F32).astype(np.float64)
    p = a64 * b64                      # exact: 24 + 24 bits < 53
    s = p + c64                        # rounded to float64
    bb = s - p                         # TwoSum: s + e == p + c exactly
    e = (p - (s - bb)) + (c64 - bb)
    r = s.astype(F32)                  # ties-to-even when e == 0
    r64 = r.astype(np.float64)
    up = np.nextafter(r, F32(np.inf)).astype(np.float64)
    dn = np.nextafter(r, F32(-np.inf)).astype(np.float64)
    # s exactly on a float32 midpoint: the exact value lies on the side of e
    to_up = (s == 0.5 * (r64 + up)) & (e > 0)
    to_dn = (s == 0.5 * (r64 + dn)) & (e < 0)
    out = np.where(to_up, up, np.where(to_dn, dn, r64)).astype(F32)
    return out


def dist2(acc, s):
    """Eq. 1, Q2 operand order: fma(da,da, fma(db,db, fma(dg,dg, dr*dr)))."""
    dr = (acc[0] - s[0]).astype(F32)
    dg = (acc[1] - s[1]).astype(F32)
    db = (acc[2] - s[2]).astype(F32)
    da = (acc[3] - s[3]).astype(F32)
    return fma32(da, da, fma32(db, db, fma32(dg, dg, (dr * dr).astype(F32))))


# ---------------------------------------------------------------------------
# the replica: R rays at once, samples S[R, M, 6] (tf, tb, r, g, b, a), m[R]
# ---------------------------------------------------------------------------
def sweep(S, m, gamma, k, write):
    """One greedy front-to-back sweep per ray (Q1 split iff
    D > gamma, merge on equality; Q8 a gap is a transparent sample: it closes
    the open segment iff ||acc|| > gamma and never opens one; a closed segment
    ends at its last content sample).  Count mode stops a ray once its count
    exceeds k (the answer is then only "> k")."""
    R, M, _ = S.shape
    g2 = (gamma * gamma).astype(F32)
    cnt = np.zeros(R, np.int64)
    opn = np.zeros(R, bool)
    done = np.zeros(R, bool)
    acc = [np.zeros(R, F32) for _ in range(4)]
    tf = np.zeros(R, F32)
    tb = np.zeros(R, F32)
    prev = np.zeros(R, F32)
    out = np.zeros((R, max(k, 1), 6), F32) if write else None
    zero = [np.zeros(R, F32)] * 4

    def emit(mask):
        if not write or not mask.any():
            return
        idx = np.nonzero(mask)[0]
        slot = cnt[idx] - 1
        ok = slot < k
        idx, slot = idx[ok], slot[ok]
        out[idx, slot] = np.stack([tf[idx], tb[idx], acc[0][idx], acc[1][idx], acc[2][idx], acc[3][idx]], 1)

    for i in range(M):
        live = (i < m) & ~done
        if not live.any():
            break
        s = [S[:, i, 2 + c] for c in range(4)]
        s_tf, s_tb = S[:, i, 0], S[:, i, 1]
        # transparent gap before the sample
        gap = live & opn & (s_tf > prev)
        gclose = gap & (dist2(acc, zero) > g2)
        emit(gclose)
        opn = opn & ~gclose
        split = live & opn & (dist2(acc, s) > g2)
        emit(split)
        start = live & (~opn | split)
        merge = live & opn & ~split
        cnt = cnt + start
        if not write:
            done = done | (cnt > k)
        tr = (F32(1.0) - acc[3]).astype(F32)
        for c in range(4):
            acc[c] = np.where(start, s[c], np.where(merge, fma32(tr, s[c], acc[c]), acc[c])).astype(F32)
        tf = np.where(start, s_tf, tf)
        tb = np.where(start | merge, s_tb, tb)
        opn = opn | start
        prev = np.where(live, s_tb, prev)
    if write:
        emit(opn)
    return cnt, out


def bisect(S, m, k, iters=16, gamma_max=2.0):
    """Per-ray bisection of gamma on [0, gamma_max] (
    Q3 the budget counts segments, Q4 feasible iff count <= k, Q5 mid =
    0.5 (lo + hi) in float32, I iterations, stop at count == k)."""
    R = S.shape[0]
    lo = np.zeros(R, F32)
    hi = np.full(R, F32(gamma_max))
    best = np.full(R, F32(gamma_max))
    act = m > k
    for _ in range(iters):
        if not act.any():
            break
        mid = (F32(0.5) * (lo + hi).astype(F32)).astype(F32)
        c, _ = sweep(S, np.where(act, m, 0), mid, k, write=False)
        feas = act & (c <= k)
        best = np.where(feas, mid, best)
        hi = np.where(feas, mid, hi)
        lo = np.where(act & ~feas, mid, lo)
        act = act & ~(feas & (c == k))
    return best


def prefix_counts(S, m, gamma):
    """Segments opened after each prefix of samples (the sweep of `sweep`,
    no early exit): P[r, q] for q = 0..M."""
    R, M, _ = S.shape
    g2 = (gamma * gamma).astype(F32)
    cnt = np.zeros(R, np.int64)
    opn = np.zeros(R, bool)
    acc = [np.zeros(R, F32) for _ in range(4)]
    prev = np.zeros(R, F32)
    zero = [np.zeros(R, F32)] * 4
    P = np.zeros((R, M + 1), np.int64)
    for i in range(M):
        live = i < m
        s = [S[:, i, 2 + c] for c in range(4)]
        gap = live & opn & (S[:, i, 0] > prev)
        opn = opn & ~(gap & (dist2(acc, zero) > g2))
        split = live & opn & (dist2(acc, s) > g2)
        start = live & (~opn | split)
        merge = live & opn & ~split
        cnt = cnt + start
        tr = (F32(1.0) - acc[3]).astype(F32)
        for c in range(4):
            acc[c] = np.where(start, s[c], np.where(merge, fma32(tr, s[c], acc[c]), acc[c])).astype(F32)
        opn = opn | start
        prev = np.where(live, S[:, i, 1], prev)
        P[:, i + 1] = cnt
    return P


def bisect_ub(S, m, k, every=8, iters=16, gamma_max=2.0):
    """The bisection with the GPU sweeps' early exits (merge.cu, sweep_rows):
    checked every `every` samples, a count sweep stops at count > k (answer
    "> k") or once count + samples left < k, recording that bound as its
    count.  Each sample opens at most one segment, so the bound is >= the full
    count; below k it decides the level as the full count does (<= k, != k).
    Returns gamma per ray."""
    R, M, _ = S.shape
    lo = np.zeros(R, F32)
    hi = np.full(R, F32(gamma_max))
    best = np.full(R, F32(gamma_max))
    act = m > k
    rows = np.arange(R)
    for _ in range(iters):
        if not act.any():
            break
        mid = (F32(0.5) * (lo + hi).astype(F32)).astype(F32)
        P = prefix_counts(S, np.where(act, m, 0), mid)
        c = P[rows, m].copy()                      # the full count
        decided = np.zeros(R, bool)
        for q in range(every, M + 1, every):       # the check points, in order
            cq = P[:, q]
            live = act & ~decided & (q < m)
            over = live & (cq > k)
            under = live & ~over & (cq + (m - q) < k)
            c = np.where(over, cq, np.where(under, cq + (m - q), c))
            decided |= over | under
        feas = act & (c <= k)
        best = np.where(feas, mid, best)
        hi = np.where(feas, mid, hi)
        lo = np.where(act & ~feas, mid, lo)
        act = act & ~(feas & (c == k))
    return best


def sweep_interval(S, m, gamma, k):
    """A count sweep (early exit at count > k) that also returns the interval
    [L, U) of g^2 over which every comparison it made decides the same way:
    L = the largest compared value that merged (<= g^2), U = the smallest
    that split (> g^2); a gap's ||acc||^2 counts as a comparison, and D^2 is
    not compared after a gap closed the segment (Q8)."""
    R, M, _ = S.shape
    g2 = (gamma * gamma).astype(F32)
    cnt = np.zeros(R, np.int64)
    opn = np.zeros(R, bool)
    done = np.zeros(R, bool)
    acc = [np.zeros(R, F32) for _ in range(4)]
    prev = np.zeros(R, F32)
    zero = [np.zeros(R, F32)] * 4
    L = np.full(R, -1.0)
    U = np.full(R, np.inf)
    for i in range(M):
        live = (i < m) & ~done
        if not live.any():
            break
        s = [S[:, i, 2 + c] for c in range(4)]
        gap = live & opn & (S[:, i, 0] > prev)
        n2 = dist2(acc, zero)
        gcl = gap & (n2 > g2)
        U = np.where(gcl, np.minimum(U, n2), U)
        L = np.where(gap & ~gcl, np.maximum(L, n2), L)
        opn = opn & ~gcl
        cmp = live & opn
        d2 = dist2(acc, s)
        split = cmp & (d2 > g2)
        U = np.where(split, np.minimum(U, d2), U)
        L = np.where(cmp & ~split, np.maximum(L, d2), L)
        start = live & (~opn | split)
        merge = live & opn & ~split
        cnt = cnt + start
        done = done | (cnt > k)
        tr = (F32(1.0) - acc[3]).astype(F32)
        for c in range(4):
            acc[c] = np.where(start, s[c], np.where(merge, fma32(tr, s[c], acc[c]), acc[c])).astype(F32)
        opn = opn | start
        prev = np.where(live, S[:, i, 1], prev)
    return cnt, L, U


def bisect_memo(S, m, k, iters=16, gamma_max=2.0):
    """The GPU's memoised bisection (merge.cu, struct Bisection): a level whose
    midpoint^2 lies in the interval of the latest sweep on the feasible (<= k)
    or infeasible (> k) side takes that sweep's answer without sweeping.
    Returns (gamma per ray, sweeps made, levels evaluated = the plain
    procedure's sweeps)."""
    R = S.shape[0]
    lo = np.zeros(R, F32)
    hi = np.full(R, F32(gamma_max))
    best = np.full(R, F32(gamma_max))
    hL, hU, hc = np.ones(R), np.zeros(R), np.zeros(R, np.int64)
    lL, lU = np.ones(R), np.zeros(R)
    act = m > k
    sweeps = levels = 0
    for _ in range(iters):
        if not act.any():
            break
        levels += int(act.sum())
        mid = (F32(0.5) * (lo + hi).astype(F32)).astype(F32)
        g2 = (mid * mid).astype(F32).astype(np.float64)
        in_h = act & (g2 >= hL) & (g2 < hU)
        in_l = act & ~in_h & (g2 >= lL) & (g2 < lU)
        need = act & ~in_h & ~in_l
        c = np.where(in_h, hc, k + 1)
        if need.any():
            cs, L, U = sweep_interval(S, np.where(need, m, 0), mid, k)
            sweeps += int(need.sum())
            c = np.where(need, cs, c)
            fe = need & (cs <= k)
            hL, hU, hc = np.where(fe, L, hL), np.where(fe, U, hU), np.where(fe, cs, hc)
            inf_ = need & (cs > k)
            lL, lU = np.where(inf_, L, lL), np.where(inf_, U, lU)
        feas = act & (c <= k)
        best = np.where(feas, mid, best)
        hi = np.where(feas, mid, hi)
        lo = np.where(act & ~feas, mid, lo)
        act = act & ~(feas & (c == k))
    return best, sweeps, levels


def depth_order(lists):
    """PAPER.md:168 (the lowest starting depth next; Q11 ties by PE id, then
    index) and Q23 (alpha == 0 dropped): one ray's lists -> its samples."""
    recs = [(r[0], s, i, r) for s, l in enumerate(lists) for i, r in enumerate(l) if r[5] != 0]
    recs.sort(key=lambda x: (x[0], x[1], x[2]))
    return np.array([x[3] for x in recs], F32).reshape(-1, 6)


def replica_recomposite(rays, k):
    """rays: list of per-ray source lists -> (count[R], out[R, k, 6], gamma[R])."""
    samples = [depth_order(l) for l in rays]
    R = len(samples)
    m = np.array([len(s) for s in samples], np.int64)
    M = max(1, int(m.max()))
    S = np.zeros((R, M, 6), F32)
    for r, s in enumerate(samples):
        S[r, :len(s)] = s
    gamma = np.where(m > k, bisect(S, m, k), F32(0))
    cnt, out = sweep(S, np.where(m > k, m, 0), gamma.astype(F32), k, write=True)
    out = out[:, :k]
    # m <= k: the samples verbatim (Q9); the rest of the slots zero (Q16)
    for r in np.nonzero(m <= k)[0]:
        out[r] = 0
        out[r, :m[r]] = S[r, :m[r]]
        cnt[r] = m[r]
    return cnt, out, gamma.astype(F32)


# ---------------------------------------------------------------------------
# random rays
# ---------------------------------------------------------------------------
def random_ray(rng, kind):
    m = int(rng.integers(2, 48))
    n_src = int(rng.integers(1, 6))
    dyadic = kind == "dyadic"
    t = F32(0)
    recs = []
    last = None
    for _ in range(m):
        if rng.random() < (0.6 if kind == "gappy" else 0.25):
            t = F32(t + F32(rng.integers(1, 8) / 8 if dyadic else rng.uniform(0.05, 1.0)))
        ln = F32(rng.integers(1, 8) / 8 if dyadic else rng.uniform(0.05, 1.0))
        if last is not None and rng.random() < 0.15:
            rgba = last                                  # repeated sample: D = 0
        elif dyadic:
            a = F32(rng.integers(1, 8) / 8)
            rgba = [F32(rng.integers(0, 9) / 8 * a) for _ in range(3)] + [a]
        else:
            a = F32(rng.uniform(0.005, 0.95))
            rgba = [F32(a * rng.random()) for _ in range(3)] + [a]
        if rng.random() < 0.03:
            rgba = [F32(0)] * 4                          # transparent record (Q23)
        recs.append([t, F32(t + ln)] + list(rgba))
        last = rgba
        t = F32(t + ln)
    recs = np.array(recs, F32)
    owner = rng.integers(0, n_src, len(recs))            # runs of several PEs interleave
    return [recs[owner == s] for s in range(n_src)]


@pytest.mark.parametrize("kind,seed", [("plain", 1), ("gappy", 2), ("dyadic", 3)])
def test_replica_matches_oracle_bitwise(orc, kind, seed):
    rng = np.random.default_rng(1000 + seed)
    rays = [random_ray(rng, kind) for _ in range(3600)]
    ms = np.array([sum(int((l[:, 5] != 0).sum()) for l in r) for r in rays])
    ks = np.array([int(rng.integers(1, max(2, mm))) for mm in ms])  # k_out = 1 .. m - 1
    checked = ties = searched = 0
    for k in np.unique(ks):
        sel = np.nonzero(ks == k)[0]
        cnt, out, gam = replica_recomposite([rays[i] for i in sel], int(k))
        for j, i in enumerate(sel):
            n, o, st = orc.recomposite(rays[i], int(k))
            assert n == cnt[j], (kind, i, k, n, cnt[j])
            assert st["gamma"] == gam[j], (kind, i, k, st["gamma"], gam[j])
            assert np.array_equal(o.view(np.uint32), out[j].view(np.uint32)), (kind, i, k)
            checked += 1
            ties += st["margin"] == 0.0
            searched += ms[i] > k
    assert checked == len(rays) and searched > 0.8 * checked
    if kind == "dyadic":
        assert ties > 50   # merge-on-equality decisions (D == gamma exactly) were exercised
    print(f"{kind}: {checked} rays bit-identical ({searched} searched, {ties} with an exact tie)")


def test_replica_fixtures():
    """The replica reproduces the hand-derived Appendix A fixtures on its own
    (F1: the paper's Ray 3; F2: non-monotone count, a margin-0
    tie; F3: a gap merged)."""
    from conftest import golden
    fx = golden("appendixA.json")
    for name in ("F1", "F2_k2", "F2_k3", "F3"):
        f = fx[name]
        cnt, out, gam = replica_recomposite([[np.array(l, F32).reshape(-1, 6) for l in f["lists"]]], f["k_out"])
        exp = np.array(f["out"], F32)
        assert cnt[0] == len(exp), name
        assert np.array_equal(out[0, :len(exp)], exp), name
        if "gamma" in f:
            assert gam[0] == F32(f["gamma"]), name


def test_fma32_exact():
    """fma32 against exact rational arithmetic on random and midpoint-prone inputs."""
    from fractions import Fraction
    rng = np.random.default_rng(5)
    a = rng.random(4000).astype(F32)
    b = rng.random(4000).astype(F32)
    c = rng.random(4000).astype(F32)
    # midpoint-prone: c = -(a*b rounded) + tiny, products of dyadics
    a[:1000] = (rng.integers(1, 1 << 12, 1000) / (1 << 12)).astype(F32)
    b[:1000] = (rng.integers(1, 1 << 13, 1000) / (1 << 13)).astype(F32)
    c[:1000] = (rng.integers(-(1 << 24), 1 << 24, 1000) / (1 << 26)).astype(F32)
    r = fma32(a, b, c)
    for i in range(len(a)):
        x = Fraction(float(a[i])) * Fraction(float(b[i])) + Fraction(float(c[i]))
        cand = F32(float(x))
        best = None
        for v in (np.nextafter(cand, F32(-np.inf)), cand, np.nextafter(cand, F32(np.inf))):
            d = abs(Fraction(float(v)) - x)
            even = (int(np.asarray(v).view(np.uint32)) & 1) == 0
            if best is None or d < best[0] or (d == best[0] and even):
                best = (d, v)
        assert r[i] == best[1], (a[i], b[i], c[i], r[i], best[1])


@pytest.mark.parametrize("every", [1, 8])
def test_upper_bound_exit_keeps_gamma(every):
    """The GPU count sweeps' early exit at count + samples left < k_out
    (merge.cu sweep_rows / long_count_sync) reaches the same gamma* as the
    plain procedure, on random rays of every kind and several k_out."""
    rng = np.random.default_rng(77 + every)
    for kind in ("plain", "gappy", "dyadic"):
        rays = [random_ray(rng, kind) for _ in range(800)]
        samples = [depth_order(l) for l in rays]
        m = np.array([len(x) for x in samples], np.int64)
        S = np.zeros((len(samples), max(1, int(m.max())), 6), F32)
        for r, x in enumerate(samples):
            S[r, :len(x)] = x
        for k in (1, 3, 8, 20):
            g0 = bisect(S, m, k)
            g1 = bisect_ub(S, m, k, every=every)
            sel = m > k
            assert sel.any()
            assert np.array_equal(g0[sel], g1[sel]), (kind, k, np.nonzero(g0[sel] != g1[sel])[0][:5])


def test_memoised_bisection_keeps_gamma():
    """The GPU's memoised bisection (a midpoint inside the validity interval of
    the latest sweep on either side of the bracket reuses that sweep's count)
    reaches the plain procedure's gamma* on random rays, and skips sweeps."""
    rng = np.random.default_rng(91)
    swept = evaluated = 0
    for kind in ("plain", "gappy", "dyadic"):
        rays = [random_ray(rng, kind) for _ in range(800)]
        samples = [depth_order(l) for l in rays]
        m = np.array([len(x) for x in samples], np.int64)
        S = np.zeros((len(samples), max(1, int(m.max())), 6), F32)
        for r, x in enumerate(samples):
            S[r, :len(x)] = x
        for k in (1, 3, 8, 20):
            sel = m > k
            g0 = bisect(S, m, k)
            g1, sweeps, levels = bisect_memo(S, m, k)
            assert np.array_equal(g0[sel], g1[sel]), (kind, k, np.nonzero(g0[sel] != g1[sel])[0][:5])
            swept += sweeps
            evaluated += levels
    assert swept < 0.95 * evaluated, (swept, evaluated)  # the memo does resolve levels
