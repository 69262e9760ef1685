"""Edge cases of the merge on the GPU against the oracle, element by element
(ties included): a one-list image (P = 1: only a ragged tail group), tiny
ragged images, lists of exactly k_out and k_out + 1 samples (the boundary
between pass-through and the gamma search, PAPER.md:176 / Q9), k_in = k_out
= 1 with many PEs, a single full-length list among empty ones, and the
loopback group on a strip of one row per rank (G = H)."""
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


def _check(vdi, orc, pes, W, H, k_in, k_out, where):
    ref = orc.composite(pes, W, H, 1, k_out)
    comp = vdi.Compositor(W, H, k_in, k_out, len(pes))
    strip = comp.empty_strip()
    comp.composite([dense_to_device(p, i) for i, p in enumerate(pes)], strip)
    torch.cuda.synchronize()
    compare(*full_to_numpy(strip), ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], where)
    comp.close()
    return ref


@pytest.mark.parametrize("W,H,n,k_in,k_out,lam", [
    (1, 1, 4, 8, 4, 30.0),      # one list: the whole image is a tail group
    (3, 2, 5, 6, 3, 20.0),      # P = 6
    (33, 1, 3, 10, 5, 12.0),    # one full group + a one-list tail
    (7, 9, 16, 1, 1, 6.0),      # k_in = k_out = 1, many PEs
    (31, 17, 2, 40, 40, 60.0),  # m up to 80 > k_out = 40: long lists, k_out at the bucket edge
])
def test_tiny_and_ragged(vdi, orc, W, H, n, k_in, k_out, lam):
    pes = synth.random_subvdis(n, W, H, k_in, lam=lam, seed=W * 100 + H, mask="full")
    ref = _check(vdi, orc, pes, W, H, k_in, k_out, f"{W}x{H} n{n} k{k_in}-{k_out}")
    assert ref["count"].max() > 0


def _exact_m_pes(n, W, H, m_of, seed):
    """n PEs whose lists hold m_of(p) samples in total (split over the PEs in
    disjoint depth runs, alternating owners)."""
    rng = np.random.default_rng(seed)
    P = W * H
    per = [[] for _ in range(n)]
    counts = np.zeros((n, P), np.uint8)
    for p in range(P):
        m = m_of(p)
        t = np.float32(1.0)
        for j in range(m):
            s = j % n
            a = np.float32(rng.uniform(0.05, 0.9))
            rgb = (rng.random(3) * a).astype(np.float32)
            per[s].append((p, [t, np.float32(t + 0.01)] + list(rgb) + [a]))
            t = np.float32(t + 0.02)
            counts[s, p] += 1
    pes = []
    for s in range(n):
        recs = sorted(per[s], key=lambda x: x[0])  # list-major, front-to-back within a list
        arr = np.array([r[1] for r in recs], np.float32).reshape(-1, 6)
        pes.append({"count": counts[s], "depth": np.ascontiguousarray(arr[:, :2]),
                    "rgba": np.ascontiguousarray(arr[:, 2:])})
    return pes


@pytest.mark.parametrize("k_out", [4, 20, 32])
def test_m_at_the_pass_through_boundary(vdi, orc, k_out):
    """Lists of exactly k_out samples pass through verbatim (Q9); lists of
    k_out + 1 and 2 k_out samples take the gamma search."""
    W, H, n = 40, 3, 4
    ms = [k_out, k_out + 1, 2 * k_out]
    pes = _exact_m_pes(n, W, H, lambda p: ms[p % 3], seed=k_out)
    k_in = max(int(p["count"].max()) for p in pes)
    ref = _check(vdi, orc, pes, W, H, k_in, k_out, f"boundary k{k_out}")
    assert (ref["count"][0::3] == k_out).all()


def test_one_long_list_among_empty(vdi, orc):
    W, H, n, k_out = 64, 4, 8, 8
    pes = _exact_m_pes(n, W, H, lambda p: 8 * 20 if p == 77 else 0, seed=3)
    ref = _check(vdi, orc, pes, W, H, 20, k_out, "one long list")
    assert ref["count"][77] > 0 and ref["count"].sum() == ref["count"][77]


def test_loopback_one_row_per_rank(vdi, orc):
    """G = H: every rank's strip is a single image row (ragged: W = 45)."""
    W, H, n, G, k_in, k_out = 45, 3, 4, 3, 10, 6
    pes_np = synth.random_subvdis(n, W, H, k_in, lam=15.0, seed=9, mask="full")
    ref = orc.composite(pes_np, W, H, 1, k_out)
    key = os.urandom(128)
    comps = [vdi.Compositor(W, H, k_in, k_out, n, n_ranks=G, rank=r, unique_id=key,
                            flags=vdi._lib.VDI_FLAG_LOOPBACK, stream=torch.cuda.Stream()) for r in range(G)]
    pes = [dense_to_device(p, i) for i, p in enumerate(pes_np)]
    image = vdi.FullVDI.empty(W, 0, H, k_out)
    strips = [c.empty_strip() for c in comps]
    torch.cuda.synchronize()
    errs = []

    def rank(r):
        try:
            mine = [p for p in pes if vdi.pe_home(n, G, p.pe_id) == r]
            comps[r].composite(mine, strips[r])
            comps[r].gather(strips[r], image if r == 0 else None)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    assert not errs, errs
    torch.cuda.synchronize()
    compare(*full_to_numpy(image), ref["count"], ref["depth"], ref["rgba"], ref["stats"]["margin"], "G = H")
    for c in comps:
        c.close()
