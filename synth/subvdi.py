"""Merge-only microbench inputs: random dense sub-VDIs (no raycast).

Recipe (SURVEY §8(d) "merge-only microbench", seed 7):
  * the ray's depth range [1, 2) is cut into 2n equal domain intervals; pixel p
    rotates their ownership by a random shift, so every PE owns two disjoint
    intervals per ray (a non-convex decomposition);
  * each domain interval holds k_in slots; PE s occupies each of its 2 k_in
    slots with probability q(p) = lam * mask(p) / (2 k_in), keeping at most
    k_in (c_s(p) ~ min(k_in, Binomial(2 k_in, q))); mask is a radial image
    profile (1 at the centre, 0 outside a disc of radius 0.48 W);
  * a record covers its whole slot, so adjacent occupied slots abut (gaps only
    where slots are empty); alpha ~ U(0.01, 0.9), rgb = alpha * U(0,1)^3;
  * overlap=True shifts every (list, PE) run by up to +-0.6 slot so records of
    different PEs overlap while each PE's run stays front-to-back sorted
     -- exercises step 2, subdivision.
Per-PE output: count u8[P], depth f32[S,2] (tf, tb), rgba f32[S,4], pixel-major,
front-to-back within a pixel (the dense layout of PAPER.md:113-115).
"""
from __future__ import annotations

import numpy as np


def random_subvdis(n_pes: int, W: int, H: int, k_in: int, lam: float = 8.0, seed: int = 7,
                   overlap: bool = False, mask: str = "disc"):
    rng = np.random.Generator(np.random.PCG64(seed))
    P = W * H
    U = 2 * k_in
    n_int = 2 * n_pes
    w = np.float32(1.0) / np.float32(n_int * k_in)
    ys, xs = np.divmod(np.arange(P, dtype=np.int64), W)
    if mask == "disc":
        r = np.hypot((xs + 0.5) / W - 0.5, ((ys + 0.5) / H - 0.5) * H / W)
        mk = np.clip(1.0 - r / 0.48, 0.0, 1.0)
    else:
        mk = np.ones(P)
    q = np.clip(lam * mk / U, 0.0, 1.0).astype(np.float32)
    shift = rng.integers(0, n_pes, P)
    out = []
    for s in range(n_pes):
        occ = rng.random((P, U), dtype=np.float32) < q[:, None]
        occ &= np.cumsum(occ, axis=1) <= k_in
        count = occ.sum(axis=1).astype(np.uint8)
        p_idx, u_idx = np.nonzero(occ)                       # pixel-major, slot-ascending
        j0 = (s - shift[p_idx]) % n_pes                      # PE s's first domain interval
        j = j0 + (u_idx // k_in) * n_pes                     # first or second interval
        slot = j * k_in + (u_idx % k_in)
        tf = np.float32(1.0) + slot.astype(np.float32) * w
        tb = np.float32(1.0) + (slot + 1).astype(np.float32) * w
        if overlap:  # one shift per (list, PE): runs stay sorted, PEs overlap
            jit = ((rng.random(P, dtype=np.float32) - np.float32(0.5)) * np.float32(1.2) * w)[p_idx]
            tf = tf + jit
            tb = tb + jit
        a = rng.uniform(0.01, 0.9, len(tf)).astype(np.float32)
        rgb = rng.random((len(tf), 3), dtype=np.float32) * a[:, None]
        depth = np.stack([tf, tb], axis=1).astype(np.float32)
        rgba = np.concatenate([rgb, a[:, None]], axis=1).astype(np.float32)
        out.append({"count": count, "depth": np.ascontiguousarray(depth),
                    "rgba": np.ascontiguousarray(rgba)})
    return out
