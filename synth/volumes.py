"""Procedural scalar fields shaped like the paper's datasets (Table 2,
PAPER.md:225-237): a Kingsnake-like u8 field (KS, 1024x1024x795) and a
Rayleigh-Taylor-like u16 mixing layer (RT, 512^3 / 1024^3), plus the 64^3
two-shell test scene.  Generated with torch on any device,
z-slab by z-slab; x-fastest layout [z][y][x].  Recipes: DESIGN.md §4.
"""
from __future__ import annotations

import math

import numpy as np
import torch


def _hash01(ix, iy, iz, seed: int):
    """Integer lattice hash -> float in [0,1) (value noise lattice)."""
    h = (ix * 73856093) ^ (iy * 19349663) ^ (iz * 83492791) ^ (seed * 2654435761)
    h = h & 0xFFFFFFFF
    h = (h ^ (h >> 13)) * 1274126177 & 0xFFFFFFFF
    h = h ^ (h >> 16)
    return (h & 0xFFFFFF).to(torch.float32) / float(1 << 24)


def _value_noise(x, y, z, freq: float, seed: int):
    """Trilinear value noise with smoothstep weights, in [-1, 1]."""
    fx, fy, fz = x * freq, y * freq, z * freq
    ix, iy, iz = torch.floor(fx), torch.floor(fy), torch.floor(fz)
    tx, ty, tz = fx - ix, fy - iy, fz - iz
    tx, ty, tz = tx * tx * (3 - 2 * tx), ty * ty * (3 - 2 * ty), tz * tz * (3 - 2 * tz)
    ix, iy, iz = ix.long(), iy.long(), iz.long()
    acc = 0.0
    for dz in (0, 1):
        wz = tz if dz else 1 - tz
        for dy in (0, 1):
            wy = ty if dy else 1 - ty
            for dx in (0, 1):
                wx = tx if dx else 1 - tx
                acc = acc + wx * wy * wz * _hash01(ix + dx, iy + dy, iz + dz, seed)
    return acc * 2 - 1


def two_shell(n: int = 64, device="cpu") -> torch.Tensor:
    """Two nested spherical shells: u8 [n][n][n]."""
    c = (torch.arange(n, device=device, dtype=torch.float32) + 0.5) / n - 0.5
    z, y, x = torch.meshgrid(c, c, c, indexing="ij")
    r = torch.sqrt(x * x + y * y + z * z)
    v = torch.zeros_like(r)
    v = torch.where((r - 0.40).abs() < 0.035, torch.full_like(r, 0.55), v)
    v = torch.where((r - 0.22).abs() < 0.045, torch.full_like(r, 0.85), v)
    v = v + 0.05 * (x + 0.5)  # gentle gradient so shells are not homogeneous
    return (v.clamp(0, 1) * 255).round().to(torch.uint8)


def ks_like(dims=(1024, 1024, 795), seed: int = 1, device="cpu") -> torch.Tensor:
    """Kingsnake-like u8 field [dz][dy][dx]: mostly empty, bone dominated.

    A coiled tube (Archimedean spiral, 2.5 turns in xy, z-wobble +-6 %, radius
    ~36 voxels at 1024) with soft tissue ~70, a skin shell ~120, vertebra
    ellipsoids ~220 every ~20 voxels of arc and thin rib rings ~200, over
    value noise < 30 (transparent under the KS transfer function).
    """
    dx, dy, dz = dims
    md = max(dims)
    vox = 1.0 / md  # world units per voxel (isotropic)
    out = torch.empty((dz, dy, dx), dtype=torch.uint8, device=device)
    xs = (torch.arange(dx, device=device, dtype=torch.float32) + 0.5) * vox
    ys = (torch.arange(dy, device=device, dtype=torch.float32) + 0.5) * vox
    cx, cy, cz = dx * vox / 2, dy * vox / 2, dz * vox / 2
    turns = 2.5
    th_max = 2 * math.pi * turns
    r0, r1 = 0.08 * dx * vox, 0.42 * dx * vox
    b = (r1 - r0) / th_max
    Rt = 36.0 * vox * (md / 1024.0)  # tube radius: 36 voxels of a 1024 grid, in world units
    skin = 2.5 * vox * (md / 1024.0)
    spacing = 20.0 * vox * (md / 1024.0)
    Y, X = torch.meshgrid(ys, xs, indexing="ij")
    px, py = X - cx, Y - cy
    rho = torch.sqrt(px * px + py * py)
    phi = torch.atan2(py, px) % (2 * math.pi)
    slab = max(1, (1 << 24) // (dx * dy))
    for z0 in range(0, dz, slab):
        z1 = min(dz, z0 + slab)
        zs = (torch.arange(z0, z1, device=device, dtype=torch.float32) + 0.5) * vox
        Z = zs[:, None, None]
        best = torch.full((z1 - z0, dy, dx), 1e9, device=device)
        best_th = torch.zeros_like(best)
        for j in range(int(math.ceil(turns)) + 1):
            th = phi + 2 * math.pi * j
            valid = th <= th_max
            R = r0 + b * th
            zc = cz + 0.06 * dz * vox * torch.sin(3 * th)
            d = torch.sqrt((rho - R)[None] ** 2 + (Z - zc[None]) ** 2)
            d = torch.where(valid[None], d, torch.full_like(d, 1e9))
            take = d < best
            best = torch.where(take, d, best)
            best_th = torch.where(take, th[None].expand_as(best), best_th)
        arc = r0 * best_th + 0.5 * b * best_th * best_th
        local = torch.remainder(arc, spacing) - spacing / 2
        v = torch.zeros_like(best)
        v = torch.where(best < Rt - skin, torch.full_like(v, 70.0), v)
        v = torch.where((best - Rt).abs() < skin, torch.full_like(v, 120.0), v)
        rib = (local.abs() < 1.5 * vox) & ((best - 0.75 * Rt).abs() < 1.5 * vox)
        v = torch.where(rib, torch.full_like(v, 200.0), v)
        vert = (local / (0.4 * spacing)) ** 2 + (best / (0.45 * Rt)) ** 2 < 1.0
        v = torch.where(vert, torch.full_like(v, 220.0), v)
        iz = torch.arange(z0, z1, device=device)[:, None, None]
        iy = torch.arange(dy, device=device)[None, :, None]
        ix = torch.arange(dx, device=device)[None, None, :]
        noise = _hash01(ix, iy, iz, seed) * 29.0
        v = torch.where(v > 0, v, noise)
        out[z0:z1] = v.clamp(0, 255).round().to(torch.uint8)
    return out


def rt_like(dims=(512, 512, 512), seed: int = 2, device="cpu") -> torch.Tensor:
    """Rayleigh-Taylor-like u16 mixing layer [dz][dy][dx]:
    rho = 1/2 (1 + tanh((z - 0.5 - 0.12 h(x,y) - 0.04 fbm(x,y,z)) / 0.015)),
    h = sum_12 a_j sin(2 pi k_j.(x,y) + phi_j), |k_j| in [2,16], a_j ~ 1/|k_j|,
    fbm = 5 octaves of hashed value noise.  Returned as int16
    holding the u16 bit patterns (consumers read the buffer as uint16)."""
    dx, dy, dz = dims
    rng = np.random.Generator(np.random.PCG64(seed))
    kmag = rng.uniform(2, 16, 12)
    kang = rng.uniform(0, 2 * math.pi, 12)
    ph = rng.uniform(0, 2 * math.pi, 12)
    amp = 1.0 / kmag
    amp = amp / amp.sum()
    out = torch.empty((dz, dy, dx), dtype=torch.int32, device=device)
    xs = (torch.arange(dx, device=device, dtype=torch.float32) + 0.5) / dx
    ys = (torch.arange(dy, device=device, dtype=torch.float32) + 0.5) / dy
    Y, X = torch.meshgrid(ys, xs, indexing="ij")
    h = torch.zeros_like(X)
    for j in range(12):
        kx, ky = kmag[j] * math.cos(kang[j]), kmag[j] * math.sin(kang[j])
        h = h + float(amp[j]) * torch.sin(2 * math.pi * (kx * X + ky * Y) + float(ph[j]))
    slab = max(1, (1 << 23) // (dx * dy))
    for z0 in range(0, dz, slab):
        z1 = min(dz, z0 + slab)
        zs = (torch.arange(z0, z1, device=device, dtype=torch.float32) + 0.5) / dz
        Z = zs[:, None, None].expand(z1 - z0, dy, dx)
        Xe, Ye = X[None].expand_as(Z), Y[None].expand_as(Z)
        fbm = torch.zeros_like(Z)
        amp_o, freq = 0.5, 4.0
        for o in range(5):
            fbm = fbm + amp_o * _value_noise(Xe, Ye, Z, freq, seed * 131 + o)
            amp_o *= 0.5
            freq *= 2.0
        rho = 0.5 * (1 + torch.tanh((Z - 0.5 - 0.12 * h[None] - 0.04 * fbm) / 0.015))
        out[z0:z1] = (rho.clamp(0, 1) * 65535).round().to(torch.int32)
    # u16 values stored bit-exactly in an int16 tensor (torch has no full uint16 support)
    return torch.where(out >= 32768, out - 65536, out).to(torch.int16)
