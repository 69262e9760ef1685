"""Cameras, transfer-function tables and domain decompositions (scene inputs).

Geometry convention: the volume's world box has longest side 1
and is centred at the origin; voxel (i, j, k) covers continuous voxel
coordinates [i, i+1) x [j, j+1) x [k, k+1).  The camera is a pinhole at
distance 1.8 from the centre looking at it, vfov 40 deg; V0
looks along -z (perpendicular to z-slabs, the worst case of PAPER.md:381),
V1 is rotated 90 deg about y.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class Camera:
    eye: tuple
    fwd: tuple
    right: tuple
    up: tuple
    tan_x: float   # tan(vfov/2) * aspect
    tan_y: float   # tan(vfov/2)
    W: int
    H: int

    def as_f32(self):
        f = lambda v: tuple(float(np.float32(x)) for x in v)
        return dataclasses.replace(self, eye=f(self.eye), fwd=f(self.fwd), right=f(self.right),
                                   up=f(self.up), tan_x=float(np.float32(self.tan_x)),
                                   tan_y=float(np.float32(self.tan_y)))


def make_camera(W: int, H: int, view: int = 0, angle_deg: float = 0.0, dist: float = 1.8,
                vfov_deg: float = 40.0) -> Camera:
    """Orbit camera about the y axis: azimuth = 90*view + angle_deg degrees."""
    az = math.radians(90.0 * view + angle_deg)
    eye = np.array([dist * math.sin(az), 0.0, dist * math.cos(az)])
    fwd = -eye / np.linalg.norm(eye)
    up0 = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up0)
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    th = math.tan(math.radians(vfov_deg) / 2)
    return Camera(tuple(eye), tuple(fwd), tuple(right), tuple(up), th * W / H, th, W, H).as_f32()


@dataclasses.dataclass(frozen=True)
class Decomposition:
    """Axis-aligned brick grid: per-axis voxel boundaries and an owner table.

    Brick (bx, by, bz) covers voxels [xb[bx], xb[bx+1]) x ... (half-open,
    SPEC.md:113) and belongs to PE owner[(bz*gy + by)*gx + bx].
    """
    xb: np.ndarray
    yb: np.ndarray
    zb: np.ndarray
    owner: np.ndarray
    n_pes: int

    @property
    def grid(self):
        return len(self.xb) - 1, len(self.yb) - 1, len(self.zb) - 1


def _split(n: int, k: int) -> np.ndarray:
    # balanced contiguous split, thicker pieces first: 10,4 -> 3,3,2,2
    base, extra = divmod(n, k)
    sizes = [base + (1 if i < extra else 0) for i in range(k)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)


def slab_decomposition(dims, n_pes: int) -> Decomposition:
    """Equal z-slabs, one per PE."""
    dx, dy, dz = dims
    if n_pes > dz:
        raise ValueError("more slabs than z voxels")
    return Decomposition(np.array([0, dx], np.int32), np.array([0, dy], np.int32), _split(dz, n_pes),
                         np.arange(n_pes, dtype=np.int32), n_pes)


def grid_decomposition(dims, g=(2, 2, 2)) -> Decomposition:
    """gx x gy x gz bricks, PE id = brick id (config C3: 2x2x2)."""
    n = g[0] * g[1] * g[2]
    return Decomposition(_split(dims[0], g[0]), _split(dims[1], g[1]), _split(dims[2], g[2]),
                         np.arange(n, dtype=np.int32), n)


def interleaved_decomposition(dims, n_pes: int, g=(8, 8, 8), seed: int = 3) -> Decomposition:
    """Non-convex decomposition: g bricks, balanced seeded random
    assignment (Fisher-Yates with numpy's PCG64, seed 3), equal bricks per PE."""
    nb = g[0] * g[1] * g[2]
    if nb % n_pes:
        raise ValueError("bricks must divide evenly among PEs")
    owner = np.repeat(np.arange(n_pes, dtype=np.int32), nb // n_pes)
    np.random.Generator(np.random.PCG64(seed)).shuffle(owner)
    return Decomposition(_split(dims[0], g[0]), _split(dims[1], g[1]), _split(dims[2], g[2]), owner, n_pes)


def tf_table(kind: str, opacity_scale: float = 1.0) -> np.ndarray:
    """256 x RGBA float32 transfer-function table (non-premultiplied), built by
    piecewise-linear interpolation of control points."""
    if kind == "ks":      # KS-like: transparent below 0.16, faint soft tissue, opaque-ish bone
        pts = [(0.00, (0, 0, 0), 0.0), (0.16, (0, 0, 0), 0.0), (0.20, (0.80, 0.45, 0.35), 0.010),
               (0.30, (0.85, 0.50, 0.40), 0.020), (0.42, (0.90, 0.70, 0.55), 0.050),
               (0.55, (0.95, 0.85, 0.70), 0.080), (0.70, (0.98, 0.95, 0.90), 0.40),
               (0.85, (1.00, 1.00, 0.97), 0.75), (1.00, (1.00, 1.00, 1.00), 0.85)]
    elif kind == "rt":    # RT-like: light fluid transparent, mixing band blue->white->orange
        pts = [(0.00, (0, 0, 0), 0.0), (0.06, (0.10, 0.20, 0.90), 0.0), (0.20, (0.15, 0.35, 0.95), 0.03),
               (0.40, (0.60, 0.75, 1.00), 0.06), (0.55, (1.00, 1.00, 1.00), 0.08),
               (0.75, (1.00, 0.65, 0.20), 0.06), (0.94, (0.95, 0.45, 0.10), 0.02),
               (1.00, (0.90, 0.40, 0.10), 0.004)]
    elif kind == "shell":  # two-shell test scene
        pts = [(0.00, (0, 0, 0), 0.0), (0.25, (0, 0, 0), 0.0), (0.40, (0.2, 0.6, 1.0), 0.15),
               (0.60, (1.0, 0.9, 0.2), 0.35), (0.80, (1.0, 0.3, 0.1), 0.60), (1.00, (1.0, 1.0, 1.0), 0.9)]
    else:
        raise ValueError(kind)
    xs = np.array([p[0] for p in pts])
    cols = np.array([p[1] for p in pts], dtype=np.float64)
    al = np.array([p[2] for p in pts], dtype=np.float64) * opacity_scale
    x = np.arange(256) / 255.0
    tab = np.zeros((256, 4), np.float64)
    for c in range(3):
        tab[:, c] = np.interp(x, xs, cols[:, c])
    tab[:, 3] = np.clip(np.interp(x, xs, al), 0.0, 1.0)
    return tab.astype(np.float32)
