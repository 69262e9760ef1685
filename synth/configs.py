"""The five BASELINE.json configurations as concrete synthetic scenes
(SURVEY §8(d) table).  A config names the volume, transfer function,
decomposition, image size and budgets; nothing here computes the method."""
from __future__ import annotations

import dataclasses

from .scene import grid_decomposition, interleaved_decomposition, slab_decomposition


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n_pes: int
    W: int
    H: int
    k_in: int
    k_out: int
    volume: str          # "shell" | "ks" | "rt"
    dims: tuple
    decomp: str          # "slab" | "grid" | "interleaved"
    tf: str
    tf_scale: float = 1.0
    desc: str = ""

    def decomposition(self):
        if self.decomp == "slab":
            return slab_decomposition(self.dims, self.n_pes)
        if self.decomp == "grid":
            return grid_decomposition(self.dims, (2, 2, 2))
        if self.decomp == "interleaved":
            return interleaved_decomposition(self.dims, self.n_pes, (8, 8, 8), seed=3)
        raise ValueError(self.decomp)


CONFIGS = {
    "C1": Config("C1", 2, 64, 64, 4, 4, "shell", (64, 64, 64), "slab", "shell",
                 desc="2 PEs, 64x64, k_in=k_out=4, 64^3 two-shell field, 2 z-slabs"),
    "C2": Config("C2", 4, 1280, 720, 20, 20, "rt", (512, 512, 512), "slab", "rt",
                 desc="4 PEs, 1280x720, k=20, RT-like 512^3, 4 z-slabs"),
    "C3": Config("C3", 8, 1920, 1080, 20, 20, "ks", (1024, 1024, 795), "grid", "ks",
                 desc="8 PEs, 1920x1080, k=20, KS-like 1024x1024x795, 2x2x2 grid"),
    "C4": Config("C4", 8, 1920, 1080, 20, 20, "ks", (1024, 1024, 795), "interleaved", "ks",
                 desc="8 PEs, 1920x1080, k=20, KS-like, non-convex interleaved 8x8x8 bricks"),
    "C5": Config("C5", 8, 3840, 2160, 32, 32, "rt", (1024, 1024, 1024), "slab", "rt",
                 desc="3840x2160, k=32, RT-like 1024^3, n z-slabs (n = 2/4/8/16)"),
}


def config_by_name(name: str, **over) -> Config:
    c = CONFIGS[name]
    return dataclasses.replace(c, **over) if over else c


def make_volume(cfg: Config, device="cpu"):
    """The config's scalar field as a torch tensor [dz][dy][dx] (u8, or u16 bits in int16)."""
    from .volumes import ks_like, rt_like, two_shell
    if cfg.volume == "shell":
        return two_shell(cfg.dims[0], device=device)
    if cfg.volume == "ks":
        return ks_like(cfg.dims, seed=1, device=device)
    if cfg.volume == "rt":
        return rt_like(cfg.dims, seed=2, device=device)
    raise ValueError(cfg.volume)
