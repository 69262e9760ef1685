"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NONE of the method's arithmetic (no tau, no gamma search,
no over-compositing, no sorting of supersegments): only the scene description
the paper's workloads are shaped like (volumes, transfer functions, cameras,
domain decompositions) and the merge-only microbench's random sub-VDIs.
Both `oracle/` and `paper_2206_14503_b200/` consume its outputs; neither
side's results ever feed back into it.  Recipes: DESIGN.md §4.
"""
from .scene import (Camera, Decomposition, make_camera, slab_decomposition, grid_decomposition,
                    interleaved_decomposition, tf_table)
from .volumes import two_shell, ks_like, rt_like
from .subvdi import random_subvdis
from .configs import CONFIGS, Config, config_by_name, make_volume

__all__ = [
    "Camera", "Decomposition", "make_camera", "slab_decomposition", "grid_decomposition",
    "interleaved_decomposition", "tf_table", "two_shell", "ks_like", "rt_like", "random_subvdis",
    "CONFIGS", "Config", "config_by_name", "make_volume",
]
