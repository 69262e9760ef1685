"""paper_2206_14503_b200 — B200-native sort-last parallel compositing of
Volumetric Depth Images (arXiv 2206.14503).

The product is libvdi.so (CUDA sm_100a + NCCL, C ABI in include/vdi.h);
this package is its thin Python binding.  See DESIGN.md.
"""
from . import _lib
from .api import (Compositor, DenseSubVDI, FullVDI, full_bytes, get_unique_id, pe_home, strip_rows)

__all__ = ["Compositor", "DenseSubVDI", "FullVDI", "full_bytes", "get_unique_id", "pe_home", "strip_rows", "_lib"]
