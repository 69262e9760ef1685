"""ctypes binding of libvdi (include/vdi.h): argument marshalling only.

Every compositing step runs in libvdi's CUDA kernels; this module only
declares the C structs and function signatures with the header's names.
Loading fails loudly (ImportError) when the built library is missing: there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# VDI_LIB_PATH selects another in-tree build (A/B experiments); default lib/libvdi.so
LIB_PATH = os.environ.get("VDI_LIB_PATH") or os.path.join(_HERE, "lib", "libvdi.so")

VDI_OK = 0
VDI_ERR_INVALID_ARG = 1
VDI_ERR_OUT_OF_MEMORY = 2
VDI_ERR_CUDA = 3
VDI_ERR_NCCL = 4
VDI_ERR_STATE = 5
VDI_ERR_CAPACITY = 6
VDI_ERR_INTERNAL = 7
VDI_FLAG_PIXEL_STATS = 0x1
VDI_FLAG_VALIDATE = 0x2
VDI_FLAG_STAGE_TIMING = 0x4
VDI_FLAG_LOOPBACK = 0x10
VDI_FLAG_HOST_SPAN = 0x20


class vdi_config(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("k_in", C.c_uint32), ("k_out", C.c_uint32),
                ("n_pes", C.c_uint32), ("n_ranks", C.c_uint32), ("rank", C.c_uint32), ("root", C.c_uint32),
                ("max_iters", C.c_uint32), ("gamma_max", C.c_float), ("flags", C.c_uint32),
                ("nccl_unique_id", C.c_void_p), ("cuda_stream", C.c_void_p)]


class vdi_dense_strip(C.Structure):
    _fields_ = [("row_begin", C.c_uint32), ("row_end", C.c_uint32), ("capacity", C.c_uint64), ("total", C.c_uint64),
                ("count", C.c_void_p), ("depth", C.c_void_p), ("rgba", C.c_void_p)]


class vdi_dense_view(C.Structure):
    _fields_ = [("pe_id", C.c_uint32), ("total", C.c_uint64), ("count", C.c_void_p), ("offset", C.c_void_p),
                ("depth", C.c_void_p), ("rgba", C.c_void_p)]


class vdi_full_view(C.Structure):
    _fields_ = [("row_begin", C.c_uint32), ("row_end", C.c_uint32), ("count", C.c_void_p),
                ("depth", C.c_void_p), ("rgba", C.c_void_p)]


class vdi_volume_desc(C.Structure):
    _fields_ = [("voxels", C.c_void_p), ("bytes_per_voxel", C.c_uint32), ("dims", C.c_uint32 * 3)]


class vdi_tf_desc(C.Structure):
    _fields_ = [("table", C.c_void_p)]


class vdi_camera(C.Structure):
    _fields_ = [("eye", C.c_float * 3), ("fwd", C.c_float * 3), ("right", C.c_float * 3),
                ("up", C.c_float * 3), ("tan_x", C.c_float), ("tan_y", C.c_float)]


class vdi_decomp_desc(C.Structure):
    _fields_ = [("grid", C.c_uint32 * 3), ("xb", C.c_void_p), ("yb", C.c_void_p), ("zb", C.c_void_p),
                ("owner", C.c_void_p)]


class vdi_counters(C.Structure):
    _fields_ = [("records_in", C.c_uint64), ("records_search", C.c_uint64), ("searched_lists", C.c_uint64), ("bytes_sent", C.c_uint64),
                ("bytes_received", C.c_uint64), ("kernel_launches", C.c_uint32), ("ms_exchange", C.c_float),
                ("ms_merge", C.c_float), ("ms_gather", C.c_float), ("bucket_lists", C.c_uint64 * 4),
                ("general_lists", C.c_uint64), ("bytes_gather", C.c_uint64), ("fallback_groups", C.c_uint64),
                ("ms_scan", C.c_float), ("ms_fast", C.c_float), ("ms_search", C.c_float), ("sweep_steps", C.c_uint64),
                ("ms_push", C.c_float)]


# name -> (restype, argtypes) exactly as declared in include/vdi.h
SIGNATURES = {
    "vdi_version": (C.c_char_p, []),
    "vdi_status_string": (C.c_char_p, [C.c_int]),
    "vdi_last_error": (C.c_char_p, [C.c_void_p]),
    "vdi_get_unique_id": (C.c_int, [C.c_void_p]),
    "vdi_composite_init": (C.c_int, [C.POINTER(vdi_config), C.POINTER(C.c_void_p)]),
    "vdi_composite_destroy": (None, [C.c_void_p]),
    "vdi_generate_subvdi": (C.c_int, [C.c_void_p, C.POINTER(vdi_volume_desc), C.POINTER(vdi_tf_desc),
                                      C.POINTER(vdi_camera), C.POINTER(vdi_decomp_desc), C.c_uint32,
                                      C.POINTER(vdi_dense_view)]),
    "vdi_generate_limit": (C.c_int, [C.c_void_p, C.POINTER(vdi_volume_desc), C.POINTER(vdi_tf_desc),
                                     C.POINTER(vdi_camera), C.POINTER(vdi_decomp_desc), C.c_uint32,
                                     C.POINTER(vdi_dense_view)]),
    "vdi_composite": (C.c_int, [C.c_void_p, C.POINTER(vdi_dense_view), C.c_uint32, C.POINTER(vdi_full_view)]),
    "vdi_composite_image": (C.c_int, [C.c_void_p, C.POINTER(vdi_dense_view), C.c_uint32, C.c_void_p]),
    "vdi_gather_image": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vdi_render_generation_view": (C.c_int, [C.c_void_p, C.POINTER(vdi_full_view), C.c_void_p]),
    "vdi_render_novel_view": (C.c_int, [C.c_void_p, C.POINTER(vdi_full_view), C.POINTER(vdi_camera),
                                        C.POINTER(vdi_camera), C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]),
    "vdi_render_dvr": (C.c_int, [C.c_void_p, C.POINTER(vdi_volume_desc), C.POINTER(vdi_tf_desc),
                                 C.POINTER(vdi_camera), C.c_uint32, C.c_uint32, C.c_void_p]),
    "vdi_composite_host": (C.c_int, [C.c_void_p, C.POINTER(vdi_dense_view), C.c_uint32,
                                     C.POINTER(vdi_full_view)]),
    "vdi_composite_fullrep": (C.c_int, [C.c_void_p, C.POINTER(vdi_full_view), C.c_void_p, C.c_uint32,
                                        C.POINTER(vdi_full_view)]),
    "vdi_dense_to_full": (C.c_int, [C.c_void_p, C.POINTER(vdi_dense_view), C.POINTER(vdi_full_view)]),
    "vdi_composite_host_dense": (C.c_int, [C.c_void_p, C.POINTER(vdi_dense_view), C.c_uint32,
                                           C.POINTER(vdi_dense_strip)]),
    "vdi_composite_host_dense_frames": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(vdi_dense_view), C.c_uint32,
                                                  C.POINTER(vdi_dense_strip)]),
    "vdi_gather": (C.c_int, [C.c_void_p, C.POINTER(vdi_full_view), C.POINTER(vdi_full_view)]),
    "vdi_gather_root": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(vdi_full_view), C.POINTER(vdi_full_view)]),
    "vdi_composite_frames": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(vdi_dense_view), C.c_uint32,
                                       C.POINTER(vdi_full_view), C.c_void_p]),
    "vdi_pixel_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vdi_get_counters": (C.c_int, [C.c_void_p, C.POINTER(vdi_counters)]),
    "vdi_strip_rows": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint32)]),
    "vdi_pe_home": (C.c_uint32, [C.c_uint32, C.c_uint32, C.c_uint32]),
    "vdi_full_bytes": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32]),
}

_lib = None


def lib():
    """The loaded libvdi.so (raises ImportError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libvdi.so not built at {LIB_PATH}: run `make` (or __graft_entry__.build()); "
                              "there is no CPU fallback")
        l = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


class VdiError(RuntimeError):
    def __init__(self, status: int, where: str):
        l = lib()
        msg = l.vdi_status_string(status).decode()
        detail = l.vdi_last_error(None).decode()
        super().__init__(f"{where}: {msg}: {detail}")
        self.status = status


def check(status: int, where: str):
    if status != VDI_OK:
        raise VdiError(status, where)
