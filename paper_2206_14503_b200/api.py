"""Python face of libvdi: the header's calls on torch CUDA tensors.

`Compositor` owns one vdi_ctx.  Methods marshal torch tensors / numpy arrays
into the C structs of include/vdi.h and call the same-named C functions; no
compositing arithmetic happens here.  torch is used only for device memory
and streams (and torch.distributed to broadcast the NCCL id).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if isinstance(t, torch.Tensor) else t.ctypes.data


@dataclass
class DenseSubVDI:
    """A dense sub-VDI: count u8[P], offset u32[P+1] (as
    int32 bits), depth f32[S,2], rgba f32[S,4]; device or host tensors."""
    pe_id: int
    total: int
    count: torch.Tensor
    offset: torch.Tensor | None
    depth: torch.Tensor
    rgba: torch.Tensor

    def view(self) -> L.vdi_dense_view:
        return L.vdi_dense_view(self.pe_id, self.total, _ptr(self.count), _ptr(self.offset), _ptr(self.depth),
                                _ptr(self.rgba))

    def to(self, device, pin=False):
        def mv(t):
            if t is None:
                return None
            t = t.to(device)
            return t.pin_memory() if pin and t.device.type == "cpu" else t
        return DenseSubVDI(self.pe_id, self.total, mv(self.count), mv(self.offset), mv(self.depth), mv(self.rgba))


@dataclass
class FullVDI:
    """Full representation of rows [row_begin, row_end)."""
    row_begin: int
    row_end: int
    count: torch.Tensor  # u8 [rows*W]
    depth: torch.Tensor  # f32 [rows*W, k, 2]
    rgba: torch.Tensor   # f32 [rows*W, k, 4]

    def view(self) -> L.vdi_full_view:
        return L.vdi_full_view(self.row_begin, self.row_end, _ptr(self.count), _ptr(self.depth), _ptr(self.rgba))

    @staticmethod
    def empty(width, row_begin, row_end, k, device="cuda", pin=False):
        P = width * (row_end - row_begin)
        kw = dict(device=device)
        t = [torch.empty(P, dtype=torch.uint8, **kw), torch.empty((P, k, 2), dtype=torch.float32, **kw),
             torch.empty((P, k, 4), dtype=torch.float32, **kw)]
        if pin:
            t = [x.pin_memory() for x in t]
        return FullVDI(row_begin, row_end, *t)


class _CudaArray:
    """Minimal __cuda_array_interface__ holder to wrap ctx-owned memory."""

    def __init__(self, ptr, shape, typestr, owner):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}
        self._owner = owner


def _wrap(ptr, shape, typestr, owner):
    if int(np.prod(shape)) == 0 or not ptr:
        dt = {"|u1": torch.uint8, "<u4": torch.int32, "<f4": torch.float32}[typestr]
        return torch.empty(shape, dtype=dt, device="cuda")
    return torch.as_tensor(_CudaArray(ptr, shape, typestr, owner), device="cuda")


def strip_rows(height, n_ranks, g):
    b, e = C.c_uint32(), C.c_uint32()
    L.check(L.lib().vdi_strip_rows(height, n_ranks, g, C.byref(b), C.byref(e)), "vdi_strip_rows")
    return b.value, e.value


def pe_home(n_pes, n_ranks, pe):
    return L.lib().vdi_pe_home(n_pes, n_ranks, pe)


def full_bytes(width, rows, k):
    return L.lib().vdi_full_bytes(width, rows, k)


def get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    L.check(L.lib().vdi_get_unique_id(buf), "vdi_get_unique_id")
    return bytes(buf)


class Compositor:
    """One libvdi context (vdi_composite_init ... vdi_composite_destroy)."""

    def __init__(self, width, height, k_in, k_out, n_pes, n_ranks=1, rank=0, max_iters=16, gamma_max=2.0,
                 flags=0, unique_id: bytes | None = None, stream: torch.cuda.Stream | None = None, root=0):
        self.lib = L.lib()
        self.width, self.height, self.k_in, self.k_out, self.n_pes = width, height, k_in, k_out, n_pes
        self.n_ranks, self.rank, self.root = n_ranks, rank, root
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self._uid = (C.c_uint8 * 128).from_buffer_copy(unique_id) if unique_id else None
        cfg = L.vdi_config(width, height, k_in, k_out, n_pes, n_ranks, rank, root, max_iters, gamma_max, flags,
                           C.cast(self._uid, C.c_void_p) if self._uid is not None else None,
                           self.stream.cuda_stream)
        h = C.c_void_p()
        L.check(self.lib.vdi_composite_init(C.byref(cfg), C.byref(h)), "vdi_composite_init")
        self.ctx = h
        self.row_begin, self.row_end = strip_rows(height, n_ranks, rank)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.vdi_composite_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- Phase 1 (SUPPORT) ---------------------------------------------------
    @staticmethod
    def _cam(camera) -> L.vdi_camera:
        return L.vdi_camera((C.c_float * 3)(*camera.eye), (C.c_float * 3)(*camera.fwd),
                            (C.c_float * 3)(*camera.right), (C.c_float * 3)(*camera.up), camera.tan_x, camera.tan_y)

    @staticmethod
    def _vol(volume, tf_table):
        assert volume.is_cuda and tf_table.is_cuda
        dz, dy, dx = volume.shape
        vol = L.vdi_volume_desc(volume.data_ptr(), volume.element_size(), (C.c_uint32 * 3)(dx, dy, dz))
        return vol, L.vdi_tf_desc(tf_table.contiguous().data_ptr())

    def generate_subvdi(self, volume: torch.Tensor, tf_table: torch.Tensor, camera, decomposition,
                        pe_id: int, limit: bool = False) -> DenseSubVDI:
        """vdi_generate_subvdi (limit=True: vdi_generate_limit, one S~ per
        sub-domain intersection): volume [dz][dy][dx] u8 (or u16 bits in int16),
        tf_table [256,4] f32 (device), camera with eye/fwd/right/up/tan_x/tan_y,
        decomposition with xb/yb/zb/owner int arrays.  Returns tensors that
        alias ctx-owned memory (valid until the next call for this pe_id)."""
        vol, tf = self._vol(volume, tf_table)
        cam = self._cam(camera)
        xb = np.ascontiguousarray(decomposition.xb, np.int32)
        yb = np.ascontiguousarray(decomposition.yb, np.int32)
        zb = np.ascontiguousarray(decomposition.zb, np.int32)
        ow = np.ascontiguousarray(decomposition.owner, np.int32)
        dec = L.vdi_decomp_desc((C.c_uint32 * 3)(len(xb) - 1, len(yb) - 1, len(zb) - 1), xb.ctypes.data,
                                yb.ctypes.data, zb.ctypes.data, ow.ctypes.data)
        out = L.vdi_dense_view()
        fn = self.lib.vdi_generate_limit if limit else self.lib.vdi_generate_subvdi
        L.check(fn(self.ctx, C.byref(vol), C.byref(tf), C.byref(cam), C.byref(dec), pe_id, C.byref(out)),
                "vdi_generate_limit" if limit else "vdi_generate_subvdi")
        P = self.width * self.height
        S = int(out.total)
        return DenseSubVDI(pe_id, S, _wrap(out.count, (P,), "|u1", self), _wrap(out.offset, (P + 1,), "<u4", self),
                           _wrap(out.depth, (S, 2), "<f4", self), _wrap(out.rgba, (S, 4), "<f4", self))

    # -- Phase 2: the hot path ------------------------------------------------
    def empty_strip(self, device="cuda", pin=False) -> FullVDI:
        return FullVDI.empty(self.width, self.row_begin, self.row_end, self.k_out, device, pin)

    def composite(self, local_pes, strip: FullVDI) -> FullVDI:
        """vdi_composite (device buffers)."""
        views = (L.vdi_dense_view * max(1, len(local_pes)))(*[p.view() for p in local_pes])
        sv = strip.view()
        L.check(self.lib.vdi_composite(self.ctx, views, len(local_pes), C.byref(sv)), "vdi_composite")
        return strip

    def composite_frames(self, frames_local_pes, images, roots=None):
        """vdi_composite_frames: frames_local_pes[f] = the PEs of frame f homed
        here; images[f] = FullVDI of rows [0, H) on the root of frame f (None
        elsewhere); roots[f] (None: the config's root for every frame)."""
        F = len(frames_local_pes)
        nl = len(frames_local_pes[0]) if F else 0
        if any(len(fr) != nl for fr in frames_local_pes) or len(images) != F:
            raise ValueError("every frame needs the same number of local PEs and one image slot")
        flat = [p.view() for fr in frames_local_pes for p in fr]
        views = (L.vdi_dense_view * max(1, len(flat)))(*flat)
        ims = (L.vdi_full_view * max(1, F))(*[im.view() if im is not None else L.vdi_full_view() for im in images])
        rs = (C.c_uint32 * max(1, F))(*roots) if roots is not None else None
        L.check(self.lib.vdi_composite_frames(self.ctx, F, views, nl, ims, C.cast(rs, C.c_void_p) if rs is not None
                                              else None), "vdi_composite_frames")
        return images

    def dense_to_full(self, pe: DenseSubVDI) -> FullVDI:
        """vdi_dense_to_full: the sub-VDI in the full representation (k_in slots)."""
        out = FullVDI.empty(self.width, 0, self.height, self.k_in)
        dv, fv = pe.view(), out.view()
        L.check(self.lib.vdi_dense_to_full(self.ctx, C.byref(dv), C.byref(fv)), "vdi_dense_to_full")
        return out

    def composite_fullrep(self, local_full, pe_ids, strip: FullVDI) -> FullVDI:
        """vdi_composite_fullrep: local_full[l] = full representation (rows
        [0, H), k_in slots) of PE pe_ids[l]."""
        views = (L.vdi_full_view * max(1, len(local_full)))(*[f.view() for f in local_full])
        ids = (C.c_uint32 * max(1, len(pe_ids)))(*pe_ids)
        sv = strip.view()
        L.check(self.lib.vdi_composite_fullrep(self.ctx, views, C.cast(ids, C.c_void_p), len(local_full),
                                               C.byref(sv)), "vdi_composite_fullrep")
        return strip

    def composite_host(self, local_pes, strip: FullVDI) -> FullVDI:
        """vdi_composite_host (host buffers; H2D + composite + D2H)."""
        views = self._host_views(local_pes)
        sv = strip.view()
        L.check(self.lib.vdi_composite_host(self.ctx, views, len(local_pes), C.byref(sv)), "vdi_composite_host")
        return strip

    def _dense_out(self, count, depth, rgba) -> L.vdi_dense_strip:
        P = (self.row_end - self.row_begin) * self.width
        for t, dt, w in ((count, torch.uint8, None), (depth, torch.float32, 2), (rgba, torch.float32, 4)):
            if t.device.type != "cpu" or t.dtype != dt or not t.is_contiguous():
                raise ValueError("dense outputs must be contiguous host tensors (u8 counts, f32 depth/rgba)")
            if w is not None and (t.dim() != 2 or t.shape[1] != w):
                raise ValueError(f"depth/rgba must be [capacity, {w}]")
        if count.numel() != P:
            raise ValueError(f"count must hold rows*W = {P} entries")
        cap = min(depth.shape[0], rgba.shape[0])
        return L.vdi_dense_strip(self.row_begin, self.row_end, cap, 0, _ptr(count), _ptr(depth), _ptr(rgba))

    @staticmethod
    def _host_views(local_pes):
        for p in local_pes:
            for t in (p.count, p.depth, p.rgba):
                if t.device.type != "cpu" or not t.is_contiguous():
                    raise ValueError("host entry points take contiguous host tensors")
        return (L.vdi_dense_view * max(1, len(local_pes)))(*[p.view() for p in local_pes])

    def composite_host_dense(self, local_pes, count, depth, rgba) -> int:
        """vdi_composite_host_dense: host sub-VDIs in, the composited strip out
        in the dense representation into host tensors count u8[rows*W],
        depth f32[cap,2], rgba f32[cap,4].  Returns the supersegment total."""
        views = self._host_views(local_pes)
        out = self._dense_out(count, depth, rgba)
        L.check(self.lib.vdi_composite_host_dense(self.ctx, views, len(local_pes), C.byref(out)),
                "vdi_composite_host_dense")
        return int(out.total)

    def composite_host_dense_frames(self, frames, outs) -> list:
        """vdi_composite_host_dense_frames: frames = [[host DenseSubVDI per local PE]
        per frame], outs = [(count, depth, rgba) host tensors per frame]; H2D,
        compositing and D2H of consecutive frames overlap.  Returns the
        supersegment total of every frame."""
        F = len(frames)
        n_local = len(frames[0]) if F else 0
        if any(len(fr) != n_local for fr in frames) or len(outs) != F:
            raise ValueError("every frame needs the same number of local PEs and one output")
        views = self._host_views([p for fr in frames for p in fr])
        ov = (L.vdi_dense_strip * max(1, F))(*[self._dense_out(c, d, r) for c, d, r in outs])
        L.check(self.lib.vdi_composite_host_dense_frames(self.ctx, F, views, n_local, ov),
                "vdi_composite_host_dense_frames")
        return [int(ov[f].total) for f in range(F)]

    def gather(self, strip: FullVDI, image: FullVDI | None, root: int | None = None):
        """vdi_gather (root=None: the config's root) / vdi_gather_root: strips ->
        the root rank (image ignored on other ranks)."""
        sv = strip.view()
        iv = image.view() if image is not None else None
        ip = C.byref(iv) if iv is not None else None
        if root is None:
            L.check(self.lib.vdi_gather(self.ctx, C.byref(sv), ip), "vdi_gather")
        else:
            L.check(self.lib.vdi_gather_root(self.ctx, root, C.byref(sv), ip), "vdi_gather_root")
        return image

    # -- limit case and rendering ---------------------------
    def composite_image(self, local_pes, strip_rgba: torch.Tensor | None = None) -> torch.Tensor:
        """vdi_composite_image: the plain volume-rendered image of this rank's
        strip, premultiplied RGBA [rows*W, 4]."""
        P = (self.row_end - self.row_begin) * self.width
        if strip_rgba is None:
            strip_rgba = torch.empty((P, 4), dtype=torch.float32, device="cuda")
        views = (L.vdi_dense_view * max(1, len(local_pes)))(*[p.view() for p in local_pes])
        L.check(self.lib.vdi_composite_image(self.ctx, views, len(local_pes), strip_rgba.data_ptr()),
                "vdi_composite_image")
        return strip_rgba

    def gather_image(self, strip_rgba: torch.Tensor, image_rgba: torch.Tensor | None):
        """vdi_gather_image: strips of vdi_composite_image -> the root's [H*W, 4] image."""
        L.check(self.lib.vdi_gather_image(self.ctx, strip_rgba.data_ptr(),
                                          image_rgba.data_ptr() if image_rgba is not None else None),
                "vdi_gather_image")
        return image_rgba

    def render_generation_view(self, vdi: FullVDI) -> torch.Tensor:
        """vdi_render_generation_view: over of each list -> RGBA [rows*W, 4]."""
        out = torch.empty((vdi.count.numel(), 4), dtype=torch.float32, device="cuda")
        v = vdi.view()
        L.check(self.lib.vdi_render_generation_view(self.ctx, C.byref(v), out.data_ptr()),
                "vdi_render_generation_view")
        return out

    def render_novel_view(self, vdi: FullVDI, gen_camera, view_camera, dims, w, h) -> torch.Tensor:
        """vdi_render_novel_view: the full VDI (rows [0, H)) from view_camera -> RGBA [h*w, 4]."""
        out = torch.empty((w * h, 4), dtype=torch.float32, device="cuda")
        v = vdi.view()
        g, c = self._cam(gen_camera), self._cam(view_camera)
        d = (C.c_uint32 * 3)(*dims)
        L.check(self.lib.vdi_render_novel_view(self.ctx, C.byref(v), C.byref(g), C.byref(c), d, w, h, out.data_ptr()),
                "vdi_render_novel_view")
        return out

    def render_dvr(self, volume, tf_table, camera, w, h) -> torch.Tensor:
        """vdi_render_dvr: ground-truth DVR of the whole volume -> RGBA [h*w, 4]."""
        out = torch.empty((w * h, 4), dtype=torch.float32, device="cuda")
        vol, tf = self._vol(volume, tf_table)
        cam = self._cam(camera)
        L.check(self.lib.vdi_render_dvr(self.ctx, C.byref(vol), C.byref(tf), C.byref(cam), w, h, out.data_ptr()),
                "vdi_render_dvr")
        return out

    def pixel_stats(self, with_margin=False):
        """vdi_pixel_stats: per-list gamma*, m (and the tie margin) of the last composite."""
        P = (self.row_end - self.row_begin) * self.width
        g = torch.empty(P, dtype=torch.float32, device="cuda")
        mg = torch.empty(P, dtype=torch.float32, device="cuda")
        m = torch.empty(P, dtype=torch.int16, device="cuda")
        L.check(self.lib.vdi_pixel_stats(self.ctx, g.data_ptr(), mg.data_ptr(), m.data_ptr()), "vdi_pixel_stats")
        return (g, m, mg) if with_margin else (g, m)

    def counters(self) -> dict:
        c = L.vdi_counters()
        L.check(self.lib.vdi_get_counters(self.ctx, C.byref(c)), "vdi_get_counters")
        d = {f: getattr(c, f) for f, _ in L.vdi_counters._fields_}
        d["bucket_lists"] = list(d["bucket_lists"])
        return d
