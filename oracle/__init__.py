"""CPU oracle (TEST INFRASTRUCTURE) — ctypes wrapper over oracle/liboracle.so.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  The product package
(paper_2206_14503_b200) never imports it and shares no code with it.
Arrays are numpy; records are (tf, tb, r, g, b, a) float32 rows.
Function-level citations live in oracle/oracle.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fopenmp", "-fPIC", "-shared", "-o", _SO, src])
    return _SO


class Stats(C.Structure):
    _fields_ = [("gamma", C.c_float), ("margin", C.c_float), ("m", C.c_int32), ("iters", C.c_int32),
                ("sweep_steps", C.c_int64), ("overlap", C.c_int32), ("count", C.c_int32)]


STATS_DTYPE = np.dtype([("gamma", np.float32), ("margin", np.float32), ("m", np.int32),
                        ("iters", np.int32), ("sweep_steps", np.int64), ("overlap", np.int32),
                        ("count", np.int32)], align=True)


class Scene(C.Structure):
    _fields_ = [("vox", C.c_void_p), ("bytes", C.c_int32), ("dx", C.c_int32), ("dy", C.c_int32),
                ("dz", C.c_int32), ("tf", C.c_void_p), ("eye", C.c_float * 3), ("fwd", C.c_float * 3),
                ("right", C.c_float * 3), ("up", C.c_float * 3), ("tan_x", C.c_float),
                ("tan_y", C.c_float), ("W", C.c_int32), ("H", C.c_int32), ("gx", C.c_int32),
                ("gy", C.c_int32), ("gz", C.c_int32), ("xb", C.c_void_p), ("yb", C.c_void_p),
                ("zb", C.c_void_p), ("owner", C.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
        _lib.orc_gamma_search.restype = C.c_float
        _lib.orc_generate_dense.restype = C.c_int64
        _lib.orc_ray_owners.restype = C.c_int64
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _recs(a):
    a = np.ascontiguousarray(np.asarray(a, np.float32).reshape(-1, 6))
    return a


# --- primitives -----------------------------------------------------------
def over(front, back):
    f = np.asarray(front, np.float32)
    b = np.asarray(back, np.float32)
    o = np.zeros(4, np.float32)
    lib().orc_over(_p(f), _p(b), _p(o))
    return o


def exclusive_scan(counts):
    c = np.ascontiguousarray(np.asarray(counts, np.uint32))
    o = np.zeros(len(c) + 1, np.uint64)
    lib().orc_exclusive_scan(_p(c), C.c_int64(len(c)), _p(o))
    return o


def sort_samples(lists):
    """lists: sequence of per-source (c_s, 6) arrays. Returns the sorted samples."""
    counts = np.array([len(l) for l in lists], np.int32)
    recs = _recs(np.concatenate([_recs(l) for l in lists]) if len(lists) else np.zeros((0, 6)))
    out = np.zeros((max(1, len(recs)), 6), np.float32)
    n = lib().orc_sort_samples(C.c_int32(len(lists)), _p(counts), _p(recs), _p(out))
    return out[:n]


def subdivide(samples):
    s = _recs(samples)
    out = np.zeros((max(1, 2 * len(s)), 6), np.float32)
    n = lib().orc_subdivide(C.c_int32(len(s)), _p(s), _p(out))
    return out[:n]


def sweep(samples, gamma, k_out, write=True):
    s = _recs(samples)
    out = np.zeros((max(1, len(s)), 6), np.float32)
    n = lib().orc_sweep(C.c_int32(len(s)), _p(s), C.c_float(gamma), C.c_int32(k_out),
                        C.c_int32(1 if write else 0), _p(out))
    return (n, out[:n]) if write else n


def gamma_search(samples, k_out, max_iters=16, gamma_max=2.0):
    s = _recs(samples)
    tm = np.zeros(max(1, max_iters), np.float32)
    tc = np.zeros(max(1, max_iters), np.int32)
    it = C.c_int32(0)
    g = lib().orc_gamma_search(C.c_int32(len(s)), _p(s), C.c_int32(k_out), C.c_int32(max_iters),
                               C.c_float(gamma_max), C.byref(it), _p(tm), _p(tc))
    return float(g), list(zip(tm[:it.value].tolist(), tc[:it.value].tolist()))


def recomposite(lists, k_out, max_iters=16, gamma_max=2.0):
    """Steps 1-6 for one list. Returns (count, out (k_out,6) zero-filled, stats dict)."""
    counts = np.array([len(l) for l in lists], np.int32)
    recs = _recs(np.concatenate([_recs(l) for l in lists])) if sum(counts) else np.zeros((1, 6), np.float32)
    out = np.zeros((max(1, k_out), 6), np.float32)
    st = Stats()
    n = lib().orc_recomposite(C.c_int32(len(lists)), _p(counts), _p(recs), C.c_int32(k_out),
                              C.c_int32(max_iters), C.c_float(gamma_max), _p(out), C.byref(st))
    return n, out[:k_out], {f: getattr(st, f) for f, _ in Stats._fields_}


def _ptr_array(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def composite(pes, W, H, G, k_out, max_iters=16, gamma_max=2.0, pix_begin=0, pix_end=-1,
              n_threads=1, with_stats=True, out=None):
    """Direct-send composite of dense sub-VDIs (dicts with count/depth/rgba
    numpy arrays).  Returns dict(count u8[P], depth f32[P,k,2], rgba f32[P,k,4], stats).
    `out` (optional): a previous result dict whose arrays are reused (a band
    composite then does not pay for zeroing whole-image outputs)."""
    P = W * H
    cnt = [np.ascontiguousarray(p["count"], np.uint8) for p in pes]
    dep = [np.ascontiguousarray(p["depth"], np.float32) for p in pes]
    rgb = [np.ascontiguousarray(p["rgba"], np.float32) for p in pes]
    if out is not None:
        oc, od, orgba, st = out["count"], out["depth"], out["rgba"], out["stats"]
        assert oc.shape == (P,) and od.shape == (P, k_out, 2) and (st is not None) == with_stats
    else:
        oc = np.zeros(P, np.uint8)
        od = np.zeros((P, k_out, 2), np.float32)
        orgba = np.zeros((P, k_out, 4), np.float32)
        st = np.zeros(P, STATS_DTYPE) if with_stats else None
    lib().orc_composite(C.c_int32(len(pes)), _ptr_array(cnt), _ptr_array(dep), _ptr_array(rgb),
                        C.c_int32(W), C.c_int32(H), C.c_int32(G), C.c_int32(k_out), C.c_int32(max_iters),
                        C.c_float(gamma_max), C.c_int64(pix_begin), C.c_int64(pix_end),
                        C.c_int32(n_threads), _p(oc), _p(od), _p(orgba),
                        _p(st) if with_stats else None)
    return {"count": oc, "depth": od, "rgba": orgba, "stats": st}


def composite_pixels(pes, pix, k_out, max_iters=16, gamma_max=2.0, offsets=None):
    """Per-pixel composite for a pixel list (sampled parity at full sizes)."""
    pix = np.ascontiguousarray(np.asarray(pix, np.int64))
    cnt = [np.ascontiguousarray(p["count"], np.uint8) for p in pes]
    if offsets is None:
        offsets = [exclusive_scan(c) for c in cnt]
    offs = [np.ascontiguousarray(o, np.uint64) for o in offsets]
    dep = [np.ascontiguousarray(p["depth"], np.float32) for p in pes]
    rgb = [np.ascontiguousarray(p["rgba"], np.float32) for p in pes]
    n = len(pix)
    oc = np.zeros(n, np.uint8)
    od = np.zeros((n, k_out, 2), np.float32)
    orgba = np.zeros((n, k_out, 4), np.float32)
    st = np.zeros(n, STATS_DTYPE)
    lib().orc_composite_pixels(C.c_int32(len(pes)), _ptr_array(cnt), _ptr_array(offs), _ptr_array(dep),
                               _ptr_array(rgb), C.c_int32(k_out), C.c_int32(max_iters),
                               C.c_float(gamma_max), C.c_int64(n), _p(pix), _p(oc), _p(od), _p(orgba),
                               _p(st))
    return {"count": oc, "depth": od, "rgba": orgba, "stats": st}


# --- generator / DVR -------------------------------------------------------
class SceneHandle:
    """Keeps the numpy buffers referenced by an orc_scene alive."""

    def __init__(self, vol, bytes_per_voxel, dims, tf, cam, dec):
        self.vol = np.ascontiguousarray(vol)
        self.tf = np.ascontiguousarray(tf, np.float32)
        self.xb = np.ascontiguousarray(dec.xb, np.int32)
        self.yb = np.ascontiguousarray(dec.yb, np.int32)
        self.zb = np.ascontiguousarray(dec.zb, np.int32)
        self.owner = np.ascontiguousarray(dec.owner, np.int32)
        s = Scene()
        s.vox = self.vol.ctypes.data
        s.bytes = bytes_per_voxel
        s.dx, s.dy, s.dz = dims
        s.tf = self.tf.ctypes.data
        s.eye[:] = cam.eye
        s.fwd[:] = cam.fwd
        s.right[:] = cam.right
        s.up[:] = cam.up
        s.tan_x, s.tan_y = cam.tan_x, cam.tan_y
        s.W, s.H = cam.W, cam.H
        s.gx, s.gy, s.gz = len(dec.xb) - 1, len(dec.yb) - 1, len(dec.zb) - 1
        s.xb, s.yb, s.zb, s.owner = (self.xb.ctypes.data, self.yb.ctypes.data, self.zb.ctypes.data,
                                     self.owner.ctypes.data)
        self.s = s
        self.W, self.H = cam.W, cam.H


def pixels_to_dense(gen, P, pix):
    """Per-pixel generator output (generate_pixels) -> full-image dense arrays
    with empty lists outside `pix` (pix sorted ascending)."""
    k = gen["depth"].shape[1]
    cnt = np.zeros(P, np.uint8)
    cnt[pix] = gen["count"]
    used = np.arange(k)[None, :] < gen["count"][:, None].astype(np.int64)
    return {"count": cnt, "depth": np.ascontiguousarray(gen["depth"][used]),
            "rgba": np.ascontiguousarray(gen["rgba"][used])}


def scene(vol, dims, tf, cam, dec):
    v = np.asarray(vol)
    bpv = 1 if v.dtype == np.uint8 else 2
    return SceneHandle(v, bpv, dims, tf, cam, dec)


def generate_dense(sc: SceneHandle, pe, k, max_iters=16, gamma_max=2.0, n_threads=1):
    P = sc.W * sc.H
    cnt = np.zeros(P, np.uint8)
    gam = np.zeros(P, np.float32)
    off = np.zeros(P + 1, np.uint64)
    cap = P * k
    dep = np.zeros((cap, 2), np.float32)
    rgba = np.zeros((cap, 4), np.float32)
    tot = lib().orc_generate_dense(C.byref(sc.s), C.c_int32(pe), C.c_int32(k), C.c_int32(max_iters),
                                   C.c_float(gamma_max), C.c_int32(n_threads), _p(cnt), _p(gam), _p(off),
                                   _p(dep), _p(rgba), C.c_int64(cap))
    if tot < 0:
        raise RuntimeError(f"orc_generate_dense failed ({tot})")
    return {"count": cnt, "gamma": gam, "offset": off, "depth": dep[:tot].copy(), "rgba": rgba[:tot].copy()}


def generate_pixels(sc: SceneHandle, pe, k, pix, max_iters=16, gamma_max=2.0, n_threads=1):
    pix = np.ascontiguousarray(np.asarray(pix, np.int64))
    n = len(pix)
    cnt = np.zeros(n, np.uint8)
    gam = np.zeros(n, np.float32)
    dep = np.zeros((n, k, 2), np.float32)
    rgba = np.zeros((n, k, 4), np.float32)
    rc = lib().orc_generate_pixels(C.byref(sc.s), C.c_int32(pe), C.c_int32(k), C.c_int32(max_iters),
                                   C.c_float(gamma_max), C.c_int64(n), _p(pix), C.c_int32(n_threads), _p(cnt),
                                   _p(gam), _p(dep), _p(rgba))
    return {"count": cnt, "gamma": gam, "depth": dep, "rgba": rgba, "capacity_exceeded": rc == -2}


def dvr(sc: SceneHandle, pix=None, n_threads=1):
    if pix is None:
        n = sc.W * sc.H
        pp = None
    else:
        pix = np.ascontiguousarray(np.asarray(pix, np.int64))
        n = len(pix)
        pp = _p(pix)
    out = np.zeros((n, 4), np.float32)
    lib().orc_dvr(C.byref(sc.s), C.c_int64(n), pp, C.c_int32(n_threads), _p(out))
    return out


def render_full(count, rgba):
    count = np.ascontiguousarray(count, np.uint8)
    P = len(count)
    k = rgba.shape[1]
    rgba = np.ascontiguousarray(rgba, np.float32)
    out = np.zeros((P, 4), np.float32)
    lib().orc_render_full(C.c_int64(P), C.c_int32(k), _p(count), _p(rgba), _p(out))
    return out


def ray_owners(sc: SceneHandle, x, y, cap=1 << 16):
    own = np.zeros(cap, np.int32)
    tlo = np.zeros(cap, np.float32)
    thi = np.zeros(cap, np.float32)
    rgba = np.zeros((cap, 4), np.float32)
    n = lib().orc_ray_owners(C.byref(sc.s), C.c_int32(x), C.c_int32(y), C.c_int64(cap), _p(own), _p(tlo),
                             _p(thi), _p(rgba))
    n = min(n, cap)
    return own[:n], tlo[:n], thi[:n], rgba[:n]


def volume_numpy(vol_tensor):
    """torch volume (u8, or u16 bits in int16) -> numpy array for the oracle."""
    a = vol_tensor.detach().cpu().numpy()
    if a.dtype == np.int16:
        a = a.view(np.uint16)
    return np.ascontiguousarray(a)
