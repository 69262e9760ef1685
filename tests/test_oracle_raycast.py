"""Closed-form pins of the oracle's Phase-1 raycast primitives (make_ray,
sample_trilinear, classify, owner_of, ray_samples; oracle/oracle.cpp) --
SUPPORT code whose output feeds every full-size parity test.  None of the
expected values comes from the oracle: each is a closed form of the scene
(DESIGN.md §4 geometry: world box with longest side 1 centred at the origin,
voxel i covering [i, i+1), pinhole rays through pixel centres, samples at
t_in + (i + 1/2) dt with dt = one voxel, Q18/Q19):

* constant transfer function -> every sample inside the box has the same
  premultiplied RGBA, so DVR = 1 - (1 - a)^n with n the number of grid samples
  in [t_in, t_out) of the ray/box intersection, computed here in float64;
* a linear-ramp field -> trilinear interpolation is exact, so each sample's
  value is the ramp at the sample point (away from the faces);
* constant u8 volumes at table knots j/255 -> classify returns tf[j]
  premultiplied;
* the brick owner of every sample against a numpy point-in-brick search."""
import numpy as np
import pytest

import synth

F32 = np.float32


def ray_f64(cam, x, y):
    """Pinhole ray through the centre of pixel (x, y), row 0 at the top."""
    sx = ((2.0 * (x + 0.5)) / cam.W - 1.0) * cam.tan_x
    sy = (1.0 - (2.0 * (y + 0.5)) / cam.H) * cam.tan_y
    v = np.array(cam.fwd, np.float64) + sx * np.array(cam.right) + sy * np.array(cam.up)
    return np.array(cam.eye, np.float64), v / np.linalg.norm(v)


def box_hit(o, d, dims):
    md = max(dims)
    half = np.array(dims, np.float64) / (2.0 * md)
    with np.errstate(divide="ignore", invalid="ignore"):
        t0 = (-half - o) / d
        t1 = (half - o) / d
    tmin = max(0.0, np.nanmax(np.minimum(t0, t1)))
    tmax = np.nanmin(np.maximum(t0, t1))
    return tmin, tmax, md


def _scene(orc, vol, dims, tf, cam, dec=None):
    dec = dec if dec is not None else synth.slab_decomposition(dims, 1)
    return orc.scene(vol, dims, tf, cam, dec)


def test_constant_tf_dvr_closed_form(orc):
    dims = (40, 32, 24)
    rng = np.random.default_rng(3)
    vol = rng.integers(0, 255, size=dims[::-1], dtype=np.uint8)  # any field: the TF ignores it
    rgba = np.array([0.7, 0.2, 0.4, 0.05], F32)
    tf = np.tile(rgba, (256, 1)).astype(F32)
    cam = synth.make_camera(33, 27, view=0, angle_deg=23.0, dist=1.3, vfov_deg=50.0)
    sc = _scene(orc, vol, dims, tf, cam)
    img = orc.dvr(sc)
    checked = hit = 0
    for y in range(cam.H):
        for x in range(cam.W):
            o, d = ray_f64(cam, x, y)
            t_in, t_out, md = box_hit(o, d, dims)
            p = y * cam.W + x
            if not t_out > t_in:
                assert np.all(img[p] == 0)
                continue
            q = (t_out - t_in) * md - 0.5
            if abs(q - round(q)) < 1e-3:
                continue  # sample count ambiguous at float precision
            n = max(0, int(np.ceil(q)))
            own, tlo, thi, srgba = orc.ray_owners(sc, x, y)
            assert len(own) == n, (x, y, len(own), n)
            if n:
                assert abs(tlo[0] - t_in) <= 2e-6 and abs(thi[-1] - (t_in + n / md)) <= 2e-6
                assert np.all(own == 0)
                np.testing.assert_allclose(srgba, np.tile(rgba * np.array([rgba[3]] * 3 + [1], F32), (n, 1)),
                                           atol=1e-7)
                hit += 1
            a = 1.0 - (1.0 - float(rgba[3])) ** n
            exp = np.array([rgba[0] * a, rgba[1] * a, rgba[2] * a, a])
            np.testing.assert_allclose(img[p], exp, atol=2e-5, err_msg=f"pixel {x},{y} n={n}")
            checked += 1
    assert checked > 500 and hit > 300


def test_linear_ramp_trilinear_exact(orc):
    dims = (48, 40, 32)
    A, B = 2000, (311, 173, 97)
    k, j, i = np.meshgrid(np.arange(dims[2]), np.arange(dims[1]), np.arange(dims[0]), indexing="ij")
    vol = (A + B[0] * i + B[1] * j + B[2] * k).astype(np.uint16)
    tf = np.stack([np.arange(256) / 255.0] * 3 + [np.ones(256)], 1).astype(F32)  # identity ramp, alpha 1
    cam = synth.make_camera(17, 13, view=1, angle_deg=-31.0, dist=1.2)
    sc = _scene(orc, vol, dims, tf, cam)
    md = max(dims)
    half = np.array(dims, np.float64) / (2.0 * md)
    checked = 0
    for y in range(cam.H):
        for x in range(cam.W):
            o, d = ray_f64(cam, x, y)
            own, tlo, thi, srgba = orc.ray_owners(sc, x, y)
            for q in range(len(own)):
                t = 0.5 * (float(tlo[q]) + float(thi[q]))
                c = (o + t * d + half) * md          # continuous voxel coordinates
                u = c - 0.5
                if np.any(np.floor(u) < 0) or np.any(np.floor(u) + 1 > np.array(dims) - 1):
                    continue  # a neighbour lies outside the volume (reads 0)
                v = (A + B[0] * u[0] + B[1] * u[1] + B[2] * u[2]) / 65535.0
                assert abs(srgba[q, 0] - v) <= 3e-5 and srgba[q, 3] == 1.0, (x, y, q, srgba[q, 0], v)
                checked += 1
    assert checked > 2000


@pytest.mark.parametrize("j", [0, 1, 37, 128, 254, 255])
def test_tf_at_table_knots(orc, j):
    dims = (8, 8, 8)
    vol = np.full(dims[::-1], j, np.uint8)
    rng = np.random.default_rng(j)
    tf = rng.random((256, 4)).astype(F32)
    cam = synth.make_camera(1, 1, view=0)       # the axial ray through the box centre
    sc = _scene(orc, vol, dims, tf, cam)
    own, tlo, thi, srgba = orc.ray_owners(sc, 0, 0)
    assert len(own) == 8 and np.all(own == 0)
    a = tf[j, 3]
    exp = np.array([tf[j, 0] * a, tf[j, 1] * a, tf[j, 2] * a, a], F32)
    np.testing.assert_allclose(srgba, np.tile(exp, (8, 1)), atol=1e-6)
    # the axial ray enters at the z face: t_in = 1.8 - 1/2, samples one voxel apart
    assert abs(tlo[0] - 1.3) <= 1e-6 and np.allclose(np.diff(tlo), 1 / 8, atol=1e-6)


def test_owner_point_in_brick(orc):
    dims = (36, 28, 20)
    dec = synth.interleaved_decomposition(dims, 4, (4, 4, 2), seed=9)
    vol = np.full(dims[::-1], 200, np.uint8)
    tf = np.tile(np.array([1, 1, 1, 0.5], F32), (256, 1))
    cam = synth.make_camera(23, 19, view=0, angle_deg=37.0, dist=1.4)
    sc = _scene(orc, vol, dims, tf, cam, dec)
    md = max(dims)
    half = np.array(dims, np.float64) / (2.0 * md)
    bounds = [np.asarray(b, np.float64) for b in (dec.xb, dec.yb, dec.zb)]
    gx, gy, _ = dec.grid
    checked = 0
    for y in range(cam.H):
        for x in range(cam.W):
            o, d = ray_f64(cam, x, y)
            own, tlo, thi, _ = orc.ray_owners(sc, x, y)
            for q in range(len(own)):
                t = 0.5 * (float(tlo[q]) + float(thi[q]))
                c = (o + t * d + half) * md
                if min(np.min(np.abs(c[a] - bounds[a])) for a in range(3)) < 1e-3:
                    continue  # within rounding of a brick face
                if np.any(c < 0) or np.any(c >= np.array(dims)):
                    assert own[q] == -1
                    continue
                b = [int(np.searchsorted(bounds[a], c[a], side="right")) - 1 for a in range(3)]
                assert own[q] == dec.owner[(b[2] * gy + b[1]) * gx + b[0]], (x, y, q)
                checked += 1
    assert checked > 3000
