"""VDI_FLAG_VALIDATE (include/vdi.h): the device-side input check of
vdi_composite.  Valid sub-VDIs (random, overlapping, generated) pass and
composite exactly as without the flag; each kind of invalid input -- a list
longer than k_in, offsets that disagree with the counts, a supersegment with
t_front >= t_back, an opacity outside [0, 1], a list out of depth order
(the lists a PE produces are depth-sorted) -- is refused with
VDI_ERR_INVALID_ARG before any merge kernel runs."""
import numpy as np
import pytest
import torch

import synth
from parity import dense_to_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vdi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2206_14503_b200 as vdi
    vdi._lib.lib()
    return vdi


W, H, K = 67, 29, 8


def _pes(overlap=False):
    return synth.random_subvdis(3, W, H, K, lam=4.0, seed=41, overlap=overlap)


@pytest.mark.parametrize("overlap", [False, True])
def test_valid_inputs_pass(vdi, overlap):
    pes = _pes(overlap)
    out = []
    for flags in (0, vdi._lib.VDI_FLAG_VALIDATE):
        comp = vdi.Compositor(W, H, K, K, len(pes), flags=flags)
        strip = comp.empty_strip()
        comp.composite([dense_to_device(p, i) for i, p in enumerate(pes)], strip)
        torch.cuda.synchronize()
        out.append(strip)
    assert torch.equal(out[0].count, out[1].count)
    assert torch.equal(out[0].depth, out[1].depth) and torch.equal(out[0].rgba, out[1].rgba)


def _corrupt(pes, kind):
    p = {k: np.array(v, copy=True) for k, v in pes[1].items()}
    c = p["count"].astype(np.int64)
    off = np.zeros(len(c) + 1, np.int64)
    np.cumsum(c, out=off[1:])
    i = int(np.nonzero(c >= 2)[0][0])   # a list with two records
    r = int(off[i])
    d = p["depth"].reshape(-1, 2)
    if kind == "count":
        p["count"][i] = K + 1
        p["offset"] = off            # consistent offsets, but the list is longer than k_in
        p["offset"][i + 1:] += K + 1 - c[i]
        d_new = np.zeros((int(p["offset"][-1]), 2), np.float32)
        rg_new = np.zeros((int(p["offset"][-1]), 4), np.float32)
        d_new[:] = np.arange(len(d_new) * 2, dtype=np.float32).reshape(-1, 2)
        rg_new[:, 3] = 0.5
        p["depth"], p["rgba"] = d_new, rg_new
    elif kind == "offset":
        p["offset"] = off.copy()
        p["offset"][i + 1] += 1
    elif kind == "front_back":
        d[r, 1] = d[r, 0]
    elif kind == "alpha":
        p["rgba"].reshape(-1, 4)[r, 3] = 1.5
    elif kind == "order":
        d[[r, r + 1]] = d[[r + 1, r]]
    return [pes[0], p, pes[2]]


@pytest.mark.parametrize("kind", ["count", "offset", "front_back", "alpha", "order"])
def test_invalid_inputs_refused(vdi, kind):
    pes = _corrupt(_pes(), kind)
    comp = vdi.Compositor(W, H, K, K, len(pes), flags=vdi._lib.VDI_FLAG_VALIDATE)
    strip = comp.empty_strip()
    with pytest.raises(vdi._lib.VdiError) as e:
        comp.composite([dense_to_device(p, i) for i, p in enumerate(pes)], strip)
    assert e.value.status == vdi._lib.VDI_ERR_INVALID_ARG
    assert "VDI_FLAG_VALIDATE" in str(e.value)
    # the context stays usable: valid inputs composite afterwards
    comp.composite([dense_to_device(p, i) for i, p in enumerate(_pes())], strip)
    torch.cuda.synchronize()


def test_generated_subvdis_pass(vdi):
    cfg = synth.config_by_name("C1")
    vol = synth.make_volume(cfg, device="cuda")
    tf = torch.from_numpy(synth.tf_table(cfg.tf, cfg.tf_scale)).cuda()
    cam = synth.make_camera(cfg.W, cfg.H)
    comp = vdi.Compositor(cfg.W, cfg.H, cfg.k_in, cfg.k_out, cfg.n_pes, flags=vdi._lib.VDI_FLAG_VALIDATE)
    pes = [comp.generate_subvdi(vol, tf, cam, cfg.decomposition(), pe) for pe in range(cfg.n_pes)]
    comp.composite(pes, comp.empty_strip())
    torch.cuda.synchronize()
