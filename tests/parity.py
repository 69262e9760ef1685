"""Parity helpers: compare the CUDA path's full-representation output with
the oracle's, element by element, under the north-star tolerances:
counts (and therefore strip ownership / slot placement) bit-exact except for
lists whose threshold decision lies within 1e-6 of a tie (listed, not
failed); colours/opacities within 1e-4 absolute; depths within 1e-5 relative."""
import numpy as np
import torch

TIE_MARGIN = 1e-6
RGBA_ATOL = 1e-4
DEPTH_RTOL = 1e-5


def dense_to_device(pe: dict, pe_id: int, device="cuda"):
    from paper_2206_14503_b200 import DenseSubVDI
    cnt = torch.from_numpy(np.ascontiguousarray(pe["count"], np.uint8)).to(device)
    if "offset" in pe:
        off = np.asarray(pe["offset"], np.uint64).astype(np.uint32)
    else:
        c = np.asarray(pe["count"], np.uint32)
        off = np.zeros(len(c) + 1, np.uint32)
        np.cumsum(c, out=off[1:])
    offt = torch.from_numpy(off.view(np.int32)).to(device)
    dep = torch.from_numpy(np.ascontiguousarray(pe["depth"], np.float32).reshape(-1, 2)).to(device)
    rgba = torch.from_numpy(np.ascontiguousarray(pe["rgba"], np.float32).reshape(-1, 4)).to(device)
    return DenseSubVDI(pe_id, int(dep.shape[0]), cnt, offt, dep, rgba)


def compare(gpu_count, gpu_depth, gpu_rgba, orc_count, orc_depth, orc_rgba, margin=None, where=""):
    """Returns (n_lists, tie_list).  Raises AssertionError on a real mismatch."""
    gc = np.asarray(gpu_count).astype(np.int64)
    oc = np.asarray(orc_count).astype(np.int64)
    gd = np.asarray(gpu_depth, np.float32)
    od = np.asarray(orc_depth, np.float32)
    gr = np.asarray(gpu_rgba, np.float32)
    orr = np.asarray(orc_rgba, np.float32)
    tie = np.zeros(len(oc), bool) if margin is None else (np.asarray(margin) < TIE_MARGIN)
    bad_cnt = (gc != oc) & ~tie
    assert not bad_cnt.any(), (f"{where}: count mismatch at lists {np.nonzero(bad_cnt)[0][:10]} "
                               f"gpu={gc[bad_cnt][:10]} orc={oc[bad_cnt][:10]}")
    ok = ~tie
    dd = np.abs(gd[ok] - od[ok])
    lim = DEPTH_RTOL * np.maximum(np.abs(od[ok]), 1e-30)
    assert np.all(dd <= lim), f"{where}: depth mismatch max rel {np.max(dd / np.maximum(np.abs(od[ok]), 1e-30))}"
    err = np.abs(gr[ok] - orr[ok]).max() if ok.any() else 0.0
    assert err <= RGBA_ATOL, f"{where}: rgba mismatch max abs {err}"
    return int(ok.sum()), np.nonzero(tie)[0].tolist()


def full_to_numpy(full):
    return (full.count.cpu().numpy(), full.depth.cpu().numpy(), full.rgba.cpu().numpy())
