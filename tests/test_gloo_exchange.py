"""World-size-2 run of the multi-rank plan on CPU (gloo), no GPU needed.

Two processes each hold the PEs the product homes on them (vdi_pe_home,
PAPER.md:218 block placement), cut every sub-VDI into the image strips of
vdi_strip_rows (one strip per rank), exchange the strip
slices all-to-all over gloo (sizes first, then payload, as the product does
over NCCL/NVLink), composite their own strip with the oracle, and gather the
strips to rank 0.  Rank 0 checks that the assembled image is
bit-identical to a single-process composite of the whole image and that the
bytes sent equal the bytes received.  This covers the partition and exchange
plan of the N>1 path; the device side of the same path is tests/mgpu_check.py.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

W, H, N_PES, K_IN, K_OUT = 37, 13, 5, 6, 4   # 13 rows over 2 ranks: ragged strips


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _slice(pe, rb, re_):
    """Rows [rb, re_) of a dense sub-VDI (count u8[P], depth, rgba)."""
    off = np.concatenate([[0], np.cumsum(pe["count"].astype(np.int64))])
    a, b = rb * W, re_ * W
    return {"count": pe["count"][a:b].copy(), "depth": pe["depth"][off[a]:off[b]].copy(),
            "rgba": pe["rgba"][off[a]:off[b]].copy()}


def _pack(pe_id, s):
    head = np.array([pe_id, len(s["count"]), len(s["depth"])], np.int64).tobytes()
    return head + s["count"].tobytes() + s["depth"].astype(np.float32).tobytes() + \
        s["rgba"].astype(np.float32).tobytes()


def _unpack(buf):
    out, p = [], 0
    while p < len(buf):
        pe_id, npix, nrec = np.frombuffer(buf[p:p + 24], np.int64)
        p += 24
        cnt = np.frombuffer(buf[p:p + npix], np.uint8).copy()
        p += int(npix)
        dep = np.frombuffer(buf[p:p + 8 * nrec], np.float32).reshape(-1, 2).copy()
        p += 8 * int(nrec)
        rgb = np.frombuffer(buf[p:p + 16 * nrec], np.float32).reshape(-1, 4).copy()
        p += 16 * int(nrec)
        out.append((int(pe_id), {"count": cnt, "depth": dep, "rgba": rgb}))
    return out


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2206_14503_b200 import api
        pes = synth.random_subvdis(N_PES, W, H, K_IN, lam=5.0, seed=23)   # same seed on every rank
        home = [pe for pe in range(N_PES) if api.pe_home(N_PES, world, pe) == rank]
        strips = [api.strip_rows(H, world, g) for g in range(world)]
        # exchange: to rank g, the rows of strip g of every PE homed here
        send = [b"".join(_pack(pe, _slice(pes[pe], *strips[g])) for pe in home) for g in range(world)]
        ssz = torch.tensor([len(b) for b in send], dtype=torch.int64)
        rsz = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rsz, ssz)
        sbuf = torch.frombuffer(bytearray(b"".join(send)), dtype=torch.uint8) if sum(map(len, send)) else \
            torch.empty(0, dtype=torch.uint8)
        rbuf = torch.empty(int(rsz.sum()), dtype=torch.uint8)
        dist.all_to_all_single(rbuf, sbuf, rsz.tolist(), ssz.tolist())
        got = sorted(_unpack(rbuf.numpy().tobytes()))          # PE order fixes the tie-break (Q-readings)
        rb, re_ = strips[rank]
        mine = oracle.composite([p for _, p in got], W, re_ - rb, 1, K_OUT, with_stats=False)
        # gather the strips to rank 0
        part = [mine["count"], mine["depth"], mine["rgba"]]
        parts = [None] * world if rank == 0 else None
        dist.gather_object(part, parts, dst=0)
        sent = torch.tensor([float(ssz.sum()), float(rsz.sum())], dtype=torch.float64)
        dist.all_reduce(sent)
        if rank == 0:
            img = [np.concatenate([p[i] for p in parts]) for i in range(3)]
            ref = oracle.composite(pes, W, H, 1, K_OUT, with_stats=False)
            q.put({"homes": [api.pe_home(N_PES, world, pe) for pe in range(N_PES)],
                   "strips": strips,
                   "identical": all(np.array_equal(a, ref[k]) for a, k in zip(img, ("count", "depth", "rgba"))),
                   "pes_received": len(got), "conserved": bool(sent[0] == sent[1])})
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_matches_single_process():
    try:
        import oracle
        oracle.lib()
    except Exception as e:   # pragma: no cover
        pytest.skip(f"oracle not built: {e}")
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # block placement: every rank homes a contiguous run of PEs, all PEs homed once
    assert res["homes"] == sorted(res["homes"]) and set(res["homes"]) == {0, 1}
    # strips tile the image rows without gaps or overlap (ragged last strip)
    (b0, e0), (b1, e1) = res["strips"]
    assert b0 == 0 and e0 == b1 and e1 == H and abs((e0 - b0) - (e1 - b1)) <= 1
    assert res["pes_received"] == N_PES      # every PE contributes to every strip
    assert res["conserved"]
    assert res["identical"]


def _frames_worker(rank, world, port, q):
    """Frames mode (vdi_composite_frames): frame f is composited whole by rank
    f mod G from every rank's PEs; each rank sends the whole sub-VDIs of its
    PEs for frame f to f's owner (sizes first, then payload)."""
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2206_14503_b200 import api
        F = 2 * world
        frames = [synth.random_subvdis(N_PES, W, H, K_IN, lam=4.0 + f, seed=40 + f) for f in range(F)]
        home = [pe for pe in range(N_PES) if api.pe_home(N_PES, world, pe) == rank]
        send = [b"".join(_pack(f * N_PES + pe, _slice(frames[f][pe], 0, H)) for f in range(g, F, world)
                         for pe in home) for g in range(world)]
        ssz = torch.tensor([len(b) for b in send], dtype=torch.int64)
        rsz = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rsz, ssz)
        sbuf = torch.frombuffer(bytearray(b"".join(send)), dtype=torch.uint8)
        rbuf = torch.empty(int(rsz.sum()), dtype=torch.uint8)
        dist.all_to_all_single(rbuf, sbuf, rsz.tolist(), ssz.tolist())
        got = sorted(_unpack(rbuf.numpy().tobytes()))
        ok, owned = True, []
        for f in range(rank, F, world):
            pes_f = [p for key, p in got if key // N_PES == f]
            assert [key % N_PES for key, _ in got if key // N_PES == f] == list(range(N_PES))
            img = oracle.composite(pes_f, W, H, 1, K_OUT, with_stats=False)
            ref = oracle.composite(frames[f], W, H, 1, K_OUT, with_stats=False)
            ok &= all(np.array_equal(img[k], ref[k]) for k in ("count", "depth", "rgba"))
            owned.append(f)
        res = [None] * world if rank == 0 else None
        dist.gather_object((owned, ok), res, dst=0)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


def test_two_rank_frames_mode_matches_single_process():
    try:
        import oracle
        oracle.lib()
    except Exception as e:   # pragma: no cover
        pytest.skip(f"oracle not built: {e}")
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_frames_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o for o, _ in res] == [[0, 2], [1, 3]]   # frame f owned by rank f mod G
    assert all(ok for _, ok in res)
