"""Multi-rank (N > 1) host logic on the CPU: the band partition, the frame
assignment, and the C ABI's band-sharding plan (dmm_shard_plan /
dmm_shard_locate, host-only entry points of libdmm_b200.so) driven through a
real multi-process exchange over torch.distributed (gloo, world 2 and 3).

The exchange moves every record of a rank's H band to the rank owning its
column in the V band (and back) -- a pure permutation of records.  Each
process stamps its H band records with their pixel coordinates at the offsets
dmm_shard_locate gives, executes dmm_shard_plan's transfers with
dist.isend / dist.irecv (own block: a local copy), and checks that every V band
slot received exactly the record of its pixel.  The GPU side (the kernels
reading / writing those offsets, bit-exact vs the oracle) is
tests/test_gpu_parity.py::test_rowcol_*."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1601_06274_b200 as dmm
from paper_1601_06274_b200 import sharding


def test_bands_partition():
    for n in (1, 2, 7, 375, 1242):
        for world in (1, 2, 3, 8):
            b = sharding.bands(n, world)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[k][1] == b[k + 1][0] for k in range(world - 1))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1


def test_frames_for_rank():
    for n, world in ((64, 8), (10, 3), (2, 4)):
        got = sorted(f for r in range(world) for f in sharding.frames_for_rank(n, world, r))
        assert got == list(range(n))


def _cfg(W=67, H=13, K=40):
    return dmm.make_config(W, H, 0, K - 1, max_iters=4)


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_locate_owns_each_pixel_once(world):
    """Every pixel's H record is owned by the rank of its row band, its V
    record by the rank of its column band (sharding.bands), at distinct,
    record-aligned offsets inside the rank's workspace."""
    cfg = _cfg()
    W, H = cfg.width, cfg.height
    rows, cols = sharding.bands(H, world), sharding.bands(W, world)
    rec = 2 * 64 + 16
    for r in range(world):
        total = dmm.shard_workspace_bytes(cfg, r, world)
        assert total > 0
        for which, owned in ((dmm.LOC_FV_H, lambda y, x: rows[r][0] <= y < rows[r][1]),
                             (dmm.LOC_FH_V, lambda y, x: cols[r][0] <= x < cols[r][1])):
            offs = []
            for y in range(H):
                for x in range(W):
                    o = dmm.shard_locate(cfg, r, world, which, y, x)
                    assert (o >= 0) == owned(y, x)
                    if o >= 0:
                        assert 0 <= o and o + rec <= total
                        offs.append(o)
            offs = np.sort(np.array(offs))
            assert np.all(np.diff(offs) >= rec)


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_plan_pairs_up(world):
    """Rank r's send to s has exactly the size of s's receive from r, and the
    blocks one rank sends (phase 0) tile its H band's record array."""
    cfg = _cfg(W=16 * world + 9, H=7 + world)
    plans = [[dmm.shard_plan(cfg, r, world, ph) for ph in (0, 1)] for r in range(world)]
    rec = 2 * 64 + 16
    for ph in (0, 1):
        for r in range(world):
            assert [p[0] for p in plans[r][ph]] == list(range(world))
            for s in range(world):
                assert plans[r][ph][s][2] == plans[s][ph][r][4]
        for r in range(world):
            sends = sorted((p[1], p[2]) for p in plans[r][ph])
            rows = sharding.bands(cfg.height, world)[r]
            cols = sharding.bands(cfg.width, world)[r]
            n_rec = (rows[1] - rows[0]) * cfg.width if ph == 0 else cfg.height * (cols[1] - cols[0])
            assert sum(b for _, b in sends) == n_rec * rec
            assert all(sends[k][0] + sends[k][1] == sends[k + 1][0] for k in range(world - 1))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stamp(ws, off, y, x, tag):
    ws[off: off + 12] = np.frombuffer(np.array([y, x, tag], np.int32).tobytes(), np.uint8)


def _read(ws, off):
    return tuple(int(v) for v in np.frombuffer(ws[off: off + 12].tobytes(), np.int32))


def _exchange(ws, plan, rank):
    reqs, bufs = [], []
    for peer, so, sb, ro, rb in plan:
        if peer == rank:
            ws[ro: ro + rb] = ws[so: so + sb].copy()
            continue
        if sb:
            reqs.append(dist.isend(torch.from_numpy(ws[so: so + sb].copy()), peer))
        if rb:
            buf = torch.empty(rb, dtype=torch.uint8)
            reqs.append(dist.irecv(buf, peer))
            bufs.append((ro, buf))
    for q in reqs:
        q.wait()
    for ro, buf in bufs:
        ws[ro: ro + buf.numel()] = buf.numpy()


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = _cfg(W=16 * world + 21, H=9 + 2 * world, K=33)
        W, H = cfg.width, cfg.height
        ws = np.zeros(dmm.shard_workspace_bytes(cfg, rank, world), np.uint8)
        bad = 0
        # phase 0: H band f_ records -> V band
        for y in range(H):
            for x in range(W):
                o = dmm.shard_locate(cfg, rank, world, dmm.LOC_FV_H, y, x)
                if o >= 0:
                    _stamp(ws, o, y, x, 100)
        _exchange(ws, dmm.shard_plan(cfg, rank, world, 0), rank)
        for y in range(H):
            for x in range(W):
                o = dmm.shard_locate(cfg, rank, world, dmm.LOC_FV_V, y, x)
                if o >= 0 and _read(ws, o) != (y, x, 100):
                    bad += 1
        # phase 1: V band D*2^F + g_ records -> H band
        for y in range(H):
            for x in range(W):
                o = dmm.shard_locate(cfg, rank, world, dmm.LOC_FH_V, y, x)
                if o >= 0:
                    _stamp(ws, o, y, x, 200)
        _exchange(ws, dmm.shard_plan(cfg, rank, world, 1), rank)
        for y in range(H):
            for x in range(W):
                o = dmm.shard_locate(cfg, rank, world, dmm.LOC_FH_H, y, x)
                if o >= 0 and _read(ws, o) != (y, x, 200):
                    bad += 1
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bad))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 3])
def test_plan_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: 0 for r in range(world)}, res
