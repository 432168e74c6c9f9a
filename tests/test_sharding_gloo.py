"""Multi-rank (N > 1) paths on the CPU: band decomposition of Algorithm 2 with
an all-to-all transpose between half-steps over torch.distributed (gloo,
world size 2 and 3), and the frame assignment of frames mode.

The per-band half-steps here are an oracle engine (test infrastructure:
oracle.hm per chain on dense int64 duals); the transposes, reductions and the
driver are the product code of paper_1601_06274_b200.sharding.  The sharded
result must be bit-identical to the unsharded oracle solve."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

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


class OracleBandEngine:
    """One rank's share of a band-sharded solve, computed with the oracle."""

    def __init__(self, D, w, T, Fb, world, rank):
        import oracle
        self.orc = oracle
        H, W, K = D.shape
        self.row_bands, self.col_bands = sharding.bands(H, world), sharding.bands(W, world)
        self.rank = rank
        (self.r0, self.r1), (self.c0, self.c1) = self.row_bands[rank], self.col_bands[rank]
        self.Ds = torch.from_numpy(D.astype(np.int64) << Fb)
        self.ws, self.T = w << Fb, T
        self.fh_rb = self.Ds[self.r0:self.r1].clone()              # D*2^F + g_ (g_ = 0)
        self.fv_rb = torch.zeros_like(self.fh_rb)
        self.fv_cb = torch.zeros((H, self.c1 - self.c0, K), dtype=torch.int64)
        self.fh_cb = torch.zeros_like(self.fv_cb)
        self.labels = torch.zeros((H, self.c1 - self.c0), dtype=torch.int64)
        self.partial = None

    def half_h(self, t, iterations):
        if self.partial is None:
            self.partial = torch.zeros(2 * iterations, dtype=torch.int64)
        for y in range(self.r1 - self.r0):
            F = self.fh_rb[y].numpy()
            h = self.orc.hm(F, self.ws, self.T)
            # f_ = h - g_ = h - (F - D_s)
            self.fv_rb[y] = torch.from_numpy(h - F) + self.Ds[self.r0 + y]
            self.partial[2 * t] += int(h.min(1).sum())

    def half_v(self, t, iterations):
        for x in range(self.c1 - self.c0):
            F = self.fv_cb[:, x].numpy()
            v = self.orc.hm(F, self.ws, self.T)
            g = torch.from_numpy(v - F)
            self.fh_cb[:, x] = self.Ds[:, self.c0 + x] + g
            self.partial[2 * t + 1] += int(v.min(1).sum())
            if t == iterations - 1:
                self.labels[:, x] = torch.from_numpy(v.argmin(1))

    def fv_rows(self):
        return self.fv_rb

    def set_fv_cols(self, x):
        self.fv_cb.copy_(x)

    def fh_cols(self):
        return self.fh_cb

    def set_fh_rows(self, x):
        self.fh_rb.copy_(x)


def _problem():
    rng = np.random.default_rng(7)
    return rng.integers(0, 25, size=(9, 13, 5)).astype(np.uint8), 3, 2, 4, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        D, w, T, Fb, iters = _problem()
        eng = OracleBandEngine(D, w, T, Fb, world, rank)
        exch = sharding.DistExchanger()
        sharding.band_dmm(eng, exch, iters)
        hist = exch.all_reduce_sum(eng.partial.clone())
        H = D.shape[0]
        wmax = max(c1 - c0 for c0, c1 in eng.col_bands)
        pad = torch.zeros((H, wmax), dtype=torch.int64)
        pad[:, : eng.labels.shape[1]] = eng.labels
        labs = exch.all_gather(pad)
        labels = torch.cat([l[:, : c1 - c0] for l, (c0, c1) in zip(labs, eng.col_bands)], dim=1)
        fpad = torch.zeros((H, wmax, D.shape[2]), dtype=torch.int64)
        fpad[:, : eng.fv_cb.shape[1]] = eng.fv_cb
        fv = torch.cat([f[:, : c1 - c0] for f, (c0, c1) in zip(exch.all_gather(fpad), eng.col_bands)], dim=1)
        if rank == 0:
            q.put((hist.numpy(), labels.numpy(), fv.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_band_sharded_equals_unsharded_gloo(orc, world):
    D, w, T, Fb, iters = _problem()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    hist, labels, fv = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = orc.dmm(D, w, w, T, Fb, iters)
    assert np.array_equal(hist, ref["bound_hist"])
    assert np.array_equal(labels, ref["labels"])
    assert np.array_equal(fv, ref["fdual"])


def test_band_lockstep_equals_unsharded(orc):
    """The same decomposition driven in one process (lockstep_band_dmm)."""
    D, w, T, Fb, iters = _problem()
    for world in (1, 2, 4):
        engines = [OracleBandEngine(D, w, T, Fb, world, r) for r in range(world)]
        sharding.lockstep_band_dmm(engines, iters)
        hist = sum(e.partial for e in engines)
        labels = torch.cat([e.labels for e in engines], dim=1)
        ref = orc.dmm(D, w, w, T, Fb, iters)
        assert np.array_equal(hist.numpy(), ref["bound_hist"])
        assert np.array_equal(labels.numpy(), ref["labels"])
