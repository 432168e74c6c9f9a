"""Randomised GPU-vs-oracle parity (a GPU box; seconds per case): random
shapes, label ranges and regulariser / penalty / refinement parameters for
every path -- the classic pair and int32 kernels, the general penalty with
edge weights, the iterative minorant, flow costs + both layers, stereo and
flow refinement, ROWCOL band sharding at world 1-5 (lockstep in one process)
-- each compared with the oracle exactly as the parity tests do.  Configurations the library rejects (DMM_E_RANGE / DMM_E_ARG) are
skipped and counted.

  python tests/fuzz_parity.py [seconds] [seed] [scale]   (scale multiplies the W / H ranges)

Test infrastructure (it runs the oracle): lives in tests/; a fixed-count run
is part of the GPU suite (tests/test_gpu_fuzz.py).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1601_06274_b200 as dmm  # noqa: E402
from oracle import refine as orf  # noqa: E402


SCALE = 1


class Skip(Exception):
    """A configuration the library rejects at creation (range / argument checks)."""


def mk(**kw):
    try:
        return dmm.Context(**kw)
    except dmm.DmmError as ex:
        raise Skip(str(ex))


def classic(rng):
    W, H = int(rng.integers(1, 300 * SCALE)), int(rng.integers(1, 200 * SCALE))
    K = int(rng.integers(1, 257))
    d_min = int(rng.integers(-8, 9))
    wh, wv, T = int(rng.integers(0, 9)), int(rng.integers(0, 9)), int(rng.integers(1, 12))
    Fb, iters, r = int(rng.choice([0, 4, 8])), int(rng.integers(1, 5)), int(rng.choice([1, 2]))
    kind = str(rng.choice(["rd", "wt-kitti"]))
    pair = bool(rng.integers(0, 2))
    left, right, _ = datagen.pair(kind, W, H, max(K, 2), seed=int(rng.integers(1 << 30)))
    ctx = mk(width=W, height=H, d_min=d_min, d_max=d_min + K - 1, w_h=wh, w_v=wv, T=T, frac_bits=Fb,
             census_radius=r, max_iters=iters)
    ctx.set_pair(pair)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(iters)
    e, b, hist = ctx.result()
    oob = ((2 * r + 1) ** 2 - 1) // 2
    D = oracle.cost_volume(oracle.census(left, r), oracle.census(right, r), d_min, K, oob)
    o = oracle.dmm(D, wh, wv, T, Fb, iters, 8)
    assert np.array_equal(ctx.cost_volume_tensor().cpu().numpy(), D), "D"
    assert np.array_equal(ctx.labels().cpu().numpy().astype(np.int32), o["labels"]), "labels"
    assert hist == [int(v) for v in o["bound_hist"]] and e == o["energy"], "energy / bounds"
    return f"classic {W}x{H}x{K} dmin={d_min} w={wh},{wv} T={T} F={Fb} it={iters} r={r} {ctx.kernel_family()}"


def general(rng):
    W, H = int(rng.integers(1, 200 * SCALE)), int(rng.integers(1, 120 * SCALE))
    K = int(rng.integers(2, 129))
    e2 = int(rng.integers(1, 33))
    e1 = int(rng.integers(0, e2 + 1))
    delta, c = int(rng.integers(0, 5)), int(rng.integers(1, 200))
    ew = bool(rng.integers(0, 2))
    iters = int(rng.integers(1, 4))
    iterative = bool(rng.integers(0, 3) == 0)
    passes, gshift = int(rng.integers(1, 5)), int(rng.integers(0, 4))
    kind = str(rng.choice(["rd", "wt-kitti"]))
    left, right, _ = datagen.pair(kind, W, H, K, seed=int(rng.integers(1 << 30)))
    pen = (e1, e2, delta, c)
    kw = dict(minorant="iterative", iter_passes=passes, iter_gshift=gshift) if iterative else {}
    ctx = mk(width=W, height=H, d_min=0, d_max=K - 1, w_h=2, w_v=3, T=4, max_iters=iters, pen=pen,
             edge_weights=ew, **kw)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(iters)
    e, b, hist = ctx.result()
    D = oracle.cost_volume(oracle.census(left), oracle.census(right), 0, K, 12)
    oh, ov = oracle.edge_weights(left) if ew else (None, None)
    if iterative:
        o = oracle.dmm_minorant(D, 2, 3, pen, 4, iters, 1, passes, gshift, oh, ov, nthreads=8)
    else:
        o = oracle.dmm_general(D, 2, 3, pen, 4, iters, oh, ov, nthreads=8)
    assert np.array_equal(ctx.labels().cpu().numpy().astype(np.int32), o["labels"]), "labels"
    assert hist == [int(v) for v in o["bound_hist"]] and e == o["energy"], "energy / bounds"
    return f"general {W}x{H}x{K} pen={pen} ew={ew} it={iters} {'iterative p=%d g=%d' % (passes, gshift) if iterative else 'hm'}"


def flow(rng):
    W, H = int(rng.integers(2, 150 * SCALE)), int(rng.integers(2, 90 * SCALE))
    K = int(rng.choice([16, 32, 48, 64]))
    u1, u2 = int(rng.integers(-K, 5)), int(rng.integers(-K, 5))
    i1, i2, _, _ = datagen.flow_pair(W, H, min(K // 2, 16), seed=int(rng.integers(1 << 30)))
    ctx = mk(width=W, height=H, d_min=u1, d_max=u1 + K - 1, batch=2, max_iters=3)
    ctx.flow_cost_volume(torch.from_numpy(i1).cuda(), torch.from_numpy(i2).cuda(), u2)
    ctx.solve(3, frame=0, nframes=2)
    c1, c2 = oracle.census(i1), oracle.census(i2)
    f1, f2 = oracle.flow_costs(c1, c2, u1, K, u2, K)
    assert np.array_equal(ctx.cost_volume_tensor(0).cpu().numpy(), f1), "f1"
    assert np.array_equal(ctx.cost_volume_tensor(1).cpu().numpy(), f2), "f2"
    for f, D in ((0, f1), (1, f2)):
        o = oracle.dmm(D, 3, 3, 4, 4, 3, 8)
        assert np.array_equal(ctx.labels(f).cpu().numpy().astype(np.int32), o["labels"]), "flow labels"
    prm = dict(eps=float(rng.uniform(0, 1)), delta=float(rng.uniform(0.2, 3)), C=float(rng.uniform(1, 6)),
               h=float(rng.choice([1.0, 0.5])), tau=float(rng.uniform(0.1, 0.4)), sigma=float(rng.uniform(0.1, 0.4)),
               warps=int(rng.integers(0, 3)), iters=int(rng.integers(0, 10)))
    g1, g2, e = ctx.flow_refine(u2, **prm)
    o1, o2, eo = orf.flow_refine(c1, c2, u1 + ctx.labels(0).cpu().numpy().astype(np.float64),
                                 u2 + ctx.labels(1).cpu().numpy().astype(np.float64), 3.0, 3.0, **prm)
    assert np.array_equal(g1.cpu().numpy(), o1.astype(np.float32)), "flow refine u1"
    assert np.array_equal(g2.cpu().numpy(), o2.astype(np.float32)), "flow refine u2"
    assert abs(e - eo) <= 1e-9 * max(abs(eo), 1.0), "flow refine energy"
    return f"flow {W}x{H} K={K} u=({u1},{u2}) refine {prm}"


def refine(rng):
    W, H = int(rng.integers(1, 200 * SCALE)), int(rng.integers(1, 120 * SCALE))
    K = int(rng.integers(2, 129))
    left, right, _ = datagen.pair("wt-kitti", W, H, K, seed=int(rng.integers(1 << 30)))
    ctx = mk(width=W, height=H, d_min=0, d_max=K - 1, max_iters=2)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(2)
    prm = dict(eps=float(rng.uniform(0, 1)), delta=float(rng.uniform(0.2, 3)), C=float(rng.uniform(1, 6)),
               h=float(rng.choice([1.0, 0.5, 2.0])), tau=float(rng.uniform(0.1, 0.4)),
               sigma=float(rng.uniform(0.1, 0.4)), warps=int(rng.integers(0, 4)), iters=int(rng.integers(0, 14)))
    u, e = ctx.refine(**prm)
    uo, eo = orf.refine(ctx.cost_volume_tensor().cpu().numpy(), ctx.labels().cpu().numpy(), 3.0, 3.0, **prm)
    assert np.array_equal(u.cpu().numpy(), uo.astype(np.float32)), "refine u"
    assert abs(e - eo) <= 1e-9 * max(abs(eo), 1.0), "refine energy"
    return f"refine {W}x{H}x{K} {prm}"


def bands(rng):
    """ROWCOL band sharding, all ranks in one process (the parity tests'
    lockstep: every rank's half-step through the C ABI, the bytes of
    dmm_shard_plan moved between the ranks' workspaces -- data movement only)."""
    from paper_1601_06274_b200 import sharding
    world = int(rng.integers(1, 6))
    W, H = int(rng.integers(world, 160 * SCALE)), int(rng.integers(world, 90 * SCALE))
    K = int(rng.choice([16, 32, 64, 100, 128, 256]))
    iters = int(rng.integers(1, 4))
    kw = dict(d_min=0, d_max=K - 1, w=3, T=4, frac_bits=4, max_iters=iters)
    left, right, _ = datagen.pair("wt-kitti", W, H, K, seed=int(rng.integers(1 << 30)))
    cfg = dmm.make_config(W, H, **kw)
    lt, rt = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
    ctxs = []
    for r in range(world):
        c = mk(width=W, height=H, shard_world=world, **kw)
        try:
            c.shard(None, r, world, dmm.SHARD_ROWCOL)
        except dmm.DmmError as ex:
            raise Skip(str(ex))
        c.cost_volume(lt, rt)
        ctxs.append(c)

    def exchange(phase):
        plans = [dmm.shard_plan(cfg, r, world, phase) for r in range(world)]
        for r in range(world):
            for peer, so, sb, ro, rb in plans[r]:
                pr = plans[peer][r]
                ctxs[peer].ws_view(pr[3], sb).copy_(ctxs[r].ws_view(so, sb))

    for t in range(iters):
        for c in ctxs:
            c.half_step(t, 0, iters)
        if world > 1:
            exchange(0)
        for c in ctxs:
            c.half_step(t, 1, iters)
        if world > 1 and t + 1 < iters:
            exchange(1)
    torch.cuda.synchronize()
    labels = np.zeros((H, W), np.int32)
    hist = np.zeros(2 * iters, np.int64)
    for r, c in enumerate(ctxs):
        boff = dmm.shard_locate(cfg, r, world, dmm.LOC_BOUNDS, 0, 0)
        hist += c.ws_view(boff, 16 * iters).view(torch.int64).cpu().numpy()
        c0, c1 = sharding.bands(W, world)[r]
        off = dmm.shard_locate(cfg, r, world, dmm.LOC_LABEL_V, 0, c0)
        labels[:, c0:c1] = c.ws_view(off, H * (c1 - c0)).view(H, c1 - c0).cpu().numpy()
    D = oracle.cost_volume(oracle.census(left), oracle.census(right), 0, K, 12)
    o = oracle.dmm(D, 3, 3, 4, 4, iters, 8)
    assert np.array_equal(labels, o["labels"]), "band labels"
    assert np.array_equal(hist, o["bound_hist"]), "band bounds"
    return f"bands {W}x{H}x{K} world={world} it={iters}"


def run(budget: float, seed: int, scale: int = 1, max_cases: int = 1 << 30, verbose: bool = True):
    """Random cases until `budget` seconds or `max_cases` cases; raises on the
    first mismatch.  Returns (cases, per-kind counts, rejected)."""
    global SCALE
    SCALE = scale
    rng = np.random.default_rng(seed)
    oracle.build()
    kinds = [classic, classic, general, flow, refine, bands]
    t0 = time.time()
    n = skipped = 0
    counts = {}
    while time.time() - t0 < budget and n < max_cases:
        fn = kinds[int(rng.integers(len(kinds)))]
        try:
            desc = fn(rng)
        except Skip:
            skipped += 1
            continue
        except AssertionError as ex:
            print("MISMATCH", fn.__name__, ex, flush=True)
            raise
        n += 1
        counts[fn.__name__] = counts.get(fn.__name__, 0) + 1
        if verbose and (n <= 5 or n % 25 == 0):
            print(n, desc, flush=True)
    if verbose:
        print(f"fuzz ok: {n} cases {counts}, {skipped} rejected configurations, {time.time() - t0:.0f} s", flush=True)
    return n, counts, skipped


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    run(budget, seed, int(sys.argv[3]) if len(sys.argv) > 3 else 1)


if __name__ == "__main__":
    main()
