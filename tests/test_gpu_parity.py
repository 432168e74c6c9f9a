"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element, on seeded synthetic inputs.  All arithmetic is integer, so the bar is
bit-exact for codes, cost volume, duals, labels, bound history and energy
(north_star: "cost volumes and labellings must match the oracle bit-exactly")."""
import numpy as np
import pytest

import datagen

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _ctx(**kw):
    import paper_1601_06274_b200 as dmm
    return dmm.Context(**kw)


def _run_gpu(left, right, d_min, K, w_h, w_v, T, Fb, iters, r=2, oob=-1, pair=True):
    H, W = left.shape
    ctx = _ctx(width=W, height=H, d_min=d_min, d_max=d_min + K - 1, w_h=w_h, w_v=w_v, T=T,
               frac_bits=Fb, census_radius=r, oob_cost=oob, max_iters=max(iters, 1))
    ctx.set_pair(pair)
    if not pair:
        assert ctx.kernel_family() == "int32"
    lt = torch.from_numpy(left).cuda()
    rt = torch.from_numpy(right).cuda()
    ctx.cost_volume(lt, rt)
    ctx.solve(iters)
    e, b, hist = ctx.result()
    out = dict(
        codes_left=ctx.codes(0).cpu().numpy().view(np.uint32),
        codes_right=ctx.codes(1).cpu().numpy().view(np.uint32),
        D=ctx.cost_volume_tensor().cpu().numpy(),
        fdual=ctx.dual(0).cpu().numpy(),
        gdual=ctx.dual(1).cpu().numpy(),
        labels=ctx.labels().cpu().numpy(),
        energy=e, bound=b, bound_hist=np.array(hist, np.int64))
    torch.cuda.synchronize()
    return out


def _run_oracle(orc, left, right, d_min, K, w_h, w_v, T, Fb, iters, r=2, oob=-1, nthreads=4):
    if oob < 0:
        oob = ((2 * r + 1) ** 2 - 1) // 2
    cl, cr = orc.census(left, r), orc.census(right, r)
    D = orc.cost_volume(cl, cr, d_min, K, oob)
    out = orc.dmm(D, w_h, w_v, T, Fb, iters, nthreads)
    out.update(codes_left=cl, codes_right=cr, D=D)
    return out


def _compare(g, o):
    assert np.array_equal(g["codes_left"], o["codes_left"])
    assert np.array_equal(g["codes_right"], o["codes_right"])
    assert np.array_equal(g["D"], o["D"])
    assert np.array_equal(g["fdual"].astype(np.int64), o["fdual"]), "f_ mismatch"
    assert np.array_equal(g["gdual"].astype(np.int64), o["gdual"]), "g_ mismatch"
    assert np.array_equal(g["bound_hist"], o["bound_hist"])
    assert np.array_equal(g["labels"].astype(np.int32), o["labels"])
    assert g["energy"] == o["energy"]
    assert g["bound"] == o["bound_hist"][-1]


def test_c1_random_dot(orc):
    """configs[0]: 64x48 random-dot, 16 disparities, truncated linear, 5 iterations."""
    c = datagen.CONFIGS["C1"]
    left, right, _ = datagen.pair(c["kind"], c["W"], c["H"], c["K"], 0)
    args = (c["d_min"], c["K"], 3, 3, 4, 4, c["iters"])
    _compare(_run_gpu(left, right, *args), _run_oracle(orc, left, right, *args))


CASES = [
    # (W, H, K, d_min, w_h, w_v, T, Fb, iters, r, kind)
    (37, 29, 5, 0, 2, 3, 2, 4, 2, 2, "rd"),
    (100, 20, 33, 0, 3, 3, 4, 4, 3, 2, "rd"),       # ragged K (pads), ragged W
    (70, 41, 64, -3, 1, 4, 1, 0, 2, 1, "rd"),       # Potts, F = 0, negative d_min, 3x3 census
    (129, 65, 128, 0, 3, 3, 4, 4, 2, 2, "wt-kitti"),
    (61, 33, 100, 2, 5, 2, 7, 8, 2, 2, "rd"),       # F = 8
    (50, 47, 200, 0, 3, 3, 4, 4, 1, 2, "wt-middlebury"),
    (40, 23, 256, 0, 2, 2, 300, 4, 2, 2, "wt-middlebury"),   # T >= K (untruncated)
    (300, 7, 32, 0, 0, 0, 4, 4, 2, 2, "rd"),        # w = 0 (WTA)
    (1, 50, 8, 0, 3, 3, 2, 4, 2, 2, "rd"),          # W = 1
    (50, 1, 8, 0, 3, 3, 2, 4, 2, 2, "rd"),          # H = 1
    (1, 1, 1, 0, 3, 3, 1, 4, 1, 2, "rd"),           # single pixel, K = 1
    (2, 2, 2, 0, 9, 9, 1, 4, 3, 1, "rd"),
    (1025, 3, 16, 0, 3, 3, 4, 4, 2, 2, "rd"),       # long rows, odd splits
    (5, 513, 16, 0, 3, 3, 4, 4, 2, 2, "rd"),        # long columns
    (1500, 24, 256, 0, 3, 3, 4, 4, 2, 2, "wt-middlebury"),   # C3 row length and K
    # C3's K = 256 with tall columns: the V level kernels (LPL = 8) run at
    # levels >= 1 (leaf level 7 at H = 1000, 6 at H = 700)
    (7, 1000, 256, 0, 3, 3, 4, 4, 2, 2, "wt-middlebury"),
    (9, 700, 256, 0, 3, 3, 4, 4, 2, 2, "wt-middlebury"),
    (33, 1000, 200, 0, 2, 3, 3, 4, 2, 2, "wt-middlebury"),   # padded K = 200 -> 256, odd W (self-paired chain)
    (16384, 3, 16, 0, 3, 3, 4, 4, 2, 2, "rd"),      # maximum width (capi.cu valid: W <= 16384)
    (3, 16384, 16, 0, 3, 3, 4, 4, 2, 2, "rd"),      # maximum height
]


@pytest.mark.parametrize("family", ["auto", "int32"])
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}xK{c[2]}" for c in CASES])
def test_parity_cases(orc, case, family):
    """Both kernel families (packed chain pairs where the range check allows
    them, and the one-chain int32 kernels) against the oracle."""
    W, H, K, d_min, w_h, w_v, T, Fb, iters, r, kind = case
    left, right, _ = datagen.pair(kind, W, H, K, seed=W * 7 + H)
    args = (d_min, K, w_h, w_v, T, Fb, iters, r)
    _compare(_run_gpu(left, right, *args, pair=(family == "auto")), _run_oracle(orc, left, right, *args))


def test_kernel_family_selection():
    """The packed pair kernels serve the benchmark configurations; a regulariser
    too large for 16-bit operands falls back to int32 (range check, capi.cu)."""
    c2 = _ctx(width=64, height=8, d_min=0, d_max=127, w=3, T=4, frac_bits=4)
    assert c2.kernel_family() == "pair"
    c3 = _ctx(width=64, height=8, d_min=0, d_max=255, w=3, T=4, frac_bits=4)
    assert c3.kernel_family() == "pair"
    big = _ctx(width=64, height=8, d_min=0, d_max=99, w_h=5, w_v=2, T=7, frac_bits=8)
    assert big.kernel_family() == "int32"
    oob = _ctx(width=64, height=8, d_min=0, d_max=15, w=1, T=1, frac_bits=0, oob_cost=200)
    assert oob.kernel_family() == "int32"      # D >= 128: packed D unpack needs D < 128
    c2.set_pair(False)
    assert c2.kernel_family() == "int32"


def test_batched_frames_equal_single(orc):
    """Frames solved in one batched launch equal frames solved one by one."""
    W, H, K = 90, 40, 24
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w=3, T=4, batch=3, max_iters=3)
    pairs = [datagen.pair("rd", W, H, K, s) for s in range(3)]
    for f, (l, r, _) in enumerate(pairs):
        ctx.cost_volume(torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda(), frame=f)
    ctx.solve(3, frame=0, nframes=3)
    for f, (l, r, _) in enumerate(pairs):
        e, b, hist = ctx.result(frame=f)
        o = _run_oracle(orc, l, r, 0, K, 3, 3, 4, 4, 3)
        assert np.array_equal(np.array(hist), o["bound_hist"])
        assert e == o["energy"]
        assert np.array_equal(ctx.labels(frame=f).cpu().numpy().astype(np.int32), o["labels"])


def test_run_host_matches_device_path(orc):
    W, H, K = 120, 60, 32
    l, r, _ = datagen.pair("wt-kitti", W, H, K, 5)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w=3, T=4, max_iters=4)
    lab, e, b = ctx.run_host(l, r, 4)
    o = _run_oracle(orc, l, r, 0, K, 3, 3, 4, 4, 4)
    assert np.array_equal(lab.numpy().astype(np.int32), o["labels"])
    assert e == o["energy"] and b == o["bound_hist"][-1]


@pytest.mark.parametrize("orient", ["row", "column"])
def test_hm_golden_chains_gpu(orient):
    """tests/golden/hm_chains.json (n = 7, 13, 25; F = 0, 4; oracle-written,
    pinned in test_oracle_chain.py) through the device path: a 1-row frame's
    f_ after H_1 is HM(D*2^F) (g_ = 0, R4); a 1-column frame's g_ after V_1 is
    HM(D*2^F) - D*2^F (the H pass of single nodes gives f_ = D*2^F)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "hm_chains.json")) as f:
        g = json.load(f)
    for c in g["chains"]:
        n, Fb = c["n"], c["F"]
        D = np.array(c["D"], np.uint8)
        lam = np.array(c["lam"], np.int64)
        W, H = (n, 1) if orient == "row" else (1, n)
        ctx = _ctx(width=W, height=H, d_min=0, d_max=g["K"] - 1, w=g["w"], T=g["T"], frac_bits=Fb, max_iters=1)
        ctx.import_cost_volume(torch.from_numpy(D.reshape(H, W, g["K"])).cuda())
        ctx.solve(1)
        e, b, hist = ctx.result()
        if orient == "row":
            got = ctx.dual(0).cpu().numpy().reshape(n, -1).astype(np.int64)
            assert np.array_equal(got, lam), (n, Fb)
            assert hist[0] == c["opt"]
        else:
            got = ctx.dual(1).cpu().numpy().reshape(n, -1).astype(np.int64)
            assert np.array_equal(got, lam - (D.astype(np.int64) << Fb)), (n, Fb)
            assert hist[1] == c["opt"]


def test_deterministic_repeat():
    W, H, K = 200, 90, 64
    l, r, _ = datagen.pair("rd", W, H, K, 9)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, max_iters=4)
    outs = []
    for _ in range(3):
        ctx.cost_volume(torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda())
        ctx.solve(4)
        outs.append((ctx.result(), ctx.labels().cpu().numpy(), ctx.dual(1).cpu().numpy()))
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        assert np.array_equal(o[1], outs[0][1]) and np.array_equal(o[2], outs[0][2])


def test_errors():
    import paper_1601_06274_b200 as dmm
    ctx = _ctx(width=16, height=8, d_min=0, d_max=7, max_iters=2)
    with pytest.raises(dmm.DmmError):
        ctx.solve(1)                       # before the cost volume -> DMM_E_STATE
    z = torch.zeros((8, 16), dtype=torch.uint8, device="cuda")
    ctx.cost_volume(z, z)
    with pytest.raises(dmm.DmmError):
        ctx.solve(0)                       # iterations = 0 -> DMM_E_ARG
    with pytest.raises(dmm.DmmError):
        ctx.solve(3)                       # > max_iters
    with pytest.raises(dmm.DmmError):
        dmm.Context(width=16, height=8, d_min=0, d_max=300)   # K > 256


@pytest.mark.parametrize("w,T,family", [(6, 3, "pair"), (6, 4, "int32")])
def test_pair_range_edge(orc, w, T, family):
    """At the edge of the packed 16-bit range check (w=6, T=3, F=4:
    16*960 + 3*288 + 4 = 16228 <= 16383) the pair kernels still run and stay
    exact; one step beyond (T=4) the int32 kernels take over."""
    W, H, K, iters = 90, 31, 64, 3
    left, right, _ = datagen.pair("rd", W, H, K, seed=77)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w=w, T=T, frac_bits=4, max_iters=iters)
    assert ctx.kernel_family() == family
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(iters)
    e, b, hist = ctx.result()
    o = _run_oracle(orc, left, right, 0, K, w, w, T, 4, iters)
    assert np.array_equal(ctx.dual(0).cpu().numpy().astype(np.int64), o["fdual"])
    assert np.array_equal(ctx.dual(1).cpu().numpy().astype(np.int64), o["gdual"])
    assert np.array_equal(ctx.labels().cpu().numpy().astype(np.int32), o["labels"])
    assert np.array_equal(np.array(hist), o["bound_hist"]) and e == o["energy"]


def test_frame_stack_apis(orc):
    """dmm_cost_volume_frames + dmm_solve(nframes) and dmm_run_host_frames
    (configs[4]-style streams) equal the oracle frame by frame."""
    W, H, K, iters, n = 70, 37, 32, 3, 3
    pairs = [datagen.pair("wt-kitti", W, H, K, seed=20 + s) for s in range(n)]
    L = torch.from_numpy(np.stack([p[0] for p in pairs]))
    R = torch.from_numpy(np.stack([p[1] for p in pairs]))
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w=3, T=4, batch=n, max_iters=iters)
    ctx.cost_volume_frames(L.cuda(), R.cuda())
    ctx.solve(iters, frame=0, nframes=n)
    orcs = [_run_oracle(orc, p[0], p[1], 0, K, 3, 3, 4, 4, iters) for p in pairs]
    for f in range(n):
        e, b, hist = ctx.result(frame=f)
        assert np.array_equal(ctx.labels(frame=f).cpu().numpy().astype(np.int32), orcs[f]["labels"])
        assert np.array_equal(np.array(hist), orcs[f]["bound_hist"]) and e == orcs[f]["energy"]
    lab, es, bs = ctx.run_host_frames(L.pin_memory(), R.pin_memory(), iters)
    for f in range(n):
        assert np.array_equal(lab[f].numpy().astype(np.int32), orcs[f]["labels"])
        assert es[f] == orcs[f]["energy"] and bs[f] == orcs[f]["bound_hist"][-1]


@pytest.mark.slow
def test_c2_full_size(orc):
    """configs[1] at full size (1242x375x128, 4 iterations), in the launch
    configuration bench.py times: complete element-by-element comparison."""
    c = datagen.CONFIGS["C2"]
    left, right, _ = datagen.pair(c["kind"], c["W"], c["H"], c["K"], 0)
    args = (c["d_min"], c["K"], 3, 3, 4, 4, c["iters"])
    g = _run_gpu(left, right, *args)
    o = _run_oracle(orc, left, right, *args, nthreads=max(1, min(16, __import__("os").cpu_count() or 1)))
    _compare(g, o)


@pytest.mark.slow
def test_c5_batch_full_size(orc):
    """configs[4] per GPU at full size in bench.py's launch configuration: 64
    KITTI-shaped frames (8 distinct pairs, cycled as bench.py does) solved as
    one batch.  Sampled frames (three distinct pairs, at batch positions 0,
    9 and 63) element by element against the oracle; every frame equals the
    other copies of its pair (batch position does not matter) and satisfies
    the bound <= energy and monotone-history properties."""
    import os
    c = datagen.CONFIGS["C5"]
    W, H, K, iters, nf = c["W"], c["H"], c["K"], c["iters"], c["frames"]
    pairs = [datagen.pair(c["kind"], W, H, K, seed=s) for s in range(8)]
    Lh = np.stack([pairs[f % 8][0] for f in range(nf)])
    Rh = np.stack([pairs[f % 8][1] for f in range(nf)])
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w=3, T=4, frac_bits=4, max_iters=iters, batch=nf)
    ctx.cost_volume_frames(torch.from_numpy(Lh).cuda(), torch.from_numpy(Rh).cuda())
    ctx.solve(iters, frame=0, nframes=nf)
    res = [ctx.result(f) for f in range(nf)]
    labs = [ctx.labels(f).cpu().numpy() for f in range(nf)]
    for f in range(nf):
        e, b, hist = res[f]
        assert b <= e and all(x <= y for x, y in zip(hist, hist[1:]))
        if f >= 8:
            assert res[f] == res[f % 8] and np.array_equal(labs[f], labs[f % 8])
    nth = max(1, min(16, os.cpu_count() or 1))
    for f in (0, 9, 63):
        l, r, _ = pairs[f % 8]
        o = _run_oracle(orc, l, r, 0, K, 3, 3, 4, 4, iters, nthreads=nth)
        e, b, hist = res[f]
        assert np.array_equal(labs[f].astype(np.int32), o["labels"])
        assert e == o["energy"] and np.array_equal(np.array(hist, np.int64), o["bound_hist"])


@pytest.mark.slow
def test_c3_full_size(orc):
    """configs[2] at full size on one GPU (1500x1000x256, 4 iterations, the
    launch configuration bench.py --config C3 times): complete element-by-
    element comparison of codes, D, f_, g_, labels, bound history, energy."""
    import os
    c = datagen.CONFIGS["C3"]
    left, right, _ = datagen.pair(c["kind"], c["W"], c["H"], c["K"], 0)
    args = (c["d_min"], c["K"], 3, 3, 4, 4, c["iters"])
    g = _run_gpu(left, right, *args)
    o = _run_oracle(orc, left, right, *args, nthreads=max(1, os.cpu_count() or 1))
    _compare(g, o)


@pytest.mark.slow
def test_c2_full_size_deterministic_records():
    """Ten full C2 solves (bench launch configuration) produce byte-identical
    dual records (f_ and D*2^F + g_, the whole workspace arrays the kernels
    write, pads excluded), labels and bound histories: no race between the
    level / leaf kernels, PDL prologues and the TMA staging."""
    import paper_1601_06274_b200 as dmm
    c = datagen.CONFIGS["C2"]
    left, right, _ = datagen.pair(c["kind"], c["W"], c["H"], c["K"], 0)
    ctx = _ctx(width=c["W"], height=c["H"], d_min=0, d_max=c["K"] - 1, w=3, T=4, frac_bits=4,
               max_iters=c["iters"])
    lt, rt = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
    ref = None
    nb = 2 * 128 + 4                      # u16 spans + int32 base of each record
    for _ in range(10):
        ctx.cost_volume(lt, rt)
        ctx.solve(c["iters"])
        cur = (ctx.buffer(dmm.BUF_FV)[:, :, :nb].clone(), ctx.buffer(dmm.BUF_FH)[:, :, :nb].clone(),
               ctx.labels(), ctx.result())
        if ref is None:
            ref = cur
        else:
            assert torch.equal(cur[0], ref[0]) and torch.equal(cur[1], ref[1])
            assert torch.equal(cur[2], ref[2]) and cur[3] == ref[3]


# ---------------------------------------------------------------- primitives
@pytest.mark.parametrize("K", [1, 5, 16, 31, 32, 33, 64, 100, 128, 129, 200, 256])
def test_msg_primitive(orc, K):
    """Device Msg vs the oracle's Msg, all code paths:
    padding (K < 32*LPL), one-hop window (T <= LPL+1) and full scan."""
    import paper_1601_06274_b200 as dmm
    rng = np.random.default_rng(K)
    for T in sorted({1, 2, 3, 4, 5, 8, 9, K, K + 3}):
        for ws in (0, 1, 48, 4080):
            a = rng.integers(-200000, 200000, size=(64, K))
            g = dmm.msg(torch.from_numpy(a.astype(np.int32)).cuda(), ws, T).cpu().numpy()
            o = np.stack([orc.msg(v, ws, T) for v in a])
            assert np.array_equal(g.astype(np.int64), o), (K, T, ws)


@pytest.mark.parametrize("K", [3, 32, 64, 128, 256])
def test_handshake_primitive(orc, K):
    """Device Handshake vs Alg.5 written with the oracle's
    Msg (reading R9: floor halving)."""
    import paper_1601_06274_b200 as dmm
    rng = np.random.default_rng(100 + K)
    for T in (1, 4, 7):
        ws = 48
        Fi, Fj, pL, pR = (rng.integers(-5000, 5000, size=(32, K)) for _ in range(4))
        gij, gji = dmm.handshake(*(torch.from_numpy(x.astype(np.int32)).cuda() for x in (Fi, Fj, pL, pR)), ws, T)
        for v in range(32):
            pji = orc.msg(Fj[v] + pR[v], ws, T)
            m = pL[v] + Fi[v] + pji
            pij = orc.msg(np.floor_divide(m - 2 * pji, 2), ws, T)
            pji2 = orc.msg(-pij, ws, T)
            assert np.array_equal(gij[v].cpu().numpy(), pij) and np.array_equal(gji[v].cpu().numpy(), pji2)


# ------------------------------------------------------- band sharding (8e)
def _rowcol_lockstep(cfg_kw, left, right, iters, world):
    """All ranks' ROWCOL contexts in one process (external transport): every
    rank runs its band half-step through dmm_half_step, then the test moves
    the bytes of dmm_shard_plan between the ranks' workspaces (pure data
    movement, no kernel waits on another rank).  Returns the assembled
    labelling and the summed bound history."""
    import paper_1601_06274_b200 as dmm
    H, W = left.shape
    cfg = dmm.make_config(W, H, **cfg_kw)
    lt, rt = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
    ctxs = []
    for r in range(world):
        c = _ctx(width=W, height=H, shard_world=world, **cfg_kw)
        c.shard(None, r, world, dmm.SHARD_ROWCOL)
        c.cost_volume(lt, rt)
        ctxs.append(c)

    def exchange(phase):
        plans = [dmm.shard_plan(cfg, r, world, phase) for r in range(world)]
        for r in range(world):
            for peer, so, sb, ro, rb in plans[r]:
                # rank r sends [so, so+sb) to peer; peer receives it at its recv offset from r
                pr = plans[peer][r]
                assert pr[4] == sb
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
        c0, c1 = sharding_bands(W, world)[r]
        off = dmm.shard_locate(cfg, r, world, dmm.LOC_LABEL_V, 0, c0)
        labels[:, c0:c1] = c.ws_view(off, H * (c1 - c0)).view(H, c1 - c0).cpu().numpy()
    return labels, hist


def sharding_bands(n, world):
    from paper_1601_06274_b200 import sharding
    return sharding.bands(n, world)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_rowcol_lockstep_equals_oracle(orc, world):
    """ROWCOL band sharding through the C ABI (dmm_shard, dmm_half_step,
    dmm_shard_plan; segmented H records written by the kernels' bulk stores):
    labels and the whole bound history bit-identical to the oracle."""
    W, H, K, iters = 131, 47, 64, 3
    left, right, _ = datagen.pair("wt-kitti", W, H, K, seed=11)
    labels, hist = _rowcol_lockstep(dict(d_min=0, d_max=K - 1, w=3, T=4, frac_bits=4, max_iters=iters),
                                    left, right, iters, world)
    o = _run_oracle(orc, left, right, 0, K, 3, 3, 4, 4, iters)
    assert np.array_equal(labels, o["labels"])
    assert np.array_equal(hist, o["bound_hist"])


def test_rowcol_lockstep_c3_shape(orc):
    """K = 256, bands crossing the leaf blocks at segment edges (world 3 of a
    70-wide frame: segments of 24/23/23 columns), 2 iterations."""
    W, H, K, iters = 70, 41, 256, 2
    left, right, _ = datagen.pair("wt-middlebury", W, H, K, seed=4)
    labels, hist = _rowcol_lockstep(dict(d_min=0, d_max=K - 1, w=3, T=4, frac_bits=4, max_iters=iters),
                                    left, right, iters, 3)
    o = _run_oracle(orc, left, right, 0, K, 3, 3, 4, 4, iters)
    assert np.array_equal(labels, o["labels"])
    assert np.array_equal(hist, o["bound_hist"])


def test_rowcol_nccl_world1(orc):
    """The NCCL path on one GPU: dmm_nccl_unique_id + dmm_shard(ROWCOL, world 1)
    + dmm_solve (all-reduce of bounds / energy, labels) == the oracle, and the
    host-buffer end-to-end call on the sharded context."""
    import paper_1601_06274_b200 as dmm
    W, H, K, iters = 96, 40, 48, 3
    left, right, _ = datagen.pair("rd", W, H, K, seed=9)
    c = _ctx(width=W, height=H, d_min=0, d_max=K - 1, max_iters=iters, shard_world=1)
    c.shard(dmm.nccl_unique_id(), 0, 1, dmm.SHARD_ROWCOL)
    c.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    c.solve(iters)
    e, b, hist = c.result()
    o = _run_oracle(orc, left, right, 0, K, 3, 3, 4, 4, iters)
    assert np.array_equal(c.labels().cpu().numpy().astype(np.int32), o["labels"])
    assert hist == [int(v) for v in o["bound_hist"]] and e == o["energy"]
    lab, e2, b2 = c.run_host(left, right, iters)
    assert np.array_equal(lab.numpy().astype(np.int32), o["labels"]) and (e2, b2) == (e, b)
    with pytest.raises(dmm.DmmError):
        c.dual(0)


def test_primitive_buffers_and_half_steps(orc):
    """dmm_half_step x 2*iters == dmm_solve (same records, bounds, labels)."""
    W, H, K, iters = 70, 33, 32, 3
    left, right, _ = datagen.pair("rd", W, H, K, seed=3)
    lt, rt = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
    import paper_1601_06274_b200 as dmm
    a = _ctx(width=W, height=H, d_min=0, d_max=K - 1, max_iters=iters)
    b = _ctx(width=W, height=H, d_min=0, d_max=K - 1, max_iters=iters)
    a.cost_volume(lt, rt)
    a.solve(iters)
    b.import_cost_volume(a.cost_volume_tensor())
    for t in range(iters):
        b.half_step(t, 0, iters)
        b.half_step(t, 1, iters)
    torch.cuda.synchronize()
    # records' 12 pad bytes are never written: compare the decoded duals
    assert torch.equal(a.dual(0), b.dual(0)) and torch.equal(a.dual(1), b.dual(1))
    assert torch.equal(a.buffer(dmm.BUF_FV)[:, :, : 2 * 32 + 4], b.buffer(dmm.BUF_FV)[:, :, : 2 * 32 + 4])
    assert torch.equal(a.labels(), b.labels())
    assert a.result()[2] == [int(v) for v in b.bound_slots()[: 2 * iters].tolist()]
    assert a.result()[0] == b.energy()


def test_energy_of_arbitrary_labelling(orc):
    """dmm_energy_of (SPEC S:62-70 energy_evaluate; Eq.3) on random and
    constant labellings equals the oracle's energy; labels >= K are rejected."""
    import paper_1601_06274_b200 as dmm
    W, H, K = 97, 41, 40
    left, right, _ = datagen.pair("rd", W, H, K, seed=5)
    ctx = _ctx(width=W, height=H, d_min=-3, d_max=K - 4, w_h=2, w_v=5, T=3, frac_bits=3)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    D = ctx.cost_volume_tensor().cpu().numpy()
    rng = np.random.default_rng(0)
    for lab in (rng.integers(0, K, size=(H, W)), np.zeros((H, W), np.int64), np.full((H, W), K - 1)):
        lt = torch.from_numpy(lab.astype(np.uint8)).cuda()
        assert ctx.energy(labels=lt) == orc.energy(D, lab.astype(np.int32), 2, 5, 3) << 3
    bad = torch.full((H, W), K, dtype=torch.uint8, device="cuda")
    with pytest.raises(dmm.DmmError):
        ctx.energy(labels=bad)


def test_partial_solve_has_no_result():
    """DMM_TUNE_DEBUG_STOP_AFTER_H: f_ after H_1 is readable, the result is not."""
    import paper_1601_06274_b200 as dmm
    W, H, K = 40, 20, 16
    left, right, _ = datagen.pair("rd", W, H, K, seed=2)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, max_iters=2)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.set_stop_after_h(True)
    ctx.solve(2)
    ctx.dual(0)
    for call in (lambda: ctx.result(), lambda: ctx.labels(), lambda: ctx.dual(1)):
        with pytest.raises(dmm.DmmError):
            call()
    ctx.set_stop_after_h(False)
    ctx.solve(2)
    assert ctx.result()[1] <= ctx.result()[0]


# ------------------------------------------------------------ NEXT-1 flow
def _flow_gpu(i1, i2, K, u1_min, u2_min, iters, **kw):
    H, W = i1.shape
    ctx = _ctx(width=W, height=H, d_min=u1_min, d_max=u1_min + K - 1, batch=2, max_iters=max(iters, 1), **kw)
    ctx.flow_cost_volume(torch.from_numpy(i1).cuda(), torch.from_numpy(i2).cuda(), u2_min)
    f1 = ctx.cost_volume_tensor(0).cpu().numpy()
    f2 = ctx.cost_volume_tensor(1).cpu().numpy()
    out = dict(f1=f1, f2=f2)
    if iters:
        ctx.solve(iters, frame=0, nframes=2)
        for f in (0, 1):
            e, b, h = ctx.result(f)
            out[f] = dict(labels=ctx.labels(f).cpu().numpy().astype(np.int32), energy=e, hist=np.array(h, np.int64))
    return out


@pytest.mark.parametrize("W,H,K,u1,u2", [(77, 45, 32, -16, -16), (40, 70, 16, -3, -12), (131, 29, 64, -40, -20),
                                         (33, 33, 48, 5, -60), (16, 9, 32, -16, -16)])
def test_flow_costs_parity(orc, W, H, K, u1, u2):
    """dmm_flow_cost_volume (fused 2-D window kernel) == oracle_flow_costs,
    bit-exact: interior and border tiles, windows partly / wholly outside."""
    i1, i2, _, _ = datagen.flow_pair(W, H, 16, seed=W + H)
    g = _flow_gpu(i1, i2, K, u1, u2, 0)
    of1, of2 = orc.flow_costs(orc.census(i1), orc.census(i2), u1, K, u2, K)
    assert np.array_equal(g["f1"], of1)
    assert np.array_equal(g["f2"], of2)


def test_flow_c4_full_size(orc):
    """configs[3] (C4) at full size: 1242x375, 32x32 window, both layers' Dual MM
    (4 iterations, solved as two frames of one context) bit-exact vs the oracle."""
    c = datagen.CONFIGS["C4"]
    W, H, K, iters = c["W"], c["H"], c["K"], c["iters"]
    i1, i2, _, _ = datagen.flow_pair(W, H, 16, seed=0)
    g = _flow_gpu(i1, i2, K, -16, -16, iters)
    of1, of2 = orc.flow_costs(orc.census(i1), orc.census(i2), -16, K, -16, K)
    assert np.array_equal(g["f1"], of1) and np.array_equal(g["f2"], of2)
    for f, D in ((0, of1), (1, of2)):
        o = orc.dmm(D, 3, 3, 4, 4, iters, nthreads=16)
        assert np.array_equal(g[f]["labels"], o["labels"])
        assert np.array_equal(g[f]["hist"], o["bound_hist"])
        assert g[f]["energy"] == o["energy"]


def test_flow_rejects_bad_window():
    import paper_1601_06274_b200 as dmm
    i1 = np.zeros((20, 30), np.uint8)
    ctx = _ctx(width=30, height=20, d_min=0, d_max=19, batch=2)
    with pytest.raises(dmm.DmmError):
        ctx.flow_cost_volume(torch.from_numpy(i1).cuda(), torch.from_numpy(i1).cuda(), 0)
    ctx1 = _ctx(width=30, height=20, d_min=0, d_max=15, batch=1)
    with pytest.raises(dmm.DmmError):
        ctx1.flow_cost_volume(torch.from_numpy(i1).cuda(), torch.from_numpy(i1).cuda(), 0)


# ------------------------------------------------- NEXT-2 continuous refinement
REFINE_U_TOL = 0.0        # float64 on both sides, same operation order, no FMA contraction: bit-exact u
REFINE_E_RTOL = 1e-9


@pytest.mark.parametrize("W,H,K,eps,delta,C,warps,iters,h,tau,sigma", [
    (96, 40, 32, 1.0, 1.0, 4.0, 5, 40, 1.0, 0.35, 0.35),
    (61, 23, 48, 0.5, 2.0, 5.0, 3, 25, 1.0, 0.35, 0.35),
    (33, 17, 16, 0.25, 1.0, 3.0, 2, 7, 1.0, 0.35, 0.35),
    (70, 45, 32, 0.5, 1.5, 4.5, 3, 13, 0.5, 0.2, 0.6),       # half-label trust region, other steps
])
def test_refine_parity(orc, W, H, K, eps, delta, C, warps, iters, h, tau, sigma):
    """dmm_refine (float64, CUDA graph of the PDHG iterations) vs the float64
    oracle (oracle/refine.py) started from the same discrete labelling.  The
    refined u is returned as float32: compared within its rounding."""
    from oracle import refine as orf
    left, right, _ = datagen.pair("wt-kitti", W, H, K, seed=W)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, max_iters=4)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(4)
    u, e = ctx.refine(eps=eps, delta=delta, C=C, warps=warps, iters=iters, h=h, tau=tau, sigma=sigma)
    D = ctx.cost_volume_tensor().cpu().numpy()
    lab = ctx.labels().cpu().numpy()
    uo, eo = orf.refine(D, lab, 3.0, 3.0, eps=eps, delta=delta, C=C, warps=warps, iters=iters, h=h, tau=tau,
                        sigma=sigma)
    du = np.abs(u.cpu().numpy().astype(np.float64) - uo)
    print(f"refine max |du| = {du.max():.3e}, energy {e:.6f} vs {eo:.6f} (rel {abs(e - eo) / abs(eo):.2e})")
    # u is returned in float32: compare with the oracle's float64 u rounded to float32
    assert np.array_equal(u.cpu().numpy(), uo.astype(np.float32)), du.max()
    assert abs(e - eo) <= REFINE_E_RTOL * abs(eo)
    # a second call with the same parameters replays the cached graph: same u
    # (the energy's double atomics may add in another order: last-bit only)
    u2, e2 = ctx.refine(eps=eps, delta=delta, C=C, warps=warps, iters=iters, h=h, tau=tau, sigma=sigma)
    assert torch.equal(u, u2) and abs(e2 - e) <= 1e-12 * abs(e)


def test_refine_c2_full_size(orc):
    """configs[1] shape: DMM (4 iterations) then 5 x 40 refinement iterations
    (the paper's timing run), float64 vs the float64 oracle."""
    from oracle import refine as orf
    c = datagen.CONFIGS["C2"]
    W, H, K = c["W"], c["H"], c["K"]
    left, right, _ = datagen.pair("wt-kitti", W, H, K, seed=0)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, max_iters=4)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(4)
    u, e = ctx.refine()
    uo, eo = orf.refine(ctx.cost_volume_tensor().cpu().numpy(), ctx.labels().cpu().numpy(), 3.0, 3.0, C=4.0)
    du = np.abs(u.cpu().numpy().astype(np.float64) - uo)
    assert np.array_equal(u.cpu().numpy(), uo.astype(np.float32)), du.max()
    assert abs(e - eo) <= REFINE_E_RTOL * abs(eo)


def _flow_refine_case(orc, W, H, K, u1_min, u2_min, prm):
    from oracle import refine as orf
    i1, i2, _, _ = datagen.flow_pair(W, H, min(K // 2, 16), seed=W * 7 + H)
    ctx = _ctx(width=W, height=H, d_min=u1_min, d_max=u1_min + K - 1, batch=2, max_iters=4)
    ctx.flow_cost_volume(torch.from_numpy(i1).cuda(), torch.from_numpy(i2).cuda(), u2_min)
    ctx.solve(4, frame=0, nframes=2)
    g1, g2, e = ctx.flow_refine(u2_min, **prm)
    u1 = u1_min + ctx.labels(0).cpu().numpy().astype(np.float64)
    u2 = u2_min + ctx.labels(1).cpu().numpy().astype(np.float64)
    o1, o2, eo = orf.flow_refine(orc.census(i1), orc.census(i2), u1, u2, 3.0, 3.0, **prm)
    return ctx, (g1, g2, e), (o1, o2, eo)


@pytest.mark.parametrize("W,H,K,u1,u2,prm", [
    (77, 45, 32, -16, -16, dict(C=4.0)),
    (61, 23, 16, -8, -3, dict(eps=0.5, delta=2.0, C=5.0, warps=3, iters=25)),
    (40, 70, 48, -20, -30, dict(eps=0.25, delta=1.0, C=3.0, warps=2, iters=7, tau=0.2, sigma=0.5)),
    (66, 50, 32, -16, -16, dict(C=4.0, warps=3, iters=10, h=0.5))])          # half-pixel differences
def test_flow_refine_parity(orc, W, H, K, u1, u2, prm):
    """dmm_flow_refine (quadratic model of Eq. 19 rebuilt per warp, Eq. 20's
    prox, float64 without FMA) vs oracle.refine.flow_refine from the same two
    discrete layers: u1, u2 bit-exact after rounding to float32."""
    ctx, (g1, g2, e), (o1, o2, eo) = _flow_refine_case(orc, W, H, K, u1, u2, prm)
    assert np.array_equal(g1.cpu().numpy(), o1.astype(np.float32))
    assert np.array_equal(g2.cpu().numpy(), o2.astype(np.float32))
    assert abs(e - eo) <= REFINE_E_RTOL * abs(eo)
    h1, h2, e2 = ctx.flow_refine(u2, **prm)              # replays the cached graph
    assert torch.equal(g1, h1) and torch.equal(g2, h2) and abs(e2 - e) <= 1e-12 * abs(e)


@pytest.mark.parametrize("W,H", [(1, 23), (37, 1), (2, 2), (65, 41), (57, 33), (16384, 3), (3, 4000)])
def test_refine_degenerate_shapes(orc, W, H):
    """Refinement on single-row / single-column frames and on frames one pixel
    past a tile boundary (stereo tile 56 x 32 inner, flow 56 x 16), iteration
    counts that are not multiples of the 4 iterations per tile launch."""
    from oracle import refine as orf
    left, right, _ = datagen.pair("wt-kitti", W, H, 16, seed=W * 31 + H)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=15, max_iters=2)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(2)
    u, e = ctx.refine(eps=0.5, delta=2.0, C=5.0, warps=2, iters=9)
    uo, eo = orf.refine(ctx.cost_volume_tensor().cpu().numpy(), ctx.labels().cpu().numpy(), 3.0, 3.0,
                        eps=0.5, delta=2.0, C=5.0, warps=2, iters=9)
    assert np.array_equal(u.cpu().numpy(), uo.astype(np.float32))
    assert abs(e - eo) <= REFINE_E_RTOL * max(abs(eo), 1.0)
    _, (g1, g2, fe), (o1, o2, foe) = _flow_refine_case(orc, W, H, 16, -8, -8, dict(C=4.0, warps=2, iters=6))
    assert np.array_equal(g1.cpu().numpy(), o1.astype(np.float32))
    assert np.array_equal(g2.cpu().numpy(), o2.astype(np.float32))
    assert abs(fe - foe) <= REFINE_E_RTOL * max(abs(foe), 1.0)


def test_refine_zero_iterations(orc):
    """iters = 0 (warps of the model only) returns the discrete labelling; warps
    = 0 likewise; the energy is the oracle's energy of the start point."""
    from oracle import refine as orf
    left, right, _ = datagen.pair("wt-kitti", 40, 20, 16, seed=5)
    ctx = _ctx(width=40, height=20, d_min=0, d_max=15, max_iters=2)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(2)
    lab = ctx.labels().cpu().numpy()
    for warps, iters in ((3, 0), (0, 5)):
        u, e = ctx.refine(warps=warps, iters=iters)
        assert np.array_equal(u.cpu().numpy(), lab.astype(np.float32))
        eo = orf.energy(ctx.cost_volume_tensor().cpu().numpy(), lab.astype(np.float64), 3.0, 3.0, 1.0, 1.0, 4.0)
        assert abs(e - eo) <= REFINE_E_RTOL * abs(eo)


def test_flow_refine_c4_full_size(orc):
    """configs[3] (C4): 1242x375, 32x32 window, 4 Dual MM iterations per layer,
    then the continuous refinement (5 warps x 40 iterations)."""
    c = datagen.CONFIGS["C4"]
    _, (g1, g2, e), (o1, o2, eo) = _flow_refine_case(orc, c["W"], c["H"], c["K"], -16, -16, dict(C=4.0))
    assert np.array_equal(g1.cpu().numpy(), o1.astype(np.float32))
    assert np.array_equal(g2.cpu().numpy(), o2.astype(np.float32))
    assert abs(e - eo) <= REFINE_E_RTOL * abs(eo)


def test_flow_refine_state_errors():
    import paper_1601_06274_b200 as dmm
    i1 = np.random.default_rng(0).integers(0, 255, (20, 30)).astype(np.uint8)
    ctx = _ctx(width=30, height=20, d_min=-8, d_max=7, batch=2)
    ctx.flow_cost_volume(torch.from_numpy(i1).cuda(), torch.from_numpy(i1).cuda(), -8)
    with pytest.raises(dmm.DmmError):
        ctx.flow_refine(-8)                              # layers not solved
    ctx.solve(1, frame=0, nframes=2)
    with pytest.raises(dmm.DmmError):
        ctx.flow_refine(-8, tau=0.0)
    ctx.flow_refine(-8, warps=1, iters=1)


# --------------------------------------- NEXT-3 general penalty + edge weights
def _gen_case(orc, kind, W, H, K, pen, ew, iters, w_h=2, w_v=3, d_min=0):
    left, right, _ = datagen.pair(kind, W, H, K, seed=W * H + K)
    ctx = _ctx(width=W, height=H, d_min=d_min, d_max=d_min + K - 1, w_h=w_h, w_v=w_v, max_iters=iters,
               pen=pen, edge_weights=ew)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(iters)
    e, b, hist = ctx.result()
    g = dict(fdual=ctx.dual(0).cpu().numpy(), gdual=ctx.dual(1).cpu().numpy(),
             labels=ctx.labels().cpu().numpy().astype(np.int32), bound_hist=np.array(hist, np.int64), energy=e)
    D = orc.cost_volume(orc.census(left), orc.census(right), d_min, K, 12)
    oh, ov = orc.edge_weights(left) if ew else (None, None)
    o = orc.dmm_general(D, w_h, w_v, pen, 4, iters, oh, ov, nthreads=8)
    return ctx, g, o, D


@pytest.mark.parametrize("kind,W,H,K,pen,ew", [
    ("rd", 70, 30, 16, (8, 16, 2, 80), False),            # eps = 1/2, delta = 2, C = 5
    ("rd", 45, 33, 32, (4, 16, 1, 48), True),              # edge-aware weights
    ("wt-kitti", 120, 36, 64, (0, 16, 3, 64), True),       # eps = 0: flat up to delta (P1-P2-like)
    ("wt-kitti", 90, 21, 128, (12, 16, 1, 96), False),
    ("rd", 33, 17, 40, (16, 16, 0, 64), False),            # classic shape, padded K
    ("rd", 13, 9, 16, (8, 16, 2, 80), True),               # chains <= 16 nodes: the leaf kernel from the root
    ("wt-kitti", 150, 24, 256, (8, 16, 2, 80), False),     # 8 labels per lane
    ("rd", 1, 40, 16, (4, 16, 1, 48), True),               # single-node rows
])
def test_general_parity(orc, kind, W, H, K, pen, ew):
    """hmg.cu (general three-piece penalty, per-edge weights, literal Alg.5)
    == oracle_dmm_general: duals, labels, bound history, energy, bit-exact."""
    ctx, g, o, D = _gen_case(orc, kind, W, H, K, pen, ew, 3)
    assert np.array_equal(g["fdual"].astype(np.int64), o["fdual"]), "f_"
    assert np.array_equal(g["gdual"].astype(np.int64), o["gdual"]), "g_"
    assert np.array_equal(g["labels"], o["labels"])
    assert np.array_equal(g["bound_hist"], o["bound_hist"])
    assert g["energy"] == o["energy"]
    lab = torch.from_numpy(o["labels"].astype(np.uint8)).cuda()
    oh, ov = orc.edge_weights(datagen.pair(kind, W, H, K, seed=W * H + K)[0]) if ew else (None, None)
    assert ctx.energy(labels=lab) == orc.energy_general(D, o["labels"], 2, 3, pen, 4, oh, ov)


def test_general_classic_shape_matches_pair_kernels():
    """General mode with the truncated-linear shape (e1 = e2 = 2^F, c = T 2^F,
    constant weights) solves the same problem as the packed pair kernels."""
    W, H, K = 96, 40, 32
    left, right, _ = datagen.pair("wt-kitti", W, H, K, seed=1)
    lt, rt = torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda()
    a = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w=3, T=4, max_iters=3)
    b = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w=3, T=4, max_iters=3, pen=(16, 16, 0, 64))
    for c in (a, b):
        c.cost_volume(lt, rt)
        c.solve(3)
    assert a.kernel_family() == "pair"
    assert a.result() == b.result()
    assert torch.equal(a.labels(), b.labels()) and torch.equal(a.dual(0), b.dual(0)) and torch.equal(a.dual(1), b.dual(1))


def test_general_c2_size_properties():
    """C2 shape (1242x375x128) with eps = 1/2 penalty and edge-aware weights:
    the oracle is too slow here, so the properties that hold at any size --
    monotone bound history, weak duality bound <= E(labels) (Prop.2),
    energy of the labels by an independent entry point."""
    W, H, K = 1242, 375, 128
    left, right, _ = datagen.pair("wt-kitti", W, H, K, seed=0)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w_h=3, w_v=3, max_iters=4, pen=(8, 16, 2, 80),
               edge_weights=True)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(4)
    e, b, hist = ctx.result()
    assert all(x <= y for x, y in zip(hist, hist[1:]))
    assert b <= e
    assert ctx.energy(labels=ctx.labels()) == e


# ------------------------------------------- NEXT-4 iterative minorant (Alg.4)
@pytest.mark.parametrize("kind,W,H,K,pen,ew,passes,gshift", [
    ("rd", 64, 48, 16, None, False, 3, 2),                # configs[0] shape, the paper's max_pass = 3, gamma = 1/4
    ("wt-kitti", 90, 31, 32, (8, 16, 2, 80), True, 3, 2),
    ("rd", 37, 29, 40, None, False, 4, 1),
    ("wt-kitti", 50, 20, 128, None, False, 1, 2),         # max_pass 1: one full (gamma = 1) pass
])
def test_iterative_minorant_parity(orc, kind, W, H, K, pen, ew, passes, gshift):
    """Dual MM with the iterative minorant on the GPU (one warp per chain)
    == oracle_dmm_minorant(minorant = 1): duals, labels, bounds, energy."""
    iters = 3
    left, right, _ = datagen.pair(kind, W, H, K, seed=K + W)
    ctx = _ctx(width=W, height=H, d_min=0, d_max=K - 1, w_h=2, w_v=3, T=4, max_iters=iters, pen=pen,
               edge_weights=ew, minorant="iterative", iter_passes=passes, iter_gshift=gshift)
    ctx.cost_volume(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    ctx.solve(iters)
    e, b, hist = ctx.result()
    D = orc.cost_volume(orc.census(left), orc.census(right), 0, K, 12)
    oh, ov = orc.edge_weights(left) if ew else (None, None)
    o = orc.dmm_minorant(D, 2, 3, pen or (16, 16, 0, 64), 4, iters, 1, passes, gshift, oh, ov, nthreads=8)
    assert np.array_equal(ctx.dual(0).cpu().numpy().astype(np.int64), o["fdual"])
    assert np.array_equal(ctx.dual(1).cpu().numpy().astype(np.int64), o["gdual"])
    assert np.array_equal(ctx.labels().cpu().numpy().astype(np.int32), o["labels"])
    assert hist == [int(v) for v in o["bound_hist"]] and e == o["energy"]
