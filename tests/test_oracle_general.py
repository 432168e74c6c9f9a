"""Pins for the NEXT-3 oracle: general penalty (Fig.2, Eq.
r-decompose P:364-375, sampled at integer label differences) and quantised
edge weights (SPEC S:99 formula, reading R30).

Independent pins: the classic parameters reproduce the pinned truncated-linear
oracle bit for bit; the integer penalty equals 2^F times the continuous
three-piece r of oracle/refine.py (a different implementation) at integer
arguments; the hierarchical minorant stays a valid, exact and maximal
minorant for non-metric penalties and per-edge weights (brute force over all
labellings); Dual MM keeps monotone bounds and weak duality on tiny grids; the
weight table has its closed-form values."""
import itertools
import math

import numpy as np
import pytest

from bruteforce import all_labellings

F_BITS = 4


def _V(pen, w, om, d):
    e1, e2, delta, c = pen
    d = np.abs(d)
    R = np.minimum(e1 * np.minimum(d, delta) + e2 * np.maximum(d - delta, 0), c)
    return (w * om * R) // 16


def test_classic_parameters_reproduce_truncated_linear(orc):
    rng = np.random.default_rng(0)
    for H, W, K, w, T in ((7, 9, 5, 3, 2), (12, 5, 16, 3, 4), (1, 11, 8, 2, 30)):
        D = rng.integers(0, 25, size=(H, W, K)).astype(np.uint8)
        a = orc.dmm(D, w, w, T, F_BITS, 3)
        b = orc.dmm_general(D, w, w, (1 << F_BITS, 1 << F_BITS, 0, T << F_BITS), F_BITS, 3)
        for k in ("fdual", "gdual", "labels", "bound_hist"):
            assert np.array_equal(a[k], b[k]), k
        assert a["energy"] == b["energy"]


def test_integer_penalty_is_sampled_continuous_r():
    """R(d) = 2^F r_{eps,delta} - r_{0,C+delta-eps delta} at integer d with
    eps = e1 / 2^F, e2 = 2^F, C = c / 2^F (oracle/refine.py's float r)."""
    from oracle import refine as rf
    for e1, delta, c in ((8, 2, 80), (4, 1, 48), (16, 3, 64), (0, 2, 40)):
        d = np.arange(-40, 41)
        R = np.minimum(e1 * np.minimum(np.abs(d), delta) + 16 * np.maximum(np.abs(d) - delta, 0), c)
        ref = 16 * rf.r_dc(d, e1 / 16, float(delta), c / 16)
        assert np.allclose(R, ref, atol=1e-9)


def _chain_energies(F, w, pen, om):
    n, K = F.shape
    X = all_labellings(n, K)
    e = F[np.arange(n)[None, :], X].sum(1)
    for p in range(n - 1):
        e = e + _V(pen, w, int(om[p]), X[:, p] - X[:, p + 1])
    return X, e


def test_hm_general_minorant_bruteforce(orc):
    """Valid (lam(x) <= F(x) for all x), exact (sum of node minima = optimum)
    and maximal (all min-marginals of F - lam are 0; Lemma 1) for
    non-metric penalties (eps < 1) with random per-edge weights."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.integers(1, 6)); K = int(rng.integers(1, 5))
        pen = (int(rng.integers(0, 9)), 0, int(rng.integers(0, 3)), int(rng.integers(0, 80)))
        pen = (pen[0], pen[0] + int(rng.integers(0, 20)), pen[2], pen[3])
        w = int(rng.integers(0, 4))
        om = rng.integers(1, 17, size=max(n - 1, 1))
        F = rng.integers(-60, 60, size=(n, K))
        lam = orc.hm_general(F, w, pen, om.astype(np.uint8))
        X, e = _chain_energies(F, w, pen, om)
        lv = lam[np.arange(n)[None, :], X].sum(1)
        assert np.all(lv <= e)
        assert lam.min(1).sum() == e.min()
        slack = e - lv
        for i in range(n):
            for k in range(K):
                assert slack[X[:, i] == k].min() == 0


def test_dmm_general_bounds_bruteforce(orc):
    """Monotone bound history, weak duality vs the brute-force optimum, bound <= E(labels)."""
    rng = np.random.default_rng(2)
    for _ in range(40):
        H, W, K = int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(2, 4))
        D = rng.integers(0, 12, size=(H, W, K)).astype(np.uint8)
        pen = (int(rng.integers(0, 16)), 16, int(rng.integers(0, 3)), int(rng.integers(16, 90)))
        img = rng.integers(0, 256, size=(H, W)).astype(np.uint8)
        oh, ov = orc.edge_weights(img)
        out = orc.dmm_general(D, 2, 3, pen, F_BITS, 4, oh, ov)
        X = all_labellings(H * W, K).reshape(-1, H, W)
        e = (D.astype(np.int64)[np.arange(H)[None, :, None], np.arange(W)[None, None, :], X] << F_BITS).sum((1, 2))
        for y in range(H):
            for x in range(W):
                if x + 1 < W:
                    e = e + _V(pen, 2, int(oh[y, x]), X[:, y, x] - X[:, y, x + 1])
                if y + 1 < H:
                    e = e + _V(pen, 3, int(ov[y, x]), X[:, y, x] - X[:, y + 1, x])
        bh = out["bound_hist"]
        assert np.all(np.diff(bh) >= 0)
        assert bh[-1] <= e.min()
        assert bh[-1] <= out["energy"]
        assert out["energy"] == orc.energy_general(D, out["labels"], 2, 3, pen, F_BITS, oh, ov)
        assert out["energy"] in set(e.tolist())


def test_edge_weight_table(orc):
    img = np.array([[0, 0, 51, 255, 255]], np.uint8)
    oh, ov = orc.edge_weights(img)
    assert list(oh[0]) == [16, round(16 * math.exp(-1)), max(1, round(16 * math.exp(-5 * 204 / 255))), 16, 16]
    assert np.all(ov == 16)          # one row: no vertical edges (unused entries = 16)
    col = np.arange(0, 256, 5, dtype=np.uint8)[:, None]
    oh, ov = orc.edge_weights(col)
    assert np.all(np.diff(ov[:-1, 0].astype(int)) == 0)           # constant step 5 -> constant weight
    ramp = np.array([[0, 1, 3, 6, 10, 15, 21, 28, 36, 45, 55, 66, 78, 91, 105, 120, 136]], np.uint8)
    oh, _ = orc.edge_weights(ramp)
    assert np.all(np.diff(oh[0, :-1].astype(int)) <= 0)           # growing steps -> non-increasing weights
    assert oh.min() >= 1 and oh.max() <= 16
