"""Pins for the oracle's Dual MM (Algorithm 2) on grids.

Independent checks: exhaustive grid enumeration, a plain Viterbi that never
calls the minorant code, Prop.1 / Prop.2 / weak-duality invariants, and the
special cases where the algorithm reduces to something with a closed form."""
import numpy as np
import pytest

from bruteforce import grid_energies, grid_modular, grid_part_energies


def _rand_D(rng, H, W, K, hi=25):
    return rng.integers(0, hi, size=(H, W, K)).astype(np.uint8)


def test_bound_monotone_and_weak_duality_bruteforce(orc):
    """b_t non-decreasing (P:255 'dual objective does not decrease'); every
    b_t <= min_x E(x) (weak duality) <= E(output labelling)."""
    rng = np.random.default_rng(10)
    cases = [(2, 2, 3), (3, 3, 2), (2, 3, 3), (3, 2, 4), (1, 5, 3), (4, 1, 3), (3, 3, 3)]
    for (H, W, K) in cases:
        for _ in range(6):
            D = _rand_D(rng, H, W, K)
            w = int(rng.integers(0, 6)); T = int(rng.integers(1, K + 1)); Fb = int(rng.integers(0, 5))
            out = orc.dmm(D, w, w, T, Fb, 4)
            b = out["bound_hist"]
            assert np.all(np.diff(b) >= 0), b
            _, e = grid_energies(D, w, w, T, 1 << Fb)
            assert b[-1] <= e.min()
            assert e.min() <= out["energy"]
            assert out["energy"] == orc.energy(D, out["labels"], w, w, T) << Fb


def test_minorant_properties_bruteforce(orc):
    """After each half-step: f_ is a modular minorant of f (f_(x) <= f(x) for
    all x) and g_ of g (Alg.2 lines 2 and 4; Prop.1), and the bound is
    min_x (f_ + g)(x) / min_x (f + g_)(x) consistent with Prop.2."""
    rng = np.random.default_rng(11)
    for (H, W, K) in [(2, 3, 3), (3, 3, 2), (2, 2, 4)]:
        for _ in range(5):
            D = _rand_D(rng, H, W, K)
            w = int(rng.integers(1, 6)); T = int(rng.integers(1, K + 1)); Fb = 4
            X, _ = grid_energies(D, w, w, T, 1 << Fb)
            fx, gx = grid_part_energies(X, D, w, w, T, 1 << Fb)
            for it in (1, 2, 3):
                out = orc.dmm(D, w, w, T, Fb, it)
                fu, gu = out["fdual"], out["gdual"]
                assert np.all(grid_modular(fu, X) <= fx)
                assert np.all(grid_modular(gu, X) <= gx)
                # b_{2t+1} = D(-f_) = min_x (f_ + g)(x)  (Prop.2)
                assert out["bound_hist"][2 * it - 1] == (grid_modular(fu, X) + gx).min()


def test_bounds_equal_viterbi_chain_optima(orc):
    """b_{2t} = sum_rows min(D_s + g_^{t} + row pairwise) and
    b_{2t+1} = sum_cols min(f_^{t+1} + col pairwise): HM's modular minimum equals
    the chain optimum (exactness), checked with a plain Viterbi."""
    rng = np.random.default_rng(12)
    for (H, W, K) in [(5, 9, 4), (7, 6, 5), (4, 13, 3)]:
        D = _rand_D(rng, H, W, K)
        w, T, Fb = 3, 2, 4
        s = 1 << Fb
        g = np.zeros((H, W, K), np.int64)
        for t in range(3):
            out = orc.dmm(D, w, w, T, Fb, t + 1)
            bh = sum(orc.chain_min(D[y].astype(np.int64) * s + g[y], w * s, T)[0] for y in range(H))
            assert out["bound_hist"][2 * t] == bh
            f = out["fdual"]
            bv = sum(orc.chain_min(f[:, x], w * s, T)[0] for x in range(W))
            assert out["bound_hist"][2 * t + 1] == bv
            g = out["gdual"]


def test_single_row_is_exact(orc):
    """H = 1: the grid is one chain, so b_0 = the optimum (SURVEY 8c pins)."""
    rng = np.random.default_rng(13)
    for _ in range(20):
        W = int(rng.integers(1, 8)); K = int(rng.integers(1, 4))
        D = _rand_D(rng, 1, W, K)
        w = int(rng.integers(0, 6)); T = int(rng.integers(1, K + 1))
        out = orc.dmm(D, w, w, T, 4, 1)
        _, e = grid_energies(D, w, w, T, 16)
        assert out["bound_hist"][0] == e.min()


def test_single_column_exact_after_v(orc):
    """W = 1: every row chain is a single node; the V half-step sees the whole
    column chain with unaries f_ = D_s, so b_1 = the optimum."""
    rng = np.random.default_rng(14)
    for _ in range(20):
        H = int(rng.integers(1, 8)); K = int(rng.integers(1, 4))
        D = _rand_D(rng, H, 1, K)
        w = int(rng.integers(0, 6)); T = int(rng.integers(1, K + 1))
        out = orc.dmm(D, w, w, T, 4, 1)
        _, e = grid_energies(D, w, w, T, 16)
        assert out["bound_hist"][1] == e.min()


def test_zero_pairwise_is_wta(orc):
    """w = 0: b_0 = sum_i min_k D_s and labels = lowest-index winner-take-all."""
    rng = np.random.default_rng(15)
    D = _rand_D(rng, 6, 7, 5)
    out = orc.dmm(D, 0, 0, 3, 4, 2)
    assert out["bound_hist"][0] == D.min(2).astype(np.int64).sum() * 16
    assert np.array_equal(out["labels"], D.argmin(2))


def test_stuck_example_fig8(orc):
    """Fig.8 structure (figure missing): 2x2 grid, 2 labels, strong
    Ising (Potts w=10), v1 prefers one label, v4 the other.  The optimum is 1;
    the hierarchical minorant propagates slack so the bound reaches it at b_1
    (the naive single-node minorant of the example would stay at 0)."""
    D = np.zeros((2, 2, 2), np.uint8)
    D[0, 0] = (1, 0)
    D[1, 1] = (0, 1)
    out = orc.dmm(D, 10, 10, 1, 4, 3)
    _, e = grid_energies(D, 10, 10, 1, 16)
    assert e.min() == 16
    assert out["bound_hist"][0] == 0
    assert out["bound_hist"][1] == 16
    assert np.all(out["bound_hist"][1:] == 16)


def test_deterministic_and_thread_invariant(orc):
    rng = np.random.default_rng(16)
    D = _rand_D(rng, 9, 11, 6)
    a = orc.dmm(D, 2, 3, 3, 4, 3, nthreads=1)
    b = orc.dmm(D, 2, 3, 3, 4, 3, nthreads=4)
    for k in ("fdual", "gdual", "labels", "bound_hist"):
        assert np.array_equal(a[k], b[k])
    assert a["energy"] == b["energy"]


def test_bad_arguments(orc):
    D = np.zeros((2, 2, 2), np.uint8)
    with pytest.raises(ValueError):
        orc.dmm(D, 1, 1, 1, 4, 0)      # iterations = 0 -> argument error
    with pytest.raises(ValueError):
        orc.dmm(D, 1, 1, 0, 4, 1)      # T < 1
