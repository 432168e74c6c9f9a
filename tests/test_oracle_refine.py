"""Pins for the continuous-refinement oracle (oracle/refine.py; NEXT-2).

Each pin is independent of the oracle's own formulas: proximal maps and the
convex conjugate against brute-force minimisation / maximisation on fine grids
(SURVEY 8(f) "prox grid-search"), the DC decomposition against a different
closed form of the three-piece penalty, the adjoint test for A, the energy at
integer labellings against the C oracle's discrete energy, and the
zero-regularisation case against a grid search of the data approximation."""
import numpy as np
import pytest

from oracle import refine as rf


def test_dc_decomposition_is_the_three_piece_penalty():
    """r = r_{eps,delta} - r_{0,C+delta-eps*delta} equals
    min(max(eps|t|, |t| - delta(1-eps)), C): slope eps up to delta, slope 1,
    truncated at C (Fig.2); eps = 1 gives the truncated-linear min(|t|, C)."""
    t = np.linspace(-20, 20, 4001)
    for eps, delta, C in ((0.5, 2.0, 4.0), (0.2, 1.0, 3.0), (1.0, 1.0, 4.0), (0.0, 3.0, 6.0)):
        ref = np.minimum(np.maximum(eps * np.abs(t), np.abs(t) - delta * (1 - eps)), C)
        assert np.allclose(rf.r_dc(t, eps, delta, C), ref, atol=1e-12)
    assert np.allclose(rf.r_dc(t, 1.0, 1.0, 4.0), np.minimum(np.abs(t), 4.0))


def test_conjugate_by_numeric_sup():
    """(w r_{a,b})^*(s) = sup_t s t - w r_{a,b}(t), by a dense grid over t."""
    t = np.linspace(-60, 60, 240001)
    for w, a, b in ((3.0, 0.5, 2.0), (1.5, 0.0, 5.0), (2.0, 1.0, 1.0)):
        for s in np.linspace(-w, w, 41):
            num = np.max(s * t - w * rf.r_ab(t, a, b))
            assert abs(num - rf.conj_w_rab(s, w, a, b)) < 1e-3


@pytest.mark.parametrize("w,a,b,step", [(3.0, 0.5, 2.0, 0.35), (1.5, 0.0, 5.0, 0.35), (2.0, 1.0, 1.0, 0.7),
                                        (4.0, 0.25, 3.0, 0.1)])
def test_prox_conj_by_grid_search(w, a, b, step):
    """prox_{step h}(t) = argmin_s step h(s) + (s - t)^2 / 2 with h = (w r_{a,b})^*
    (finite on [-w, w]), against a grid of s and the grid-evaluated conjugate."""
    s = np.linspace(-w, w, 40001)
    hs = b * np.maximum(0.0, np.abs(s) - a * w)
    for t in np.linspace(-3 * w, 3 * w, 61):
        ref = s[np.argmin(step * hs + 0.5 * (s - t) ** 2)]
        assert abs(rf.prox_conj(t, w, a, b, step) - ref) < 1e-3


def test_prox_data_by_grid_search():
    """Prox of tau * D~ (two slopes + indicator of [u0 - h, u0 + h])."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        u0 = rng.uniform(0, 50)
        s1 = rng.uniform(-10, 10)
        s2 = s1 + rng.uniform(0, 10)
        tau, h = rng.uniform(0.05, 1.0), rng.uniform(0.5, 2.0)
        uh = u0 + rng.uniform(-8, 8)
        grid = np.linspace(u0 - h, u0 + h, 20001)
        Dt = np.where(grid <= u0, s1 * (grid - u0), s2 * (grid - u0))
        ref = grid[np.argmin(tau * Dt + 0.5 * (grid - uh) ** 2)]
        got = rf.prox_data(np.array([uh]), np.array([u0]), np.array([s1]), np.array([s2]), tau, h)[0]
        assert abs(got - ref) < 2e-4


def test_adjoint():
    rng = np.random.default_rng(1)
    for H, W in ((1, 5), (4, 1), (7, 9)):
        u = rng.normal(size=(H, W))
        ph, pv = rng.normal(size=(H, W - 1)), rng.normal(size=(H - 1, W))
        ah, av = rf.A(u)
        assert abs((ah * ph).sum() + (av * pv).sum() - (u * rf.AT(ph, pv, (H, W))).sum()) < 1e-9


def test_energy_at_integer_labels_is_the_discrete_energy(orc):
    """eps = 1, C = T, w = w_h / w_v: E(u) at an integer labelling equals the
    discrete energy of Eq.3 computed by the C oracle."""
    rng = np.random.default_rng(2)
    D = rng.integers(0, 25, size=(9, 13, 11)).astype(np.uint8)
    lab = rng.integers(0, 11, size=(9, 13)).astype(np.int32)
    e = rf.energy(D, lab.astype(np.float64), 3.0, 2.0, 1.0, 1.0, 4.0)
    assert abs(e - orc.energy(D, lab, 3, 2, 4)) < 1e-9


def test_zero_regularisation_is_per_pixel_minimisation():
    """w = 0: the duals stay 0 and every pixel minimises its own convex data
    approximation on [u0 - h, u0 + h] (one warp): compare with a grid search."""
    rng = np.random.default_rng(3)
    D = rng.integers(0, 25, size=(6, 7, 9)).astype(np.uint8)
    lab = rng.integers(1, 8, size=(6, 7))
    u, _ = rf.refine(D, lab, 0.0, 0.0, warps=1, iters=400)
    s1, s2 = rf.slopes(D, lab.astype(np.float64), 1.0)
    for y in range(6):
        for x in range(7):
            u0 = float(lab[y, x])
            grid = np.linspace(u0 - 1, u0 + 1, 4001)
            Dt = np.where(grid <= u0, s1[y, x] * (grid - u0), s2[y, x] * (grid - u0))
            best = Dt.min()
            got = s1[y, x] * (u[y, x] - u0) if u[y, x] <= u0 else s2[y, x] * (u[y, x] - u0)
            assert got <= best + 1e-6


def test_refinement_runs_and_interpolates():
    """Interpolated D at integer u equals the sampled cost; a refinement of a
    smooth slanted-plane problem moves the staircase towards the plane."""
    H, W, K = 12, 40, 16
    xs = np.arange(W)
    true = 3.0 + 0.2 * xs                            # slanted plane, sub-pixel
    k = np.arange(K)
    D = np.broadcast_to(np.abs(k[None, :] - true[:, None]) * 4.0, (H, W, K)).round().astype(np.uint8)
    lab = np.broadcast_to(np.rint(true), (H, W)).astype(np.int64)
    assert np.array_equal(rf.D_interp(D, lab.astype(np.float64)), D[np.arange(H)[:, None], np.arange(W), lab])
    u, e = rf.refine(D, lab, 0.5, 0.5, eps=1.0, delta=1.0, C=4.0)
    assert np.abs(u - true[None, :]).mean() < np.abs(lab - true[None, :]).mean()


# ------------------------------------------------------- flow (Sec. 3.2)
def test_flow_cost_bilinear_at_integers_is_the_census_cost(orc):
    """D at integer displacements is the census Hamming cost of the discrete
    stage: the minimum over the vertical window equals oracle_flow_costs' f1."""
    import datagen
    i1, i2, _, _ = datagen.flow_pair(40, 24, 8, seed=1)
    c1, c2 = orc.census(i1), orc.census(i2)
    f1, f2 = orc.flow_costs(c1, c2, -8, 16, -8, 16)
    H, W = c1.shape
    for a in range(-8, 8):
        best = np.full((H, W), np.inf)
        for b in range(-8, 8):
            d = rf.flow_cost_bilinear(c1, c2, np.full((H, W), float(a)), np.full((H, W), float(b)))
            assert np.array_equal(d, rf.flow_cost_int(c1, c2, np.full((H, W), a), np.full((H, W), b)))
            best = np.minimum(best, d)
        assert np.array_equal(best, f1[:, :, a + 8].astype(np.float64))


def test_prox_quadratic_by_grid_search():
    rng = np.random.default_rng(5)
    for _ in range(300):
        u0, L, Q = rng.uniform(-10, 10), rng.uniform(-20, 20), rng.uniform(0, 30)
        tau, h = rng.uniform(0.05, 1.0), rng.uniform(0.5, 2.0)
        uh = u0 + rng.uniform(-5, 5)
        grid = np.linspace(u0 - h, u0 + h, 20001)
        obj = tau * (L * (grid - u0) + 0.5 * Q * (grid - u0) ** 2) + 0.5 * (grid - uh) ** 2
        got = rf.prox_quadratic(np.array([uh]), np.array([u0]), np.array([L]), np.array([Q]), tau, h)[0]
        assert abs(got - grid[np.argmin(obj)]) < 2e-4


def test_flow_refine_zero_regularisation(orc):
    """w = 0, one warp: each component minimises its own quadratic model on
    [u0 - h, u0 + h] (closed form of Eq. 19 restricted to the box)."""
    import datagen
    i1, i2, g1, g2 = datagen.flow_pair(30, 20, 8, seed=2)
    c1, c2 = orc.census(i1), orc.census(i2)
    u1 = np.clip(g1, -7, 7).astype(np.float64)
    u2 = np.clip(g2, -7, 7).astype(np.float64)
    r1, r2, _ = rf.flow_refine(c1, c2, u1, u2, 0.0, 0.0, warps=1, iters=400)
    L1, Q1, L2, Q2 = rf.flow_quadratic(c1, c2, u1, u2, 1.0)
    for u0, L, Q, r in ((u1, L1, Q1, r1), (u2, L2, Q2, r2)):
        grid = u0[..., None] + np.linspace(-1, 1, 2001)[None, None, :]
        obj = L[..., None] * (grid - u0[..., None]) + 0.5 * Q[..., None] * (grid - u0[..., None]) ** 2
        mn = obj.min(-1)
        got = L * (r - u0) + 0.5 * Q * (r - u0) ** 2
        assert np.all(got <= mn + 1e-6)
