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


def test_psd_part_is_eigenvalue_clipping():
    """psd_part's closed form equals V max(Lambda, 0) V^T by numpy's eigh."""
    rng = np.random.default_rng(6)
    for _ in range(500):
        a, b, c = rng.normal(scale=10, size=3)
        if rng.random() < 0.2:
            b = 0.0
        lam, V = np.linalg.eigh(np.array([[a, b], [b, c]]))
        ref = V @ np.diag(np.maximum(lam, 0.0)) @ V.T
        pa, pb, pc = rf.psd_part(a, b, c)
        assert np.allclose([[pa, pb], [pb, pc]], ref, atol=1e-9 * (1 + np.abs(lam).max()))
    # already PSD: unchanged (bit-exact); negative definite: 0
    assert tuple(map(float, rf.psd_part(4.0, 1.0, 3.0))) == (4.0, 1.0, 3.0)
    assert tuple(map(float, rf.psd_part(-4.0, 1.0, -3.0))) == (0.0, 0.0, 0.0)


def test_flow_quadratic_recovers_a_quadratic_cost():
    """Central differences are exact on a quadratic: D(u) = g^T u + u^T B u / 2
    gives L = g + B u and Q = PSD part of B (a saddle B is clipped)."""
    rng = np.random.default_rng(7)
    u1 = rng.uniform(-5, 5, size=(4, 5))
    u2 = rng.uniform(-5, 5, size=(4, 5))
    for B in (np.array([[3.0, 1.0], [1.0, 2.0]]), np.array([[2.0, 3.0], [3.0, -1.0]]),
              np.array([[-1.0, 0.5], [0.5, -2.0]])):
        g = np.array([0.7, -1.3])
        cost = lambda v1, v2: g[0] * v1 + g[1] * v2 + 0.5 * (B[0, 0] * v1 * v1 + 2 * B[0, 1] * v1 * v2 + B[1, 1] * v2 * v2)  # noqa: E731
        L1, L2, Qa, Qb, Qc = rf.flow_quadratic(None, None, u1, u2, 1.0, cost=cost)
        assert np.allclose(L1, g[0] + B[0, 0] * u1 + B[0, 1] * u2, atol=1e-9)
        assert np.allclose(L2, g[1] + B[1, 0] * u1 + B[1, 1] * u2, atol=1e-9)
        lam, V = np.linalg.eigh(B)
        P = V @ np.diag(np.maximum(lam, 0.0)) @ V.T
        assert np.allclose(Qa, P[0, 0], atol=1e-9) and np.allclose(Qb, P[0, 1], atol=1e-9)
        assert np.allclose(Qc, P[1, 1], atol=1e-9)


def test_prox_quadratic_by_grid_search():
    """Eq. 20's prox: (a) a diagonal Q separates, so the clamped quotient is the
    exact box-constrained prox (1-D grid search per component); (b) a general
    PSD Q with the box inactive is the unconstrained prox (2-D grid search)."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        u0 = rng.uniform(-10, 10, 2)
        L = rng.uniform(-20, 20, 2)
        Qd = rng.uniform(0, 30, 2)
        tau, h = rng.uniform(0.05, 1.0), rng.uniform(0.5, 2.0)
        uh = u0 + rng.uniform(-5, 5, 2)
        got = rf.prox_quadratic(uh[0], uh[1], u0[0], u0[1], L[0], L[1], Qd[0], 0.0, Qd[1], tau, h)
        for k in range(2):
            grid = np.linspace(u0[k] - h, u0[k] + h, 20001)
            obj = tau * (L[k] * (grid - u0[k]) + 0.5 * Qd[k] * (grid - u0[k]) ** 2) + 0.5 * (grid - uh[k]) ** 2
            assert abs(float(got[k]) - grid[np.argmin(obj)]) < 2e-4
    n = 0
    while n < 40:
        u0 = rng.uniform(-3, 3, 2)
        M = rng.normal(size=(2, 2))
        Q = M @ M.T * rng.uniform(0.5, 5)
        L = rng.uniform(-4, 4, 2)
        tau = rng.uniform(0.1, 1.0)
        uh = u0 + rng.uniform(-1, 1, 2)
        got = np.array([float(v) for v in rf.prox_quadratic(uh[0], uh[1], u0[0], u0[1], L[0], L[1],
                                                             Q[0, 0], Q[0, 1], Q[1, 1], tau, 1e6)])
        if np.abs(got - u0).max() > 2.5:
            continue
        n += 1
        g1, g2 = np.meshgrid(np.linspace(u0[0] - 3, u0[0] + 3, 1201), np.linspace(u0[1] - 3, u0[1] + 3, 1201),
                             indexing="ij")
        d1, d2 = g1 - u0[0], g2 - u0[1]
        obj = tau * (L[0] * d1 + L[1] * d2 + 0.5 * (Q[0, 0] * d1 * d1 + 2 * Q[0, 1] * d1 * d2 + Q[1, 1] * d2 * d2)) \
            + 0.5 * ((g1 - uh[0]) ** 2 + (g2 - uh[1]) ** 2)
        i = np.unravel_index(np.argmin(obj), obj.shape)
        assert abs(got[0] - g1[i]) < 1e-2 and abs(got[1] - g2[i]) < 1e-2


def test_flow_refine_zero_regularisation(orc):
    """w = 0: the duals stay 0 and the primal iterates u <- prox(u) of every
    pixel converge to the minimiser of its own quadratic model where that lies
    inside the box and Q is well conditioned: Q u = Q u0 - L (np.linalg.solve)."""
    import datagen
    i1, i2, g1, g2 = datagen.flow_pair(30, 20, 8, seed=2)
    c1, c2 = orc.census(i1), orc.census(i2)
    u1 = np.clip(g1, -7, 7).astype(np.float64)
    u2 = np.clip(g2, -7, 7).astype(np.float64)
    r1, r2, _ = rf.flow_refine(c1, c2, u1, u2, 0.0, 0.0, warps=1, iters=400)
    L1, L2, Qa, Qb, Qc = rf.flow_quadratic(c1, c2, u1, u2, 1.0)
    checked = 0
    for y in range(u1.shape[0]):
        for x in range(u1.shape[1]):
            Q = np.array([[Qa[y, x], Qb[y, x]], [Qb[y, x], Qc[y, x]]])
            if np.linalg.eigvalsh(Q).min() < 0.5:
                continue
            star = np.array([u1[y, x], u2[y, x]]) - np.linalg.solve(Q, [L1[y, x], L2[y, x]])
            if np.abs(star - [u1[y, x], u2[y, x]]).max() >= 1.0:
                continue
            checked += 1
            assert abs(r1[y, x] - star[0]) < 1e-9 and abs(r2[y, x] - star[1]) < 1e-9
    assert checked > 20


def test_flow_cost_bilinear_between_integers(orc):
    """R35: on an edge of the integer grid the cost is the linear interpolation
    of its two endpoints; at a cell centre the mean of the four corners."""
    import datagen
    i1, i2, _, _ = datagen.flow_pair(36, 20, 8, seed=3)
    c1, c2 = orc.census(i1), orc.census(i2)
    H, W = c1.shape
    rng = np.random.default_rng(9)
    a = rng.integers(-6, 6, size=(H, W))
    b = rng.integers(-6, 6, size=(H, W))
    fx = rng.uniform(0, 1, size=(H, W))
    D = lambda da, db: rf.flow_cost_int(c1, c2, a + da, b + db)   # noqa: E731
    got = rf.flow_cost_bilinear(c1, c2, a + fx, b.astype(np.float64))
    assert np.allclose(got, (1 - fx) * D(0, 0) + fx * D(1, 0), atol=1e-12)
    got = rf.flow_cost_bilinear(c1, c2, a.astype(np.float64), b + fx)
    assert np.allclose(got, (1 - fx) * D(0, 0) + fx * D(0, 1), atol=1e-12)
    got = rf.flow_cost_bilinear(c1, c2, a + 0.5, b + 0.5)
    assert np.allclose(got, (D(0, 0) + D(1, 0) + D(0, 1) + D(1, 1)) / 4, atol=1e-12)
