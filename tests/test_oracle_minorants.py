"""Pins for the NEXT-4 minorant variants and the TRW-S comparator.

* Uniform minorant (Alg.3, oracle/minorants.py): the paper-printed tables of
  the appendix example (tests/golden/appendix_uniform.json)
  and Lemma 2 (lambda >= m / n).
* Iterative minorant (Alg.4, C oracle; the GPU runs the same): valid, exact and
  maximal by brute force, for truncated-linear and general penalties with
  edge weights.
* Naive minorant (m / n): valid and exact (not maximal).
* TRW-S: a lower bound (<= brute-force optimum), non-decreasing.
* Convergence surrogate of Fig.3 / Fig.10 on a
  synthetic 40 x 40 x 16 crop: the naive minorant is far behind, the
  hierarchical and iterative minorants and TRW-S end within 0.1 %, and the
  hierarchical DMM leads TRW-S per iteration ("DMM can perform even better than
  the sequential baseline in terms of iterations")."""
import json
import os
from fractions import Fraction

import numpy as np

from bruteforce import all_labellings
from oracle import minorants as mn

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _appendix_F():
    with open(os.path.join(GOLD, "appendix_chain.json")) as f:
        return np.array(json.load(f)["unary_labels_by_nodes"]).T.tolist()      # nodes x labels


def _table(lam):
    return [[lam[i][k] for i in range(len(lam))] for k in range(len(lam[0]))]   # labels x nodes


def test_uniform_minorant_paper_tables():
    with open(os.path.join(GOLD, "appendix_uniform.json")) as f:
        g = json.load(f)
    F = _appendix_F()
    hist = []
    lam = mn.uniform_minorant(F, mn.potts(1), hist)
    first = [[v - min(row) for v in row] for row in hist[0][1]]
    assert _table(first) == g["potts1_first_minorant"]["table"]
    assert _table(lam) == g["potts1_final_minorant"]["table"]
    assert [e for e, _ in hist[:2]] == g["potts1_first_two_eps"]["eps"]
    lam5 = mn.uniform_minorant(F, mn.potts(5))
    assert _table(lam5) == [[Fraction(v) for v in row] for row in g["potts5_final_minorant"]["table"]]


def test_uniform_minorant_lemma2():
    """lambda >= m / n (normalised min-marginals over the chain length)."""
    rng = np.random.default_rng(0)
    for _ in range(25):
        n, K = int(rng.integers(2, 6)), int(rng.integers(2, 4))
        F = rng.integers(0, 10, size=(n, K)).tolist()
        V = mn.trunc_lin(int(rng.integers(1, 4)), int(rng.integers(1, 3)))
        lam = mn.uniform_minorant(F, V)
        m = mn.min_marginals(F, V)
        for i in range(n):
            for k in range(K):
                assert lam[i][k] >= (m[i][k] - min(m[i])) / n


def _chain_energies(F, w, pen, om):
    n, K = F.shape
    X = all_labellings(n, K)
    e = F[np.arange(n)[None, :], X].sum(1)
    e1, e2, d, c = pen
    for p in range(n - 1):
        dd = np.abs(X[:, p] - X[:, p + 1])
        e = e + (w * int(om[p]) * np.minimum(e1 * np.minimum(dd, d) + e2 * np.maximum(dd - d, 0), c)) // 16
    return X, e


def test_iterative_minorant_bruteforce(orc):
    rng = np.random.default_rng(1)
    for _ in range(250):
        n, K = int(rng.integers(1, 6)), int(rng.integers(1, 5))
        e1 = int(rng.integers(0, 17))
        pen = (e1, 16, int(rng.integers(0, 3)), int(rng.integers(0, 90)))
        w = int(rng.integers(0, 4))
        om = rng.integers(1, 17, size=max(n - 1, 1))
        F = rng.integers(-50, 50, size=(n, K))
        lam = orc.iter_minorant(F, w, pen, om.astype(np.uint8), int(rng.integers(1, 5)), int(rng.integers(0, 4)))
        X, e = _chain_energies(F, w, pen, om)
        lv = lam[np.arange(n)[None, :], X].sum(1)
        assert np.all(lv <= e)                       # minorant
        assert lam.min(1).sum() == e.min()           # exact
        slack = e - lv
        for i in range(n):                           # maximal (last pass gamma = 1)
            for k in range(K):
                assert slack[X[:, i] == k].min() == 0


def test_naive_minorant_valid_and_exact(orc):
    """C oracle (fixed point, floor): a valid minorant with sum of node minima
    <= F*; in exact arithmetic (oracle/minorants.py) m / n is exact: n F* / n."""
    rng = np.random.default_rng(2)
    for _ in range(150):
        n, K = int(rng.integers(1, 6)), int(rng.integers(1, 5))
        pen = (16, 16, 0, int(rng.integers(16, 90)))
        F = rng.integers(0, 50, size=(n, K))
        om = np.full(max(n - 1, 1), 16)
        lam = orc.naive_minorant(F, 2, pen, om.astype(np.uint8))
        X, e = _chain_energies(F, 2, pen, om)
        lv = lam[np.arange(n)[None, :], X].sum(1)
        assert np.all(lv <= e)
        assert lam.min(1).sum() <= e.min()
        lf = mn.naive_minorant(F.tolist(), lambda a, b: Fraction(2 * min(abs(a - b) * 16, pen[3])))
        assert sum(min(row) for row in lf) == e.min()


def test_trws_lower_bound_bruteforce():
    rng = np.random.default_rng(3)
    for _ in range(15):
        H, W, K = int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(2, 4))
        D = rng.integers(0, 10, size=(H, W, K))
        X = all_labellings(H * W, K).reshape(-1, H, W)
        e = D[np.arange(H)[None, :, None], np.arange(W)[None, None, :], X].sum((1, 2)).astype(float)
        e = e + 2 * np.minimum(np.abs(X[:, :, :-1] - X[:, :, 1:]), 2).sum((1, 2))
        e = e + 3 * np.minimum(np.abs(X[:, :-1, :] - X[:, 1:, :]), 2).sum((1, 2))
        b = mn.trws(D, 2, 3, 2, 6)
        assert max(b) <= e.min() + 1e-9
        assert all(b[i] <= b[i + 1] + 1e-9 for i in range(len(b) - 1))


def test_convergence_surrogate_fig3(orc):
    import datagen
    left, right, _ = datagen.pair("wt-kitti", 40, 40, 16, seed=3)
    D = orc.cost_volume(orc.census(left), orc.census(right), 0, 16, 12)
    pen, it = (16, 16, 0, 64), 8
    b = {name: orc.dmm_minorant(D, 3, 3, pen, 4, it, mi, 3, 2)["bound_hist"][1::2] / 16.0
         for name, mi in (("hierarchical", 0), ("iterative", 1), ("naive", 2))}
    b["trws"] = np.array(mn.trws(D, 3, 3, 4, it))
    for k in ("hierarchical", "iterative", "trws"):
        assert np.all(b["naive"] < b[k] - 50)                       # naive far behind at every iteration
    final = [b[k][-1] for k in ("hierarchical", "iterative", "trws")]
    assert (max(final) - min(final)) / max(final) < 1e-3
    assert np.all(b["hierarchical"][:3] > b["trws"][:3])            # DMM leads TRW-S per iteration
