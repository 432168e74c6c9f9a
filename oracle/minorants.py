"""Oracle-only minorant constructions and the TRW-S comparator (NEXT-4 of
SURVEY 8(f)); TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Exact rational arithmetic (fractions.Fraction) in pure Python, for the small
chains / grids of the appendix examples and the convergence surrogate:

* ``min_marginals`` -- Def. P:631-636 by the messages of Eq. P:637-649.
* ``uniform_minorant`` -- the maximal uniform minorant, Algorithm 3
  (P:692-718), with reading R12: O = the labels whose min-marginal of f - lambda
  equals the residual optimum (P:711 prints "[[m = 0]]"); the step
  max{eps | eps <1 - O, x> <= (f - lambda)(x) - F*(f - lambda) for all x} is a
  minimum-ratio path problem (Lawler), solved exactly by Dinkelbach's
  iteration with a Viterbi pass per step.  The returned lambda excludes the
  constant F* of f (the printed tables do) and is node-normalised.
* ``naive_minorant`` -- min-marginals / n (Fig.3).
* ``trws`` -- sequential tree-reweighted message passing (TRW-S, Kolmogorov
  2006, cited P:165 / P:651-667 as the baseline) on a 4-connected grid with
  the row / column chain decomposition (each node in 2 chains, each edge in 1).
"""
from __future__ import annotations

from fractions import Fraction
from typing import Callable, List, Sequence

import numpy as np

Pairwise = Callable[[int, int], Fraction]


def potts(w) -> Pairwise:
    return lambda a, b: Fraction(0) if a == b else Fraction(w)


def trunc_lin(w, T) -> Pairwise:
    return lambda a, b: Fraction(w) * min(abs(a - b), T)


def _msgs(F: List[List[Fraction]], V: Pairwise):
    n, K = len(F), len(F[0])
    left = [[Fraction(0)] * K for _ in range(n)]
    right = [[Fraction(0)] * K for _ in range(n)]
    for i in range(1, n):
        left[i] = [min(left[i - 1][a] + F[i - 1][a] + V(a, b) for a in range(K)) for b in range(K)]
    for i in range(n - 2, -1, -1):
        right[i] = [min(right[i + 1][a] + F[i + 1][a] + V(a, b) for a in range(K)) for b in range(K)]
    return left, right


def min_marginals(F, V: Pairwise):
    """m_i(k) = min over labellings with x_i = k of the chain energy (Def. P:631)."""
    F = [[Fraction(v) for v in row] for row in F]
    left, right = _msgs(F, V)
    return [[left[i][k] + F[i][k] + right[i][k] for k in range(len(F[0]))] for i in range(len(F))]


def _viterbi(F, V: Pairwise):
    """(min value, an optimal labelling) of the chain."""
    n, K = len(F), len(F[0])
    cost = [list(F[0])]
    back = []
    for i in range(1, n):
        row, bk = [], []
        for b in range(K):
            best, arg = None, 0
            for a in range(K):
                v = cost[-1][a] + V(a, b)
                if best is None or v < best:
                    best, arg = v, a
            row.append(best + F[i][b])
            bk.append(arg)
        cost.append(row)
        back.append(bk)
    k = min(range(K), key=lambda b: cost[-1][b])
    val = cost[-1][k]
    x = [k]
    for bk in reversed(back):
        x.append(bk[x[-1]])
    return val, x[::-1]


def uniform_minorant(F, V: Pairwise, history: list | None = None):
    """Algorithm 3, reading R12.  Returns lambda [n][K] (Fractions),
    node-normalised, without the constant F*; `history` (optional) receives
    (eps, lambda-after-step) per iteration."""
    F = [[Fraction(v) for v in row] for row in F]
    n, K = len(F), len(F[0])
    fstar = _viterbi(F, V)[0]
    lam = [[Fraction(0)] * K for _ in range(n)]
    while True:
        R = [[F[i][k] - lam[i][k] for k in range(K)] for i in range(n)]
        m = min_marginals(R, V)
        rstar = min(m[0])
        if all(m[i][k] == rstar for i in range(n) for k in range(K)):
            break
        O = [[m[i][k] == rstar for k in range(K)] for i in range(n)]
        # min ratio of (R(x) - rstar) / <1 - O, x> over labellings with <1-O, x> > 0 (Dinkelbach)
        eps = min(m[i][k] - rstar for i in range(n) for k in range(K) if not O[i][k])
        while True:
            Fe = [[R[i][k] - (0 if O[i][k] else eps) for k in range(K)] for i in range(n)]
            val, x = _viterbi(Fe, V)
            if val - rstar >= 0:
                break
            c = sum(0 if O[i][x[i]] else 1 for i in range(n))
            r = sum(R[i][x[i]] for i in range(n)) + sum(V(x[i], x[i + 1]) for i in range(n - 1))
            eps = (r - rstar) / c
        lam = [[lam[i][k] + (0 if O[i][k] else eps) for k in range(K)] for i in range(n)]
        if history is not None:
            history.append((eps, [row[:] for row in lam]))
    return [[v - min(row) for v in row] for row in lam]


def naive_minorant(F, V: Pairwise):
    """lambda_i = m_i / n."""
    m = min_marginals(F, V)
    n = len(m)
    return [[v / n for v in row] for row in m]


# --------------------------------------------------------------- TRW-S
def trws(D, w_h: float, w_v: float, T: int, iters: int):
    """Sequential TRW-S on the 4-connected grid with truncated-linear pairwise
    w min(|a-b|, T) (float64).  Rows and columns are the monotonic chains
    (node weight rho_s = 2, edge weight 1).  Returns the lower bound after
    every forward + backward iteration (the bound of the reparametrised chain
    decomposition, as in Kolmogorov 2006 Sec. 5)."""
    D = np.asarray(D, np.float64)
    H, W, K = D.shape
    k = np.arange(K)
    Vh = w_h * np.minimum(np.abs(k[:, None] - k[None, :]), T)
    Vv = w_v * np.minimum(np.abs(k[:, None] - k[None, :]), T)
    # messages into node (y, x) from its left / right / up / down neighbour
    mL = np.zeros((H, W, K)); mR = np.zeros((H, W, K)); mU = np.zeros((H, W, K)); mDn = np.zeros((H, W, K))

    def send(th_hat, m_back, V):
        out = np.min(0.5 * th_hat[:, None] - m_back[:, None] + V, axis=0)
        return out - out.min()

    bounds = []
    for _ in range(iters):
        for forward in (True, False):
            ys = range(H) if forward else range(H - 1, -1, -1)
            for y in ys:
                xs = range(W) if forward else range(W - 1, -1, -1)
                for x in xs:
                    th = D[y, x] + mL[y, x] + mR[y, x] + mU[y, x] + mDn[y, x]
                    if forward:
                        if x + 1 < W:
                            mL[y, x + 1] = send(th, mR[y, x], Vh)
                        if y + 1 < H:
                            mU[y + 1, x] = send(th, mDn[y, x], Vv)
                    else:
                        if x > 0:
                            mR[y, x - 1] = send(th, mL[y, x], Vh)
                        if y > 0:
                            mDn[y - 1, x] = send(th, mU[y, x], Vv)
        # bound: reparametrised unaries split in halves between the row and the
        # column chain of every node; each chain's minimum by dynamic programming
        th = D + mL + mR + mU + mDn
        lb = 0.0
        for y in range(H):                       # row chains: 0.5 th + reparametrised horizontal edges
            u = 0.5 * th[y]
            c = u[0].copy()
            for x in range(1, W):
                c = np.min(c[:, None] + Vh - mR[y, x - 1][:, None] - mL[y, x][None, :], axis=0) + u[x]
            lb += c.min()
        for x in range(W):                       # column chains: 0.5 th + reparametrised vertical edges
            u = 0.5 * th[:, x]
            c = u[0].copy()
            for y in range(1, H):
                c = np.min(c[:, None] + Vv - mDn[y - 1, x][:, None] - mU[y, x][None, :], axis=0) + u[y]
            lb += c.min()
        bounds.append(lb)
    return bounds
