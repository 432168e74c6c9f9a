"""Exhaustive enumeration helpers for the oracle pins (tiny instances only).

These evaluate the *definitions* (Eq.3 P:150 energies, Def. P:631 min-marginals,
Eq.7 P:222 modular minorants) by listing every labelling; they share nothing
with the oracle's dynamic programming.
"""
import itertools

import numpy as np


def pen(ws, T, a, b):
    return ws * np.minimum(np.abs(np.asarray(a) - np.asarray(b)), T)


def all_labellings(n, K):
    """(K^n, n) int array of every labelling."""
    return np.array(list(itertools.product(range(K), repeat=n)), dtype=np.int64).reshape(-1, n)


def chain_energies(F, ws, T):
    """Energy F(x) = sum F_i(x_i) + sum ws min(|x_i - x_{i+1}|, T) for all x."""
    F = np.asarray(F, np.int64)
    n, K = F.shape
    X = all_labellings(n, K)
    e = F[np.arange(n)[None, :], X].sum(1)
    if n > 1:
        e = e + pen(ws, T, X[:, :-1], X[:, 1:]).sum(1)
    return X, e


def modular_values(lam, X):
    lam = np.asarray(lam, np.int64)
    n = lam.shape[0]
    return lam[np.arange(n)[None, :], X].sum(1)


def chain_min_marginals(F, ws, T):
    X, e = chain_energies(F, ws, T)
    F = np.asarray(F)
    n, K = F.shape
    m = np.full((n, K), np.iinfo(np.int64).max, np.int64)
    for i in range(n):
        for k in range(K):
            m[i, k] = e[X[:, i] == k].min()
    return m


def grid_energies(D, w_h, w_v, T, scale=1):
    """All labellings of an (H, W) grid with unaries D (H, W, K) scaled by `scale`."""
    D = np.asarray(D, np.int64) * scale
    H, W, K = D.shape
    X = all_labellings(H * W, K).reshape(-1, H, W)
    e = D[np.arange(H)[None, :, None], np.arange(W)[None, None, :], X].sum((1, 2))
    if W > 1:
        e = e + pen(w_h * scale, T, X[:, :, :-1], X[:, :, 1:]).sum((1, 2))
    if H > 1:
        e = e + pen(w_v * scale, T, X[:, :-1, :], X[:, 1:, :]).sum((1, 2))
    return X, e


def grid_part_energies(X, D, w_h, w_v, T, scale):
    """(f(x), g(x)) for the chain split of reading R3: f = unaries + horizontal
    pairwise, g = vertical pairwise."""
    D = np.asarray(D, np.int64) * scale
    H, W, K = D.shape
    f = D[np.arange(H)[None, :, None], np.arange(W)[None, None, :], X].sum((1, 2))
    if W > 1:
        f = f + pen(w_h * scale, T, X[:, :, :-1], X[:, :, 1:]).sum((1, 2))
    g = np.zeros_like(f)
    if H > 1:
        g = g + pen(w_v * scale, T, X[:, :-1, :], X[:, 1:, :]).sum((1, 2))
    return f, g


def grid_modular(lam, X):
    lam = np.asarray(lam, np.int64)
    H, W, K = lam.shape
    return lam[np.arange(H)[None, :, None], np.arange(W)[None, None, :], X].sum((1, 2))
