"""Pins for the oracle's chain primitives: Msg, min-marginals, Viterbi, HM.

Every pin is independent of the oracle's own arithmetic: exhaustive enumeration,
closed forms, or values printed in the paper (tests/golden/)."""
import json
import os

import numpy as np
import pytest

from bruteforce import chain_energies, chain_min_marginals, modular_values

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _appendix():
    with open(os.path.join(GOLD, "appendix_chain.json")) as f:
        return json.load(f)


# ----------------------------------------------------------------- Msg
def test_msg_dt_equals_definition(orc):
    """O(K) lower envelope == O(K^2) enumeration of Eq. msg-pass."""
    rng = np.random.default_rng(1)
    for _ in range(3000):
        K = int(rng.integers(1, 40))
        ws = int(rng.integers(0, 50))
        T = int(rng.integers(1, K + 3))
        a = rng.integers(-1000, 1000, size=K)
        assert np.array_equal(orc.msg(a, ws, T), orc.msg(a, ws, T, direct=True))


def test_msg_closed_forms(orc):
    # zero pairwise: out(b) = min_a a(a)  (SPEC S:137 TRIVIAL)
    a = np.array([5, -3, 7, 2])
    assert np.array_equal(orc.msg(a, 0, 3), np.full(4, -3))
    # Potts (T=1) weight w, source (0,5,5) -> (0, min(5,w), min(5,w))
    for w in (1, 3, 5, 9):
        assert list(orc.msg([0, 5, 5], w, 1)) == [0, min(5, w), min(5, w)]
    # truncated linear w=1, T=2, source (0,10,10,10) -> (0,1,2,2)
    assert list(orc.msg([0, 10, 10, 10], 1, 2)) == [0, 1, 2, 2]
    # shift equivariance Msg(a + c) = Msg(a) + c (exact integers)
    a = np.array([3, 9, -4, 0, 12])
    assert np.array_equal(orc.msg(a + 17, 4, 2), orc.msg(a, 4, 2) + 17)


def test_msg_symmetric_direction(orc):
    """f_ij symmetric => Msg_ij(a) reversed == Msg_ji(a reversed) (K-reversal)."""
    rng = np.random.default_rng(2)
    for _ in range(200):
        K = int(rng.integers(1, 20))
        a = rng.integers(-50, 50, size=K)
        assert np.array_equal(orc.msg(a[::-1], 3, 4)[::-1], orc.msg(a, 3, 4))


def test_msg_bounce_identity(orc):
    """Msg(-Msg(t)) == -Msg(t): a Msg output phi is V-Lipschitz for the metric
    V(a,b) = ws*min(|a-b|,T) (triangle inequality of min(|.|,T)), so
    max_a phi(a) - V(a,b) = phi(b).  This is the identity the GPU Handshake
    uses for Alg.5's bounce-back phi_ji' = Msg(-phi_ij) (DESIGN.md
    "Bounce identity"); pinned here by O(K^2) enumeration, independently of the
    oracle's DT, and it fails for a non-metric pairwise term (checked below)."""
    rng = np.random.default_rng(11)

    def msg_enum(a, V):
        return np.array([min(a[x] + V[x][b] for x in range(len(a))) for b in range(len(a))])

    for _ in range(1500):
        K = int(rng.integers(1, 24))
        ws = int(rng.integers(0, 60))
        T = int(rng.integers(1, K + 3))
        V = [[ws * min(abs(x - b), T) for b in range(K)] for x in range(K)]
        t = rng.integers(-800, 800, size=K)
        phi = msg_enum(t, V)
        assert np.array_equal(msg_enum(-phi, V), -phi)
        assert np.array_equal(orc.msg(-orc.msg(t, ws, T), ws, T), -orc.msg(t, ws, T))
    # a non-metric pairwise term (squared distance) breaks it: the identity is
    # a property of the truncated-linear (metric) regulariser, not of Msg
    Vq = [[(x - b) ** 2 for b in range(3)] for x in range(3)]
    t = np.array([0, 100, 100])
    phi = msg_enum(t, Vq)
    assert not np.array_equal(msg_enum(-phi, Vq), -phi)


# ---------------------------------------------------------- min-marginals
def test_min_marginals_paper_potts5(orc):
    """Paper-printed min-marginals, Potts strength 5."""
    g = _appendix()
    F = np.array(g["unary_labels_by_nodes"]).T           # nodes x labels
    m = orc.min_marginals(F, 5, 1)
    mn = m - m.min(1, keepdims=True)
    assert np.array_equal(mn.T, np.array(g["potts5_min_marginals_normalised"]))


def test_min_marginals_bruteforce(orc):
    rng = np.random.default_rng(3)
    for _ in range(150):
        n = int(rng.integers(1, 6)); K = int(rng.integers(1, 5))
        ws = int(rng.integers(0, 6)); T = int(rng.integers(1, K + 2))
        F = rng.integers(-20, 30, size=(n, K))
        assert np.array_equal(orc.min_marginals(F, ws, T), chain_min_marginals(F, ws, T))


def test_chain_min_bruteforce(orc):
    rng = np.random.default_rng(4)
    for _ in range(150):
        n = int(rng.integers(1, 6)); K = int(rng.integers(1, 5))
        ws = int(rng.integers(0, 6)); T = int(rng.integers(1, K + 2))
        F = rng.integers(-20, 30, size=(n, K))
        X, e = chain_energies(F, ws, T)
        v, x = orc.chain_min(F, ws, T)
        assert v == e.min()
        # lexicographically smallest optimum (X is enumerated in lex order)
        assert list(x) == list(X[np.argmin(e)])


def test_energy_spec_example(orc):
    """SPEC S:66 example: appendix chain, Potts 1, unary argmin labelling -> 3."""
    g = _appendix()
    F = np.array(g["unary_labels_by_nodes"]).T
    D = F.reshape(1, 6, 3).astype(np.uint8)
    lab = np.array(g["potts1_energy_of_unary_argmin"]["labels"]).reshape(1, 6)
    assert orc.energy(D, lab, 1, 0, 1) == g["potts1_energy_of_unary_argmin"]["energy"]


# --------------------------------------------------- hierarchical minorant
def _check_minorant(F, ws, T, lam):
    X, e = chain_energies(F, ws, T)
    lv = modular_values(lam, X)
    # minorant: lam(x) <= F(x) for every labelling (Def. P:193 / Prop.1)
    assert np.all(lv <= e)
    # exact: sum of per-node minima == chain optimum (so exact at x*, Prop.1)
    assert lam.min(1).sum() == e.min()
    # maximal: all min-marginals of F - lam are 0 (Lemma 1)
    slack = e - lv
    n, K = lam.shape
    for i in range(n):
        for k in range(K):
            assert slack[X[:, i] == k].min() == 0, (i, k)


def test_hm_minorant_exact_maximal_bruteforce(orc):
    """HM is a valid, exact and maximal minorant on random chains
    (floor rounding of reading R9 included: inputs are arbitrary integers)."""
    rng = np.random.default_rng(5)
    for _ in range(400):
        n = int(rng.integers(1, 7)); K = int(rng.integers(1, 5))
        ws = int(rng.integers(0, 9)); T = int(rng.integers(1, K + 2))
        F = rng.integers(-15, 40, size=(n, K))
        _check_minorant(F, ws, T, orc.hm(F, ws, T))


def test_hm_zero_pairwise(orc):
    """ws = 0: pieces never interact; lambda_i = F_i + c_i with sum c_i = 0."""
    rng = np.random.default_rng(6)
    for _ in range(50):
        n = int(rng.integers(1, 30)); K = int(rng.integers(1, 9))
        F = rng.integers(-100, 100, size=(n, K))
        lam = orc.hm(F, 0, 3)
        c = lam - F
        assert np.all(c == c[:, :1])
        assert c[:, 0].sum() == 0


def test_hm_single_node(orc):
    F = np.array([[4, -2, 7]])
    assert np.array_equal(orc.hm(F, 5, 2), F)


def test_hm_two_node_prose_in_reals(orc):
    """Two-node procedure in exact arithmetic: with even inputs the
    floor of reading R9 never rounds, and Alg.5 must equal the prose:
    lam1 = m1/2 + m1^{f-lam}, lam2 = m2^{f-lam} (paper's 4 bullet steps)."""
    rng = np.random.default_rng(7)
    for _ in range(300):
        K = int(rng.integers(1, 6)); ws = 2 * int(rng.integers(0, 6)); T = int(rng.integers(1, K + 2))
        F = 2 * rng.integers(-20, 20, size=(2, K))
        P = ws * np.minimum(np.abs(np.arange(K)[:, None] - np.arange(K)[None, :]), T)
        m1 = F[0] + (F[1][None, :] + P).min(1)               # min-marginal at node 1
        l1 = m1 // 2                                          # exact (even)
        phi12 = ((F[0] - l1)[:, None] + P).min(0)
        l2 = phi12 + F[1]                                     # whole remaining m2
        phi21 = ((F[1] - l2)[None, :] + P).min(1)
        l1 = l1 + (F[0] - l1 + phi21)                         # lam1 += m1^{f-lam}
        lam = orc.hm(F, ws, T)
        assert np.array_equal(lam[0], l1) and np.array_equal(lam[1], l2)


def test_hm_appendix_chain_independent_prototype(orc):
    """Values from the survey's independent prototype (not paper
    values -- the paper prints none for HM)."""
    with open(os.path.join(GOLD, "hm_appendix_survey.json")) as f:
        g = json.load(f)
    F = np.array(_appendix()["unary_labels_by_nodes"]).T
    assert np.array_equal(orc.hm(F * 16, 16, 1), np.array(g["potts1_F4"]))
    assert np.array_equal(orc.hm(F * 16, 80, 1), np.array(g["potts5_F4"]))
    assert np.array_equal(orc.hm(F, 1, 1), np.array(g["potts1_F0"]))


def test_hm_long_chain_exact(orc):
    """Exactness on long chains against Viterbi (n up to 300, K up to 20)."""
    rng = np.random.default_rng(8)
    for n in (7, 31, 64, 100, 301):
        K = int(rng.integers(2, 21)); ws = int(rng.integers(0, 60)); T = int(rng.integers(1, K + 1))
        F = rng.integers(0, 400, size=(n, K))
        lam = orc.hm(F, ws, T)
        assert lam.min(1).sum() == orc.chain_min(F, ws, T)[0]
        # maximality via DP min-marginals of F - lam (dp itself pinned above)
        mm = orc.min_marginals(F - lam, ws, T)
        assert np.all(mm == 0)


# ------------------------------------- HM rounding / split pins (R7, R9)
def _split_tree_check(lam, lo, hi, opt):
    """Every piece [lo, hi] of the recursion (R5, left part floor(len/2), R7)
    whose optimum is `opt` hands ceil(opt/2) to its left part and floor(opt/2)
    to its right part: the Handshake splits the min-marginal m_i with floor
    halving (Alg.5 line 3, reading R9), so the right part receives
    min floor((m_i - 2 phi_ji)/2) + min phi_ji = floor(opt/2), and exactness of
    the whole minorant leaves the rest to the left part.  A piece's optimum is
    the sum of its nodes' minima (exactness, recursively)."""
    piece = lam[lo:hi + 1].min(1).sum()
    assert piece == opt, (lo, hi, piece, opt)
    if lo == hi:
        return
    i = lo + (hi - lo + 1) // 2 - 1
    _split_tree_check(lam, lo, i, -(-opt // 2))
    _split_tree_check(lam, i + 1, hi, opt // 2)


def test_hm_recursive_optimum_split(orc):
    """Pins R7 (split point) and R9 (floor halving) at every level of the
    recursion: a ceil-halving or ceil-split variant fails on odd optima / odd
    lengths.  The chain optimum comes from the plain Viterbi (never calls HM)."""
    rng = np.random.default_rng(21)
    for _ in range(600):
        n = int(rng.integers(1, 70)); K = int(rng.integers(1, 7))
        ws = int(rng.integers(0, 40)); T = int(rng.integers(1, K + 2))
        F = rng.integers(-50, 200, size=(n, K))
        lam = orc.hm(F, ws, T)
        _split_tree_check(lam, 0, n - 1, orc.chain_min(F, ws, T)[0])


def _hm_chains():
    with open(os.path.join(GOLD, "hm_chains.json")) as f:
        return json.load(f)


def test_hm_golden_chains(orc):
    """Odd-length and deeper chains (n = 7, 13, 25; F = 0, 4) of
    tests/golden/hm_chains.json: the stored values satisfy the independent pins
    (Viterbi optimum, recursive optimum split, maximality via DP min-marginals,
    brute-force minorant on n = 7) and the oracle reproduces them."""
    g = _hm_chains()
    ws0, T = g["w"], g["T"]
    for c in g["chains"]:
        D = np.array(c["D"], np.int64) << c["F"]
        lam = np.array(c["lam"], np.int64)
        ws = ws0 << c["F"]
        v, _ = orc.chain_min(D, ws, T)
        assert v == c["opt"]
        _split_tree_check(lam, 0, c["n"] - 1, v)
        assert np.all(orc.min_marginals(D - lam, ws, T) == 0)
        if c["n"] == 7:
            _check_minorant(D, ws, T, lam)
        assert np.array_equal(orc.hm(D, ws, T), lam)


def test_hm_golden_hand_check(orc):
    """The hand-worked first Handshake of chains[0] (Alg.5 lines 1-4 with the
    O(K^2) Msg definition): its messages agree with the brute-force Msg and the
    stored lambda's top-level split matches the hand-computed optima."""
    g = _hm_chains()
    h = g["_hand_check"]
    c = g["chains"][0]
    D = np.array(c["D"], np.int64)
    ws, T = g["w"], g["T"]
    assert np.array_equal(orc.msg(np.array(h["alg5_line3_floor_half_m_i_minus_2phi_ji"]), ws, T, direct=True),
                          h["alg5_line3_phi_ij"])
    assert np.array_equal(orc.msg(-np.array(h["alg5_line3_phi_ij"]), ws, T, direct=True),
                          h["alg5_line4_phi_ji_bounced"])
    assert np.array_equal(orc.msg(D[3] + np.array(h["phi_into_j_from_right"]), ws, T, direct=True),
                          h["alg5_line1_phi_ji"])
    lam = np.array(c["lam"])
    assert lam[:3].min(1).sum() == h["left_part_optimum"] and lam[3:].min(1).sum() == h["right_part_optimum"]
    # leaves of the left part see phi_ji' at node i = 2 as their right boundary
    assert min(np.array(h["alg5_line2_m_i"])) == h["chain_optimum"] == c["opt"]
