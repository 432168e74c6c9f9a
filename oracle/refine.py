"""Continuous refinement oracle (NEXT-2 of SURVEY 8(f)): the non-convex
primal-dual refinement of a discrete stereo labelling, Sec. 2.4
and Sec. 3.1 of arXiv 1601.06274.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, smoke() and
bench.py's cpu_baseline / reference legs may import it.  Plain numpy, float64,
one function per step of the method in the paper's order and notation; no
fusion or reordering beyond what the iterates state.

Problem (Eq. compact_formulation): min_u D(u) + R(Au), with
  (Au)_ij = u_i - u_j over the 4-connected edges,
  R(Au) = sum_ij w_ij r((Au)_ij)  (Eq. regularizer-form),
  r = r_{eps,delta} - r_{0, C + delta - eps*delta}  (Eq. r-decompose),
  r_{a,b}(t) = a|t| if |t| <= b else |t| - b(1 - a).
Iterates (Eq. cont_iterates) on x = (u, q), y = (p, d = 1) with
A(x) = [Au; -<Au, q>], G(x) = R_-^*(q) + D~(u), F^*(y) = R_+^*(p),
grad A(x) = [[A, 0], [-A^T q, -Au]]:
  u+ = prox_{tau D~}(u - tau A^T (p - q))
  q+ = prox_{tau R_-^*}(q + tau A u)
  p+ = prox_{sigma R_+^*}(p + sigma A(2 u+ - u))
Prox of (w r_{a,b})^* (Eq. pprox): t' = t if |t| <= a w else
sign(t) max(a w, |t| - b * step), then clamp to [-w, w].
Data term: the two-slope convex approximation around the current
point, with the indicator of [u0 - h, u0 + h]; its prox; embedded in
a warping loop: `warps` re-approximations x `iters` iterations
(5 x 40 in the paper's timing run).

Readings of garbled / silent passages (R24-R28):
  R24 slopes: s1 = (D(u0) - D(u0 - h)) / h (left), s2 = (D(u0 + h) - D(u0)) / h
      (right); P:427's s2 = (D(u0) - D(u0+h))/h is -s1, a typo; "set s1 = s2 =
      (s1+s2)/2 if s2 < s1" then makes the function convex.
  R25 data prox: the exact prox of the two-slope function (kink at u0 maps to
      u0 in the middle case, P:434-440 prints "u^ - 0"), then the clamp.
  R26 D at a real label u: linear interpolation of the sampled cost volume,
      u clamped to [0, K-1] for the lookup.
  R27 constants: h = 1 label, tau = sigma = 0.35 (tau*sigma*||A||^2 < 1,
      ||A||^2 <= 8), p = q = 0 at the start and kept across warps, u starts at
      the discrete labelling; eps, delta, C, w from the caller (eps = 1,
      C = T, w = w_h / w_v reproduces the discrete truncated-linear model).
  R28 the conjugate's domain "alpha < |t*| < omega" is read as
      |t*| <= omega (value beta * max(0, |t*| - alpha*omega)), whose prox is
      P:390-397 exactly.
"""
from __future__ import annotations

import numpy as np


# ------------------------------------------------------------ regulariser
def r_ab(t, a: float, b: float):
    """r_{a,b}(t)."""
    t = np.abs(np.asarray(t, np.float64))
    return np.where(t <= b, a * t, t - b * (1.0 - a))


def r_dc(t, eps: float, delta: float, C: float):
    """r = r_{eps,delta} - r_{0, C + delta - eps*delta} (Eq. r-decompose)."""
    return r_ab(t, eps, delta) - r_ab(t, 0.0, C + delta - eps * delta)


def conj_w_rab(s, w: float, a: float, b: float):
    """(w r_{a,b})^*(s) (reading R28): b * max(0, |s| - a w) on |s| <= w, +inf outside."""
    s = np.abs(np.asarray(s, np.float64))
    return np.where(s <= w + 1e-12, b * np.maximum(0.0, s - a * w), np.inf)


def prox_conj(t, w, a: float, b: float, step: float):
    """Prox of step * (w r_{a,b})^* (Eq. pprox), componentwise."""
    t = np.asarray(t, np.float64)
    aw = a * w
    tp = np.where(np.abs(t) <= aw, t, np.sign(t) * np.maximum(aw, np.abs(t) - b * step))
    return np.clip(tp, -w, w)


# ---------------------------------------------------------------- operator A
def A(u):
    """(Au)_ij = u_i - u_j: horizontal edges (y, x)-(y, x+1) and vertical
    edges (y, x)-(y+1, x), each indexed by its first pixel."""
    return u[:, :-1] - u[:, 1:], u[:-1, :] - u[1:, :]


def AT(ph, pv, shape):
    """Adjoint of A: node i gets +p_ij of its edges as first node, -p of the
    edges where it is the second node."""
    out = np.zeros(shape, np.float64)
    out[:, :-1] += ph
    out[:, 1:] -= ph
    out[:-1, :] += pv
    out[1:, :] -= pv
    return out


# ------------------------------------------------------------------ data
def D_interp(D, u):
    """D at a real label u (reading R26): linear interpolation between labels."""
    H, W, K = D.shape
    uc = np.clip(u, 0.0, K - 1.0)
    k0 = np.minimum(np.floor(uc).astype(np.int64), K - 1)
    k1 = np.minimum(k0 + 1, K - 1)
    f = uc - k0
    yy, xx = np.mgrid[0:H, 0:W]
    d0 = D[yy, xx, k0].astype(np.float64)
    d1 = D[yy, xx, k1].astype(np.float64)
    return (1.0 - f) * d0 + f * d1


def slopes(D, u0, h: float):
    """Two-slope convex approximation around u0 (reading R24)."""
    s1 = (D_interp(D, u0) - D_interp(D, u0 - h)) / h
    s2 = (D_interp(D, u0 + h) - D_interp(D, u0)) / h
    avg = 0.5 * (s1 + s2)
    bad = s2 < s1
    return np.where(bad, avg, s1), np.where(bad, avg, s2)


def prox_data(uh, u0, s1, s2, tau: float, h: float):
    """Prox of tau * D~ (reading R25): soft threshold towards the
    kink u0 with the left / right slopes, then clamp to [u0 - h, u0 + h]."""
    v = np.where(uh > u0 + tau * s2, uh - tau * s2, np.where(uh < u0 + tau * s1, uh - tau * s1, u0))
    return np.clip(v, u0 - h, u0 + h)


# ---------------------------------------------------------------- energy
def energy(D, u, w_h: float, w_v: float, eps: float, delta: float, C: float):
    """E(u) = D(u) + R(Au) (Eq. mrf_formulation, regularizer-form P:134)."""
    ah, av = A(u)
    return float(D_interp(D, u).sum() + w_h * r_dc(ah, eps, delta, C).sum() + w_v * r_dc(av, eps, delta, C).sum())


# ------------------------------------------------------------ the method
def refine(D, labels, w_h: float, w_v: float, eps: float = 1.0, delta: float = 1.0, C: float = 4.0,
           h: float = 1.0, tau: float = 0.35, sigma: float = 0.35, warps: int = 5, iters: int = 40):
    """Refine a discrete labelling (label units) of cost volume D [H][W][K].
    Returns the real-valued labelling u [H][W] (label units; disparity =
    d_min + u) and its energy."""
    D = np.asarray(D)
    H, W, K = D.shape
    u = np.asarray(labels, np.float64).copy()
    ph = np.zeros((H, W - 1)); pv = np.zeros((H - 1, W))
    qh = np.zeros((H, W - 1)); qv = np.zeros((H - 1, W))
    bp = C + delta - eps * delta                      # beta of R_-
    for _ in range(warps):
        u0 = u.copy()
        s1, s2 = slopes(D, u0, h)
        for _ in range(iters):
            # x^{k+1} = (I + tau dG)^{-1}(x^k - tau [grad A(x^k)]^T y^k), d = 1
            uh = u - tau * AT(ph - qh, pv - qv, (H, W))
            u_new = prox_data(uh, u0, s1, s2, tau, h)
            ah, av = A(u)
            qh = prox_conj(qh + tau * ah, w_h, 0.0, bp, tau)
            qv = prox_conj(qv + tau * av, w_v, 0.0, bp, tau)
            # y^{k+1} = (I + sigma dF^*)^{-1}(y^k + sigma A(2 x^{k+1} - x^k))
            bh, bv = A(2.0 * u_new - u)
            ph = prox_conj(ph + sigma * bh, w_h, eps, delta, sigma)
            pv = prox_conj(pv + sigma * bv, w_v, eps, delta, sigma)
            u = u_new
    return u, energy(D, u, w_h, w_v, eps, delta, C)


# ===================================================== optical flow (Sec. 3.2)
# The continuous refinement of a flow field u = (u1, u2): the same
# regulariser on each component (Eq. regularizer-form sums r over k = 1, 2,
# P:134-136), the data term approximated around u0 by the quadratic of Eq. 19
# with finite-difference gradient L and Hessian Q (step h), then
# the prox of Eq. 20.  Readings (R34-R36):
#   R34 Q is the full 2x2 finite-difference Hessian (second differences along
#       each component, the cross difference off the diagonal), its PSD part
#       by clipping the negative eigenvalue; the prox of Eq. 20 is the exact
#       prox of the quadratic, (I + tau Q) u = uh + tau (Q u0 - L), then the
#       componentwise clamp.  Eq. 20 prints the diagonal case with a garbled
#       denominator "1 + tau L^k" (read 1 + tau Q_kk).
#   R35 D(u) at a real displacement: bilinear interpolation of the census
#       Hamming costs at the four surrounding integer displacements (out-of-
#       image displacements cost oob, as in the discrete stage, R23).
#   R36 L^k = (D(u0 + h e_k) - D(u0 - h e_k)) / (2h), Q_kk = (D(u0 + h e_k) -
#       2 D(u0) + D(u0 - h e_k)) / h^2, Q_12 = (D(u0 + h e1 + h e2) - D(u0 + h e1
#       - h e2) - D(u0 - h e1 + h e2) + D(u0 - h e1 - h e2)) / (4 h^2) (central
#       differences), h = 1.

def _popc32(x):
    x = x.astype(np.uint32)
    x = x - ((x >> 1) & 0x55555555)
    x = (x & 0x33333333) + ((x >> 2) & 0x33333333)
    x = (x + (x >> 4)) & 0x0F0F0F0F
    return ((x * 0x01010101) & 0xFFFFFFFF) >> 24


def flow_cost_int(c1, c2, a, b, oob: int = 12):
    """D(x, y; a, b) = popcount(c1(x,y) ^ c2(x+a, y+b)) at integer displacements
    (arrays a, b of shape [H][W]), oob outside the image (Eq. flow-decoupled-costs)."""
    H, W = c1.shape
    yy, xx = np.mgrid[0:H, 0:W]
    xs, ys = xx + a, yy + b
    ok = (xs >= 0) & (xs < W) & (ys >= 0) & (ys < H)
    v = _popc32(c1 ^ c2[np.clip(ys, 0, H - 1), np.clip(xs, 0, W - 1)]).astype(np.float64)
    return np.where(ok, v, float(oob))


def flow_cost_bilinear(c1, c2, u1, u2, oob: int = 12):
    """D at real displacements (reading R35)."""
    a0 = np.floor(u1)
    b0 = np.floor(u2)
    fx = u1 - a0
    fy = u2 - b0
    a0 = a0.astype(np.int64)
    b0 = b0.astype(np.int64)
    d00 = flow_cost_int(c1, c2, a0, b0, oob)
    d10 = flow_cost_int(c1, c2, a0 + 1, b0, oob)
    d01 = flow_cost_int(c1, c2, a0, b0 + 1, oob)
    d11 = flow_cost_int(c1, c2, a0 + 1, b0 + 1, oob)
    return ((1.0 - fx) * (1.0 - fy) * d00 + fx * (1.0 - fy) * d10) + ((1.0 - fx) * fy * d01 + fx * fy * d11)


def psd_part(a, b, c):
    """Positive-semidefinite part of the symmetric 2x2 [[a, b], [b, c]] (reading
    R34): the negative eigenvalue clipped to 0.  Eigenvalues m +- rad with
    m = (a + c)/2, rad = sqrt(((a - c)/2)^2 + b^2); when l1 = m + rad > 0 >
    l2 = m - rad the part is l1 P1, P1 = (Q - l2 I) / (l1 - l2)."""
    a, b, c = (np.asarray(v, np.float64) for v in (a, b, c))
    m = 0.5 * (a + c)
    dl = 0.5 * (a - c)
    rad = np.sqrt(dl * dl + b * b)
    l1 = m + rad
    l2 = m - rad
    mixed = (l1 > 0.0) & (l2 < 0.0)
    s = np.where(mixed, l1 / np.where(mixed, 2.0 * rad, 1.0), 0.0)
    pa = np.where(l2 >= 0.0, a, np.where(mixed, s * (a - l2), 0.0))
    pb = np.where(l2 >= 0.0, b, np.where(mixed, s * b, 0.0))
    pc = np.where(l2 >= 0.0, c, np.where(mixed, s * (c - l2), 0.0))
    return pa, pb, pc


def flow_quadratic(c1, c2, u1, u2, h: float, oob: int = 12, cost=None):
    """(L1, L2, Qa, Qb, Qc) of Eq. 19 around (u1, u2) (readings R34, R36): the
    central-difference gradient and Hessian [[Qa, Qb], [Qb, Qc]] of D (step h),
    PSD part.  `cost(u1, u2)` defaults to the bilinear census cost (R35)."""
    if cost is None:
        cost = lambda v1, v2: flow_cost_bilinear(c1, c2, v1, v2, oob)  # noqa: E731
    d0 = cost(u1, u2)
    dp1 = cost(u1 + h, u2)
    dm1 = cost(u1 - h, u2)
    dp2 = cost(u1, u2 + h)
    dm2 = cost(u1, u2 - h)
    dpp = cost(u1 + h, u2 + h)
    dpm = cost(u1 + h, u2 - h)
    dmp = cost(u1 - h, u2 + h)
    dmm = cost(u1 - h, u2 - h)
    L1 = (dp1 - dm1) / (2.0 * h)
    L2 = (dp2 - dm2) / (2.0 * h)
    a = (dp1 - 2.0 * d0 + dm1) / (h * h)
    c = (dp2 - 2.0 * d0 + dm2) / (h * h)
    b = ((dpp - dpm) - (dmp - dmm)) / (4.0 * h * h)
    Qa, Qb, Qc = psd_part(a, b, c)
    return L1, L2, Qa, Qb, Qc


def prox_quadratic(uh1, uh2, u01, u02, L1, L2, Qa, Qb, Qc, tau: float, h: float):
    """Prox of tau * D~ for the quadratic of Eq. 19 (Eq. 20, reading R34): the
    minimiser of tau (L^T (u - u0) + (u - u0)^T Q (u - u0) / 2) + |u - uh|^2 / 2,
    i.e. (I + tau Q) u = uh + tau (Q u0 - L) solved by Cramer's rule, then each
    component clamped to [u0 - h, u0 + h] (Eq. 20's clamp).  For a diagonal Q
    this is Eq. 20's componentwise quotient with the denominator 1 + tau Q_kk."""
    r1 = uh1 + tau * ((Qa * u01 + Qb * u02) - L1)
    r2 = uh2 + tau * ((Qb * u01 + Qc * u02) - L2)
    a11 = 1.0 + tau * Qa
    a22 = 1.0 + tau * Qc
    a12 = tau * Qb
    det = a11 * a22 - a12 * a12
    v1 = (a22 * r1 - a12 * r2) / det
    v2 = (a11 * r2 - a12 * r1) / det
    return np.clip(v1, u01 - h, u01 + h), np.clip(v2, u02 - h, u02 + h)


def flow_energy(c1, c2, u1, u2, w_h, w_v, eps, delta, C, oob: int = 12):
    e = flow_cost_bilinear(c1, c2, u1, u2, oob).sum()
    for u in (u1, u2):
        ah, av = A(u)
        e += w_h * r_dc(ah, eps, delta, C).sum() + w_v * r_dc(av, eps, delta, C).sum()
    return float(e)


def flow_refine(c1, c2, u1, u2, w_h: float, w_v: float, eps: float = 1.0, delta: float = 1.0, C: float = 4.0,
                h: float = 1.0, tau: float = 0.35, sigma: float = 0.35, warps: int = 5, iters: int = 40,
                oob: int = 12):
    """Refine an integer flow field (u1, u2) (pixels).  Per warp the quadratic
    model is rebuilt at the current u; then `iters` iterations of the stereo
    refinement's PDHG run on both components in lockstep: the primal step's
    prox is the joint 2-D prox of Eq. 20 (the components couple there and in
    the model), the duals p, q of each component's regulariser are separate
    (Eq. regularizer-form sums r over k = 1, 2).  Returns (u1, u2, energy)."""
    c1 = np.asarray(c1, np.uint32)
    c2 = np.asarray(c2, np.uint32)
    H, W = c1.shape
    us = [np.asarray(u1, np.float64).copy(), np.asarray(u2, np.float64).copy()]
    st = [dict(ph=np.zeros((H, W - 1)), pv=np.zeros((H - 1, W)), qh=np.zeros((H, W - 1)), qv=np.zeros((H - 1, W)))
          for _ in range(2)]
    bp = C + delta - eps * delta
    for _ in range(warps):
        L1, L2, Qa, Qb, Qc = flow_quadratic(c1, c2, us[0], us[1], h, oob)
        u01, u02 = us[0].copy(), us[1].copy()
        for _ in range(iters):
            uh = [us[k] - tau * AT(st[k]["ph"] - st[k]["qh"], st[k]["pv"] - st[k]["qv"], (H, W)) for k in range(2)]
            un = prox_quadratic(uh[0], uh[1], u01, u02, L1, L2, Qa, Qb, Qc, tau, h)
            for k in range(2):
                s, u = st[k], us[k]
                ah, av = A(u)
                s["qh"] = prox_conj(s["qh"] + tau * ah, w_h, 0.0, bp, tau)
                s["qv"] = prox_conj(s["qv"] + tau * av, w_v, 0.0, bp, tau)
                bh, bv = A(2.0 * un[k] - u)
                s["ph"] = prox_conj(s["ph"] + sigma * bh, w_h, eps, delta, sigma)
                s["pv"] = prox_conj(s["pv"] + sigma * bv, w_v, eps, delta, sigma)
            us = [un[0], un[1]]
    return us[0], us[1], flow_energy(c1, c2, us[0], us[1], w_h, w_v, eps, delta, C, oob)
