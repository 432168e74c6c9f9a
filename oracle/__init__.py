"""CPU oracle for census + Dual MM with hierarchical minorants (arXiv 1601.06274).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1601_06274_b200``) never imports it.

This module is argument marshalling (numpy <-> ctypes) over ``dmm_oracle.c``;
every step of the arithmetic is in that file, which cites PAPER.md per function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dmm_oracle.c")
_LIB = os.path.join(_HERE, "libdmm_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP) into oracle/libdmm_oracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dmm_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-fopenmp", "-Wall", "-Wextra",
             "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int, ctypes.c_int64
        lib.oracle_census.argtypes = [P, i32, i32, i32, P]
        lib.oracle_cost_volume.argtypes = [P, P, i32, i32, i32, i32, i32, P]
        lib.oracle_flow_costs.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, P, P]
        lib.oracle_msg_direct.argtypes = [P, i32, i64, i32, P]
        lib.oracle_msg.argtypes = [P, i32, i64, i32, P]
        lib.oracle_min_marginals.argtypes = [P, i32, i32, i64, i32, P]
        lib.oracle_chain_min.argtypes = [P, i32, i32, i64, i32, P]
        lib.oracle_chain_min.restype = i64
        lib.oracle_hm.argtypes = [P, i32, i32, i64, i32, P]
        lib.oracle_dmm.argtypes = [P, i32, i32, i32, i32, i32, i32, i32, i32, P, P, P, P, P, i32]
        lib.oracle_energy.argtypes = [P, P, i32, i32, i32, i32, i32, i32]
        lib.oracle_energy.restype = i64
        lib.oracle_edge_weights.argtypes = [P, i32, i32, P, P]
        lib.oracle_dmm_general.argtypes = [P, i32, i32, i32, i32, i32, Pen, P, P, i32, i32, P, P, P, P, P, i32]
        lib.oracle_energy_general.argtypes = [P, P, i32, i32, i32, i32, i32, Pen, P, P, i32]
        lib.oracle_energy_general.restype = i64
        lib.oracle_hm_general.argtypes = [P, i32, i32, i32, Pen, P, P]
        lib.oracle_iter_minorant.argtypes = [P, i32, i32, i32, Pen, P, i32, i32, P]
        lib.oracle_naive_minorant.argtypes = [P, i32, i32, i32, Pen, P, P]
        lib.oracle_dmm_minorant.argtypes = [P, i32, i32, i32, i32, i32, Pen, P, P, i32, i32, i32, i32, i32,
                                            P, P, P, P, P, i32]
        _lib = lib
    return _lib


class Pen(ctypes.Structure):
    """oracle_pen: R(d) = min(e1*min(d, delta) + e2*max(d - delta, 0), c) (units 2^-F)."""
    _fields_ = [("e1", ctypes.c_int32), ("e2", ctypes.c_int32), ("delta", ctypes.c_int32), ("c", ctypes.c_int32)]


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def census(img, r: int = 2) -> np.ndarray:
    img = _c(img, np.uint8)
    H, W = img.shape
    out = np.zeros((H, W), np.uint32)
    if _load().oracle_census(_p(img), W, H, r, _p(out)):
        raise ValueError("oracle_census: bad arguments")
    return out


def cost_volume(cl, cr, d_min: int, K: int, oob: int = 12) -> np.ndarray:
    cl, cr = _c(cl, np.uint32), _c(cr, np.uint32)
    H, W = cl.shape
    D = np.zeros((H, W, K), np.uint8)
    if _load().oracle_cost_volume(_p(cl), _p(cr), W, H, d_min, K, oob, _p(D)):
        raise ValueError("oracle_cost_volume: bad arguments")
    return D


def flow_costs(c1, c2, u1_min: int, K1: int, u2_min: int, K2: int, oob: int = 12):
    """Optimistic decoupled flow costs (Eq. flow-decoupled-costs):
    returns (f1 [H][W][K1], f2 [H][W][K2])."""
    c1, c2 = _c(c1, np.uint32), _c(c2, np.uint32)
    H, W = c1.shape
    f1 = np.zeros((H, W, K1), np.uint8)
    f2 = np.zeros((H, W, K2), np.uint8)
    if _load().oracle_flow_costs(_p(c1), _p(c2), W, H, u1_min, K1, u2_min, K2, oob, _p(f1), _p(f2)):
        raise ValueError("oracle_flow_costs: bad arguments")
    return f1, f2


def msg(a, ws: int, T: int, direct: bool = False) -> np.ndarray:
    a = _c(a, np.int64)
    out = np.zeros_like(a)
    fn = _load().oracle_msg_direct if direct else _load().oracle_msg
    fn(_p(a), a.shape[0], ws, T, _p(out))
    return out


def min_marginals(F, ws: int, T: int) -> np.ndarray:
    F = _c(F, np.int64)
    n, K = F.shape
    m = np.zeros_like(F)
    _load().oracle_min_marginals(_p(F), n, K, ws, T, _p(m))
    return m


def chain_min(F, ws: int, T: int):
    F = _c(F, np.int64)
    n, K = F.shape
    x = np.zeros(n, np.int32)
    v = _load().oracle_chain_min(_p(F), n, K, ws, T, _p(x))
    return int(v), x


def hm(F, ws: int, T: int) -> np.ndarray:
    F = _c(F, np.int64)
    n, K = F.shape
    lam = np.zeros_like(F)
    _load().oracle_hm(_p(F), n, K, ws, T, _p(lam))
    return lam


def dmm(D, w_h: int, w_v: int, T: int, Fbits: int, iters: int, nthreads: int = 1):
    """Returns dict(fdual, gdual, labels, bound_hist, energy) (all exact ints)."""
    D = _c(D, np.uint8)
    H, W, K = D.shape
    f = np.zeros((H, W, K), np.int64)
    g = np.zeros((H, W, K), np.int64)
    lab = np.zeros((H, W), np.int32)
    bh = np.zeros(2 * max(iters, 1), np.int64)
    e = np.zeros(1, np.int64)
    rc = _load().oracle_dmm(_p(D), W, H, K, w_h, w_v, T, Fbits, iters, _p(f), _p(g), _p(lab),
                            _p(bh), _p(e), nthreads)
    if rc:
        raise ValueError("oracle_dmm: bad arguments")
    return dict(fdual=f, gdual=g, labels=lab, bound_hist=bh, energy=int(e[0]))


def energy(D, labels, w_h: int, w_v: int, T: int) -> int:
    D = _c(D, np.uint8)
    labels = _c(labels, np.int32)
    H, W, K = D.shape
    return int(_load().oracle_energy(_p(D), _p(labels), W, H, K, w_h, w_v, T))


def solve(left, right, d_min: int, K: int, w: int = 3, T: int = 4, Fbits: int = 4,
          iters: int = 4, r: int = 2, oob: int | None = None, nthreads: int = 1):
    """Whole path on the CPU: census x2 -> cost volume -> DMM."""
    if oob is None:
        oob = ((2 * r + 1) ** 2 - 1) // 2
    cl, cr = census(left, r), census(right, r)
    D = cost_volume(cl, cr, d_min, K, oob)
    out = dmm(D, w, w, T, Fbits, iters, nthreads)
    out.update(codes_left=cl, codes_right=cr, D=D)
    return out


# ---------------------------------------------------- NEXT-3 general model
def edge_weights(img):
    """Quantised edge-aware weights (om_h, om_v) in [1, 16] (reading R30)."""
    img = _c(img, np.uint8)
    H, W = img.shape
    oh = np.zeros((H, W), np.uint8)
    ov = np.zeros((H, W), np.uint8)
    _load().oracle_edge_weights(_p(img), W, H, _p(oh), _p(ov))
    return oh, ov


def hm_general(F, w: int, pen, om=None) -> np.ndarray:
    F = _c(F, np.int64)
    n, K = F.shape
    lam = np.zeros_like(F)
    omc = None if om is None else _c(om, np.uint8)
    _load().oracle_hm_general(_p(F), n, K, w, Pen(*pen), _p(omc), _p(lam))
    return lam


def dmm_general(D, w_h: int, w_v: int, pen, Fbits: int, iters: int, om_h=None, om_v=None, nthreads: int = 1):
    """Dual MM with the general penalty pen = (e1, e2, delta, c) and optional
    edge weights; returns dict(fdual, gdual, labels, bound_hist, energy)."""
    D = _c(D, np.uint8)
    H, W, K = D.shape
    f = np.zeros((H, W, K), np.int64)
    g = np.zeros((H, W, K), np.int64)
    lab = np.zeros((H, W), np.int32)
    bh = np.zeros(2 * max(iters, 1), np.int64)
    e = np.zeros(1, np.int64)
    oh = None if om_h is None else _c(om_h, np.uint8)
    ov = None if om_v is None else _c(om_v, np.uint8)
    rc = _load().oracle_dmm_general(_p(D), W, H, K, w_h, w_v, Pen(*pen), _p(oh), _p(ov), Fbits, iters, _p(f), _p(g),
                                    _p(lab), _p(bh), _p(e), nthreads)
    if rc:
        raise ValueError("oracle_dmm_general: bad arguments")
    return dict(fdual=f, gdual=g, labels=lab, bound_hist=bh, energy=int(e[0]))


def energy_general(D, labels, w_h: int, w_v: int, pen, Fbits: int, om_h=None, om_v=None) -> int:
    D = _c(D, np.uint8)
    labels = _c(labels, np.int32)
    H, W, K = D.shape
    oh = None if om_h is None else _c(om_h, np.uint8)
    ov = None if om_v is None else _c(om_v, np.uint8)
    return int(_load().oracle_energy_general(_p(D), _p(labels), W, H, K, w_h, w_v, Pen(*pen), _p(oh), _p(ov), Fbits))


# ------------------------------------------------------ NEXT-4 minorants
def iter_minorant(F, w: int, pen, om=None, max_pass: int = 3, gshift: int = 2) -> np.ndarray:
    F = _c(F, np.int64)
    n, K = F.shape
    lam = np.zeros_like(F)
    omc = None if om is None else _c(om, np.uint8)
    _load().oracle_iter_minorant(_p(F), n, K, w, Pen(*pen), _p(omc), max_pass, gshift, _p(lam))
    return lam


def naive_minorant(F, w: int, pen, om=None) -> np.ndarray:
    F = _c(F, np.int64)
    n, K = F.shape
    lam = np.zeros_like(F)
    omc = None if om is None else _c(om, np.uint8)
    _load().oracle_naive_minorant(_p(F), n, K, w, Pen(*pen), _p(omc), _p(lam))
    return lam


def dmm_minorant(D, w_h: int, w_v: int, pen, Fbits: int, iters: int, minorant: int, max_pass: int = 3,
                 gshift: int = 2, om_h=None, om_v=None, nthreads: int = 1):
    """Dual MM with minorant 0 hierarchical / 1 iterative / 2 naive."""
    D = _c(D, np.uint8)
    H, W, K = D.shape
    f = np.zeros((H, W, K), np.int64)
    g = np.zeros((H, W, K), np.int64)
    lab = np.zeros((H, W), np.int32)
    bh = np.zeros(2 * max(iters, 1), np.int64)
    e = np.zeros(1, np.int64)
    oh = None if om_h is None else _c(om_h, np.uint8)
    ov = None if om_v is None else _c(om_v, np.uint8)
    rc = _load().oracle_dmm_minorant(_p(D), W, H, K, w_h, w_v, Pen(*pen), _p(oh), _p(ov), Fbits, iters, minorant,
                                     max_pass, gshift, _p(f), _p(g), _p(lab), _p(bh), _p(e), nthreads)
    if rc:
        raise ValueError("oracle_dmm_minorant: bad arguments")
    return dict(fdual=f, gdual=g, labels=lab, bound_hist=bh, energy=int(e[0]))
