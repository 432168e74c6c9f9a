"""Seeded synthetic stereo pairs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no census, no costs, no messages):
it only draws images.  Recipes:

* ``random_dot``  (RD): left = i.i.d. uniform u8; ground-truth disparity =
  background plane + 2-3 fronto-parallel rectangles + one slanted plane rounded
  to integers; right = forward warp x -> x - d with a z-buffer (larger d wins),
  holes refilled with fresh uniform noise.
* ``warped_texture`` (WT): texture = 4 octaves (16, 8, 4, 2 px cells) of bilinearly upsampled
  uniform noise normalised to 0..255 plus N(0, 2^2) pixel noise; disparity either
  KITTI-like (ground plane d = clamp(0.35 (y - 170), 0, 110) scaled to the
  label range, background 5, six box "cars" with d in [20, 90]) or
  Middlebury-like (4-6 slanted planes spanning d in [30, 250] scaled to the
  label range); right view by the same z-buffer warp plus independent noise.

All generators take ``numpy.random.default_rng(seed)`` seeds and return
``(left, right, disparity)`` as ``uint8 (H, W)``, ``uint8 (H, W)``, ``int32 (H, W)``.
"""
from __future__ import annotations

import numpy as np


def _forward_warp(left: np.ndarray, disp: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    """right(y, x - d) = left(y, x); larger d wins (z-buffer); holes = fresh noise."""
    H, W = left.shape
    ys, xs = np.mgrid[0:H, 0:W]
    xr = xs - disp
    ok = (xr >= 0) & (xr < W)
    tgt = (ys * W + np.clip(xr, 0, W - 1))[ok]
    d = disp[ok]
    zbuf = np.full(H * W, -1, np.int64)
    np.maximum.at(zbuf, tgt, d)
    win = zbuf[tgt] == d           # unique per target: same y, same d => distinct x
    right = rng.integers(0, 256, size=H * W, dtype=np.int64)
    right[tgt[win]] = left[ok][win]
    return right.reshape(H, W).astype(np.uint8)


def _rects(rng, H, W, n, dlo, dhi, disp):
    for _ in range(n):
        h = int(rng.integers(max(2, H // 8), max(3, H // 3)))
        w = int(rng.integers(max(2, W // 8), max(3, W // 3)))
        y0 = int(rng.integers(0, max(1, H - h)))
        x0 = int(rng.integers(0, max(1, W - w)))
        disp[y0:y0 + h, x0:x0 + w] = int(rng.integers(dlo, dhi + 1))


def random_dot(W: int, H: int, max_disp: int, seed: int = 0):
    """RD pair with ground-truth disparities in [0, max_disp]."""
    rng = np.random.default_rng(seed)
    left = rng.integers(0, 256, size=(H, W), dtype=np.int64).astype(np.uint8)
    disp = np.full((H, W), int(rng.integers(0, max(1, max_disp // 4) + 1)), np.int64)
    # slanted plane over the lower third
    ys, xs = np.mgrid[0:H, 0:W]
    y0 = 2 * H // 3
    slant = np.rint(max_disp * 0.25 + (max_disp * 0.5) * (xs / max(W - 1, 1))).astype(np.int64)
    disp[y0:, :] = slant[y0:, :]
    _rects(rng, H, W, int(rng.integers(2, 4)), max_disp // 3, max_disp, disp)
    disp = np.clip(disp, 0, max_disp)
    right = _forward_warp(left, disp, rng)
    return left, right, disp.astype(np.int32)


def _texture(rng, H, W):
    acc = np.zeros((H, W), np.float64)
    for octave in range(4):
        cell = 2 ** (4 - octave)             # 16, 8, 4, 2 px
        gh, gw = H // cell + 2, W // cell + 2
        g = rng.random((gh, gw))
        yy = np.arange(H) / cell
        xx = np.arange(W) / cell
        y0 = np.floor(yy).astype(int); x0 = np.floor(xx).astype(int)
        fy = (yy - y0)[:, None]; fx = (xx - x0)[None, :]
        a = g[y0][:, x0]; b = g[y0][:, x0 + 1]; c = g[y0 + 1][:, x0]; d = g[y0 + 1][:, x0 + 1]
        acc += (a * (1 - fx) * (1 - fy) + b * fx * (1 - fy) + c * (1 - fx) * fy + d * fx * fy) / (2 ** octave)
    acc = (acc - acc.min()) / max(acc.max() - acc.min(), 1e-12) * 255.0
    return acc


def warped_texture(W: int, H: int, max_disp: int, seed: int = 0, scene: str = "kitti"):
    """WT pair; scene 'kitti' (ground plane + cars) or 'middlebury' (slanted planes)."""
    rng = np.random.default_rng(seed)
    tex = _texture(rng, H, W)
    s = max_disp / (110.0 if scene == "kitti" else 250.0)
    ys, xs = np.mgrid[0:H, 0:W]
    if scene == "kitti":
        disp = np.full((H, W), 5.0 * s)
        gp = np.clip(0.35 * (ys - 170 * H / 375.0) * (375.0 / H), 0, 110) * s
        disp = np.maximum(disp, gp)
        for _ in range(6):
            h = int(rng.integers(max(2, H // 10), max(3, H // 4)))
            w = int(rng.integers(max(2, W // 16), max(3, W // 6)))
            y0 = int(rng.integers(H // 3, max(H // 3 + 1, H - h)))
            x0 = int(rng.integers(0, max(1, W - w)))
            disp[y0:y0 + h, x0:x0 + w] = rng.uniform(20, 90) * s
    elif scene == "middlebury":
        disp = np.full((H, W), 30.0 * s)
        n = int(rng.integers(4, 7))
        for q in range(n):
            a, b = rng.uniform(-0.05, 0.05, size=2) * (1000.0 / max(H, W))
            c = rng.uniform(30, 250)
            plane = np.clip(c + a * (xs - W / 2) + b * (ys - H / 2), 30, 250) * s
            if q == 0:
                disp = plane
            else:
                h = int(rng.integers(H // 6, H // 2)); w = int(rng.integers(W // 6, W // 2))
                y0 = int(rng.integers(0, H - h)); x0 = int(rng.integers(0, W - w))
                disp[y0:y0 + h, x0:x0 + w] = plane[y0:y0 + h, x0:x0 + w]
    else:
        raise ValueError(scene)
    disp = np.clip(np.rint(disp), 0, max_disp).astype(np.int64)
    left = np.clip(tex + rng.normal(0, 2, size=(H, W)), 0, 255).astype(np.uint8)
    right = _forward_warp(np.clip(tex, 0, 255).astype(np.uint8), disp, rng)
    right = np.clip(right + rng.normal(0, 2, size=(H, W)), 0, 255).astype(np.uint8)
    return left, right, disp.astype(np.int32)


def flow_pair(W: int, H: int, max_flow: int = 16, seed: int = 0):
    """Optical-flow pair (configs[3]): I1 = a warped texture,
    flow u = a smooth affine field plus two moving boxes, integer and within
    [-max_flow, max_flow - 1] per component; I2 is built so that
    I2(x + u1, y + u2) = I1(x, y): the texture sampled at the displaced
    coordinates, with a z-order-free backward construction (I1 samples the
    texture at x + u, I2 is the texture itself) plus independent N(0, 2^2)
    noise.  Returns (I1, I2, u1, u2) as uint8, uint8, int32, int32 (H, W)."""
    rng = np.random.default_rng(seed)
    pad = max_flow + 2
    tex = _texture(rng, H + 2 * pad, W + 2 * pad)
    ys, xs = np.mgrid[0:H, 0:W]
    a = rng.uniform(-0.5, 0.5, size=6)
    u1 = a[0] * max_flow * 0.5 + a[1] * max_flow * (xs - W / 2) / W + a[2] * max_flow * (ys - H / 2) / H
    u2 = a[3] * max_flow * 0.5 + a[4] * max_flow * (xs - W / 2) / W + a[5] * max_flow * (ys - H / 2) / H
    for _ in range(2):
        h = int(rng.integers(max(2, H // 8), max(3, H // 3)))
        w = int(rng.integers(max(2, W // 10), max(3, W // 4)))
        y0 = int(rng.integers(0, max(1, H - h)))
        x0 = int(rng.integers(0, max(1, W - w)))
        u1[y0:y0 + h, x0:x0 + w] = rng.uniform(-max_flow, max_flow - 1)
        u2[y0:y0 + h, x0:x0 + w] = rng.uniform(-max_flow, max_flow - 1)
    u1 = np.clip(np.rint(u1), -max_flow, max_flow - 1).astype(np.int64)
    u2 = np.clip(np.rint(u2), -max_flow, max_flow - 1).astype(np.int64)
    t = np.clip(tex, 0, 255)
    i1 = t[pad + ys + u2, pad + xs + u1]
    i2 = t[pad:pad + H, pad:pad + W]
    i1 = np.clip(i1 + rng.normal(0, 2, size=(H, W)), 0, 255).astype(np.uint8)
    i2 = np.clip(i2 + rng.normal(0, 2, size=(H, W)), 0, 255).astype(np.uint8)
    return i1, i2, u1.astype(np.int32), u2.astype(np.int32)


# Named configurations of BASELINE.json "configs".
CONFIGS = {
    "C1": dict(W=64, H=48, K=16, d_min=0, iters=5, kind="rd"),
    "C2": dict(W=1242, H=375, K=128, d_min=0, iters=4, kind="wt-kitti"),
    "C3": dict(W=1500, H=1000, K=256, d_min=0, iters=4, kind="wt-middlebury"),
    # configs[3]: optical flow, discrete stage: 32 x 32 label window (u1, u2 in [-16, 15]),
    # decoupled into two K = 32 layers (Eq. flow-decoupled-costs)
    "C4": dict(W=1242, H=375, K=32, d_min=-16, iters=4, kind="flow"),
    # configs[4]: a stream of 64 KITTI-shaped pairs, frames sharded over the GPUs
    "C5": dict(W=1242, H=375, K=128, d_min=0, iters=4, kind="wt-kitti", frames=64),
}


def pair(kind: str, W: int, H: int, K: int, seed: int = 0):
    """Pair of the given kind with disparities inside [0, K-1]."""
    if kind == "rd":
        return random_dot(W, H, K - 1, seed)
    if kind == "wt-kitti":
        return warped_texture(W, H, K - 1, seed, "kitti")
    if kind == "wt-middlebury":
        return warped_texture(W, H, K - 1, seed, "middlebury")
    raise ValueError(kind)
