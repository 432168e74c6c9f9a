"""Pins for the oracle's optimistic decoupled flow costs (Eq. flow-decoupled-
costs; NEXT-1 of SURVEY 8(f)).

None of these re-types the oracle's formula: they check what the definition
fixes -- exact translations give a zero cost at the true displacement, the
two layers share their minimum (both are the minimum of the same 2-D window),
and one-row / one-column windows reduce to the stereo cost volume (pinned
separately in test_oracle_census.py) on the original / transposed codes."""
import numpy as np
import pytest


def _codes(orc, img):
    return orc.census(img, 2)


def test_flow_exact_translation_zero_cost(orc):
    """I2(x + s1, y + s2) = I1(x, y) exactly: every pixel whose census windows
    are inside both images has f1 = 0 at u1 = s1 and f2 = 0 at u2 = s2."""
    rng = np.random.default_rng(0)
    big = rng.integers(0, 256, size=(60, 80)).astype(np.uint8)
    for s1, s2 in ((3, -2), (-5, 4), (0, 0), (7, 7)):
        H, W = 30, 40
        y0, x0 = 15, 20
        i1 = big[y0:y0 + H, x0:x0 + W]
        i2 = big[y0 - s2:y0 - s2 + H, x0 - s1:x0 - s1 + W]   # i2[y + s2, x + s1] = i1[y, x]
        c1, c2 = _codes(orc, i1), _codes(orc, i2)
        f1, f2 = orc.flow_costs(c1, c2, -8, 16, -8, 16)
        ys, xs = np.mgrid[0:H, 0:W]
        inside = (ys >= 2) & (ys < H - 2) & (xs >= 2) & (xs < W - 2)
        inside &= (ys + s2 >= 2) & (ys + s2 < H - 2) & (xs + s1 >= 2) & (xs + s1 < W - 2)
        assert inside.sum() > 100
        assert np.all(f1[inside][:, s1 + 8] == 0)
        assert np.all(f2[inside][:, s2 + 8] == 0)


def test_flow_layers_share_the_window_minimum(orc):
    rng = np.random.default_rng(1)
    i1 = rng.integers(0, 256, size=(21, 33)).astype(np.uint8)
    i2 = rng.integers(0, 256, size=(21, 33)).astype(np.uint8)
    f1, f2 = orc.flow_costs(_codes(orc, i1), _codes(orc, i2), -5, 11, -3, 7, oob=12)
    assert np.array_equal(f1.min(axis=2), f2.min(axis=2))
    assert f1.max() <= 24 and f2.max() <= 24


def test_flow_one_row_window_is_stereo(orc):
    """K2 = 1, u2 = 0: f1[a] = D_stereo[K1-1-a] with d_min = -(u1_min + K1 - 1)
    (stereo matches x - d, flow x + u1)."""
    rng = np.random.default_rng(2)
    i1 = rng.integers(0, 256, size=(17, 45)).astype(np.uint8)
    i2 = rng.integers(0, 256, size=(17, 45)).astype(np.uint8)
    c1, c2 = _codes(orc, i1), _codes(orc, i2)
    for u1_min, K1 in ((-6, 13), (0, 9), (-20, 40)):
        f1, f2 = orc.flow_costs(c1, c2, u1_min, K1, 0, 1, oob=12)
        D = orc.cost_volume(c1, c2, -(u1_min + K1 - 1), K1, 12)
        assert np.array_equal(f1, D[:, :, ::-1])
        assert np.array_equal(f2[:, :, 0], D.min(axis=2))


def test_flow_one_column_window_is_transposed_stereo(orc):
    """K1 = 1, u1 = 0: f2 is the stereo cost volume of the transposed codes."""
    rng = np.random.default_rng(3)
    i1 = rng.integers(0, 256, size=(29, 23)).astype(np.uint8)
    i2 = rng.integers(0, 256, size=(29, 23)).astype(np.uint8)
    c1, c2 = _codes(orc, i1), _codes(orc, i2)
    u2_min, K2 = -7, 15
    f1, f2 = orc.flow_costs(c1, c2, 0, 1, u2_min, K2, oob=9)
    Dt = orc.cost_volume(c1.T.copy(), c2.T.copy(), -(u2_min + K2 - 1), K2, 9)
    assert np.array_equal(f2, Dt.transpose(1, 0, 2)[:, :, ::-1])


def test_flow_window_outside_image_is_oob(orc):
    rng = np.random.default_rng(4)
    i1 = rng.integers(0, 256, size=(8, 8)).astype(np.uint8)
    c = _codes(orc, i1)
    f1, f2 = orc.flow_costs(c, c, 100, 4, 0, 3, oob=17)
    assert np.all(f1 == 17) and np.all(f2 == 17)


def test_flow_bad_arguments(orc):
    c = np.zeros((4, 4), np.uint32)
    with pytest.raises(ValueError):
        orc.flow_costs(c, c, 0, 0, 0, 4)
