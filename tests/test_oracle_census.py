"""Pins for the oracle's census transform and Hamming cost volume."""
import numpy as np
import pytest

import datagen


def _offsets(r):
    """Raster order of the window offsets, centre skipped (reading R17)."""
    return [(dy, dx) for dy in range(-r, r + 1) for dx in range(-r, r + 1) if (dy, dx) != (0, 0)]


def test_constant_image_zero_codes(orc):
    assert not orc.census(np.full((7, 9), 77, np.uint8)).any()


def test_single_dark_pixel(orc):
    """A dark pixel on a flat background: each neighbour within the window has
    exactly the one bit facing it set; the dark pixel's own code is 0."""
    for r in (1, 2):
        img = np.full((11, 11), 100, np.uint8)
        img[5, 5] = 0
        c = orc.census(img, r)
        offs = _offsets(r)
        assert c[5, 5] == 0
        for y in range(11):
            for x in range(11):
                dy, dx = 5 - y, 5 - x
                if (dy, dx) == (0, 0):
                    continue
                if max(abs(dy), abs(dx)) <= r:
                    assert c[y, x] == 1 << offs.index((dy, dx))
                else:
                    assert c[y, x] == 0


def test_bright_centre_all_bits(orc):
    img = np.zeros((5, 5), np.uint8)
    img[2, 2] = 9
    assert orc.census(img, 2)[2, 2] == (1 << 24) - 1


def test_ramp_left_half(orc):
    """Horizontal ramp I = x: interior codes have exactly the dx < 0 bits set."""
    img = np.tile(np.arange(20, dtype=np.uint8) * 3, (9, 1))
    c = orc.census(img, 2)
    want = sum(1 << b for b, (dy, dx) in enumerate(_offsets(2)) if dx < 0)
    assert np.all(c[:, 2:-2] == want)
    # replicated border: at x = 0 the dx < 0 neighbours equal the centre -> clear
    assert np.all(c[:, 0] == 0)


def test_monotone_map_invariance(orc):
    rng = np.random.default_rng(20)
    img = rng.integers(0, 128, size=(30, 40)).astype(np.uint8)
    lut = (np.arange(128) + np.cumsum(rng.integers(0, 2, size=128))).astype(np.uint8)
    assert np.all(np.diff(lut.astype(int)) > 0)        # strictly increasing
    mapped = lut[img]
    assert np.array_equal(orc.census(img), orc.census(mapped))


def test_cost_identical_images(orc):
    rng = np.random.default_rng(21)
    img = rng.integers(0, 256, size=(12, 20)).astype(np.uint8)
    c = orc.census(img)
    D = orc.cost_volume(c, c, 0, 6, 12)
    assert not D[:, :, 0].any()
    assert D.max() <= 24


def test_cost_shift_argmin(orc):
    """right = left shifted by s px => argmin_k D = s in the interior."""
    rng = np.random.default_rng(22)
    W, H, s = 60, 16, 7
    left = rng.integers(0, 256, size=(H, W)).astype(np.uint8)
    right = np.zeros_like(left)
    right[:, : W - s] = left[:, s:]
    D = orc.cost_volume(orc.census(left), orc.census(right), 0, 16, 12)
    inner = D[2:-2, s + 2 : W - 2 - s]
    assert np.all(inner[:, :, s] == 0)
    # dark centres give near-empty codes, so other zero-cost labels occur rarely
    assert (inner.argmin(2) == s).mean() > 0.95


def test_cost_oob_and_popcount_bounds(orc):
    rng = np.random.default_rng(23)
    cl = rng.integers(0, 1 << 24, size=(4, 10)).astype(np.uint32)
    cr = rng.integers(0, 1 << 24, size=(4, 10)).astype(np.uint32)
    for dmin in (-3, 0, 2):
        D = orc.cost_volume(cl, cr, dmin, 8, 12)
        for x in range(10):
            for k in range(8):
                xr = x - dmin - k
                if 0 <= xr < 10:
                    want = np.array([bin(int(a) ^ int(b)).count("1") for a, b in zip(cl[:, x], cr[:, xr])])
                    assert np.array_equal(D[:, x, k], want)
                else:
                    assert np.all(D[:, x, k] == 12)


def test_cost_swap_symmetry(orc):
    """D_LR(x, d) = D_RL(x - d, -d)."""
    rng = np.random.default_rng(24)
    a = rng.integers(0, 256, size=(8, 30)).astype(np.uint8)
    b = rng.integers(0, 256, size=(8, 30)).astype(np.uint8)
    ca, cb = orc.census(a), orc.census(b)
    Dab = orc.cost_volume(ca, cb, 0, 5, 12)
    Dba = orc.cost_volume(cb, ca, -4, 5, 12)    # disparities -4..0
    for x in range(5, 30):
        for d in range(5):
            assert np.array_equal(Dab[:, x, d], Dba[:, x - d, 4 - d])


def test_bad_radius(orc):
    with pytest.raises(ValueError):
        orc.census(np.zeros((4, 4), np.uint8), 3)


def test_datagen_shapes_and_determinism():
    for kind, W, H, K in [("rd", 64, 48, 16), ("wt-kitti", 200, 80, 32), ("wt-middlebury", 150, 100, 64)]:
        l1, r1, d1 = datagen.pair(kind, W, H, K, 3)
        l2, r2, d2 = datagen.pair(kind, W, H, K, 3)
        assert l1.shape == (H, W) and l1.dtype == np.uint8 and r1.dtype == np.uint8
        assert np.array_equal(l1, l2) and np.array_equal(r1, r2) and np.array_equal(d1, d2)
        assert d1.min() >= 0 and d1.max() <= K - 1
