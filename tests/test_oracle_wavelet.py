"""Pins for the oracle's S3/S4 wavelet compression (Alg. 1, Eq. 15-22)."""
import math
import os

import numpy as np
import pytest
from scipy.interpolate import RegularGridInterpolator

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load_grid(name):
    rows = [l.split() for l in open(os.path.join(GOLD, name)) if l.strip() and not l.startswith("#")]
    return np.array(rows, dtype=float)


def test_level_sizes_and_counts(oracle_lib):
    """Nested grid sizes per axis (Eq. 15) and points first appearing at
    each level (closed form n_j^2 - n_{j-1}^2), fixture tests/golden/wavelet_levels.txt."""
    for line in open(os.path.join(GOLD, "wavelet_levels.txt")):
        if line.startswith("#") or not line.strip():
            continue
        n_s, sizes_s, counts_s = line.split(":")
        n = int(n_s)
        sizes = [int(v) for v in sizes_s.split()]
        counts = [int(v) for v in counts_s.split()]
        J = oracle_lib.max_level(n)
        assert J == int(math.floor(math.log2(n))) == len(sizes) - 1
        _, lv = oracle_lib.wavelet_details(n, np.zeros(n * n))
        lv = lv.reshape(n, n)
        got_counts = [int(np.sum(lv == j)) for j in range(J + 1)]
        assert got_counts == counts, (n, got_counts, counts)
        for j in range(J + 1):   # per-axis size of G^j: rows with any level<=j point in column 0
            assert int(np.sum(lv[:, 0] <= j)) == sizes[j]
            assert int(np.sum(lv[0, :] <= j)) == sizes[j]


def test_hand_derived_6x6(oracle_lib):
    """Details of b = c^2 on a 6x6 grid derived by hand (fixture with derivation)."""
    n = 6
    c = np.arange(n, dtype=float)
    b = np.tile(c * c, (n, 1))
    d, lv = oracle_lib.wavelet_details(n, b.ravel())
    assert np.array_equal(d.reshape(n, n), _load_grid("wavelet_6x6_colquad.txt"))
    assert np.array_equal(lv.reshape(n, n), _load_grid("wavelet_6x6_levels.txt"))


@pytest.mark.parametrize("n", [3, 6, 9, 21, 50, 101])
def test_bilinear_ramp_has_zero_details(oracle_lib, n):
    """Linear interpolation (incl. the one-sided right-edge extrapolation) reproduces
    (bi)linear maps exactly when N != 2^J (R7); integer coefficients keep it exact."""
    r, c = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    b = 7.0 + 3.0 * r - 5.0 * c + 2.0 * r * c
    d, _ = oracle_lib.wavelet_details(n, b.ravel())
    assert np.all(d == 0.0)


@pytest.mark.parametrize("n", [9, 21, 37])
def test_details_match_scipy_bilinear(oracle_lib, n):
    """Eq. 22: d = b - (interpolation from the adjacent coarser level).  scipy's
    RegularGridInterpolator(method='linear', fill_value=None) on the level-(j-1) lattice is
    the tensor-product linear interpolant with linear extrapolation past the last coarse node,
    i.e. R7's stencil for N != 2^J.  Compare on random maps, level by level."""
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    d, lv = oracle_lib.wavelet_details(n, b.ravel())
    d = d.reshape(n, n)
    lv = lv.reshape(n, n)
    J = oracle_lib.max_level(n)
    for j in range(1, J + 1):
        H = 2 ** (J - j + 1)          # stride of the coarse level j-1
        coarse = np.arange(0, n, H)
        itp = RegularGridInterpolator((coarse, coarse), b[np.ix_(coarse, coarse)], method="linear",
                                      bounds_error=False, fill_value=None)
        rr, cc = np.nonzero(lv == j)
        ref = b[rr, cc] - itp(np.stack([rr, cc], axis=1).astype(float))
        assert np.max(np.abs(d[rr, cc] - ref)) < 1e-12, j


def test_constant_map_keeps_coarsest_only(oracle_lib):
    """Constant map => all details vanish => keep = G^0; sigma = S/|G^0|."""
    for n in [21, 81, 101]:
        keep, lv, d, ee = oracle_lib.compress(n, np.full(n * n, 3.25), 0.01)
        assert np.array_equal(keep, np.flatnonzero(lv == 0))
        assert len(keep) == 4


def test_monotone_and_bounds(oracle_lib):
    """eps1 < eps2 => keep(eps1) superset of keep(eps2); G^0 subset of keep;
    1 <= sigma <= S/|G^0|; Table 2 trend: sigma increasing in eps
    (PAPER.md:518-520)."""
    n = 41
    rng = np.random.default_rng(3)
    r, c = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    b = np.exp(-((r - 12.3) ** 2 + (c - 20.1) ** 2) / 30.0) + 0.4 * np.exp(-((r - 30) ** 2 + (c - 8) ** 2) / 8.0)
    b = b.ravel() + 1e-3 * rng.random(n * n)
    prev = None
    sigmas = []
    for eps in [0.2, 0.1, 0.05, 0.01, 0.001]:
        keep, lv, d, ee = oracle_lib.compress(n, b, eps)
        ks = set(keep.tolist())
        assert set(np.flatnonzero(lv == 0).tolist()) <= ks
        if prev is not None:
            assert prev <= ks
        prev = ks
        sigmas.append(n * n / len(keep))
        assert 1 <= sigmas[-1] <= n * n / 4
        assert np.all(np.diff(keep) > 0)
    assert all(a > b_ for a, b_ in zip(sigmas, sigmas[1:]))


def test_threshold_tie_is_kept_and_absolute_mode(oracle_lib):
    """R5: keep iff |d| >= eps_eff (Alg. 1 line 7, ties kept); absolute mode uses eps as is."""
    n = 6
    c = np.arange(n, dtype=float)
    b = np.tile(c * c, (n, 1)).ravel()       # details -4, -1, 3 (hand-derived fixture)
    keep, lv, d, ee = oracle_lib.compress(n, b, 3.0, eps_mode=1)
    assert ee == 3.0
    kept = set(keep.tolist())
    assert kept == set(np.flatnonzero((lv == 0) | (np.abs(d) >= 3.0)).tolist())
    assert 5 in kept and 2 in kept and 1 not in kept
    # relative: eps_eff = eps * max|b| = (3/25) * 25 = 3.0 exactly
    keep2, _, _, ee2 = oracle_lib.compress(n, b, 3.0 / 25.0, eps_mode=0)
    assert abs(ee2 - 3.0) < 1e-15


def test_degenerate_zero_map_relative(oracle_lib):
    """R6: max|b| = 0 in relative mode keeps G^0 only (not the whole grid)."""
    keep, lv, _, _ = oracle_lib.compress(21, np.zeros(441), 0.1)
    assert len(keep) == 4 and np.all(lv[keep] == 0)


def test_full_grid_and_tiny_eps(oracle_lib):
    """Full-grid mode keeps everything; eps -> 0+ keeps every point with d != 0."""
    n = 9
    b = np.random.default_rng(1).random(n * n)
    keep, *_ = oracle_lib.compress(n, b, 0.5, full_grid=True)
    assert np.array_equal(keep, np.arange(n * n))
    keep, *_ = oracle_lib.compress(n, b, 1e-300)
    assert len(keep) == n * n


def test_eq19_error_bound(oracle_lib):
    """Eq. 19: reconstructing a smooth map from the kept points by the
    interpolation cascade (discarded details set to 0) errs by at most C*eps_eff, C ~ 1
    (SPEC.md:375 uses C = 10).  Cascaded reading only here (R8)."""
    n = 33
    r, c = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    b = (np.exp(-((r - 10) ** 2 + (c - 14) ** 2) / 40.0) + 0.5 * np.exp(-((r - 25) ** 2 + (c - 24) ** 2) / 15.0)
         + 0.2 * np.exp(-((r - 5) ** 2 + (c - 28) ** 2) / 90.0))
    for eps in [0.1, 0.03, 0.01]:
        keep, lv, d, ee = oracle_lib.compress(n, b.ravel(), eps)
        lv = lv.reshape(n, n)
        kept = np.zeros(n * n, bool)
        kept[keep] = True
        kept = kept.reshape(n, n)
        J = oracle_lib.max_level(n)
        rec = np.where(lv == 0, b, 0.0)
        for j in range(1, J + 1):
            H = 2 ** (J - j + 1)
            coarse = np.arange(0, n, H)
            itp = RegularGridInterpolator((coarse, coarse), rec[np.ix_(coarse, coarse)], method="linear",
                                          bounds_error=False, fill_value=None)
            rr, cc = np.nonzero(lv == j)
            pred = itp(np.stack([rr, cc], axis=1).astype(float))
            rec[rr, cc] = np.where(kept[rr, cc], b[rr, cc], pred)
        assert np.max(np.abs(rec - b)) <= 10 * ee
