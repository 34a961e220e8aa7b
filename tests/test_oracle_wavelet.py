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


# ---------------------------------------------------------------------------------------
# NEXT-1: the 4-point (cubic, Deslauriers-Dubuc family)
# interpolating predictor, reading R19.

def _coarse_counts(n, J):
    """Per-axis number of G^j nodes (multiples of 2^(J-j) in [0, n-1])."""
    return [(n - 1) // (1 << (J - j)) + 1 for j in range(J + 1)]


@pytest.mark.parametrize("n", [21, 50, 81, 101])
def test_cubic_reproduces_bicubic_maps(oracle_lib, n):
    """4-point Lagrange interpolation is exact for cubics: details vanish exactly at every
    level whose coarse lattice has >= 4 nodes per axis (integer bicubic map: all values,
    weights k/16 and partial sums are exact in fp64).  Bilinear maps vanish everywhere
    (the linear fallback of the coarsest levels is exact for them too)."""
    J = oracle_lib.max_level(n)
    r, c = np.meshgrid(np.arange(n, dtype=float), np.arange(n, dtype=float), indexing="ij")
    b = (2 * c ** 3 - 3 * c ** 2 + c - 7) * (r ** 3 + 5 * r - 2)
    d, lv = oracle_lib.wavelet_details(n, b.ravel(), order=3)
    cnt = _coarse_counts(n, J)
    full = [l for l in range(1, J + 1) if cnt[l - 1] >= 4]
    assert full, "test grid too small"
    for l in full:
        assert np.all(d[lv == l] == 0.0), (n, l)
    lo = [l for l in range(1, J + 1) if cnt[l - 1] < 4]
    assert any(np.any(d[lv == l] != 0.0) for l in lo)   # the linear fallback is not exact for cubics
    bl = 7.0 + 3.0 * r - 5.0 * c + 2.0 * r * c
    d2, _ = oracle_lib.wavelet_details(n, bl.ravel(), order=3)
    assert np.all(d2 == 0.0)


def _lagrange_1d(f, i, h, n):
    """Independent route: numpy.polyfit through the 4 nearest coarse nodes (the node choice
    is reading R19; the weights come from the library fit), or None when fewer than 4."""
    cand = [i + k * h for k in (-7, -5, -3, -1, 1, 3, 5, 7) if 0 <= i + k * h <= n - 1]
    if len(cand) < 4:
        return None
    near = sorted(sorted(cand, key=lambda p: (abs(p - i), p))[:4])
    # R19 prefers the symmetric set, then the set shifted away from the nearer boundary
    xs = np.array(near, dtype=float) - i
    return lambda vals: np.polyval(np.polyfit(xs, vals, 3), 0.0), near


@pytest.mark.parametrize("n", [13, 21, 40])
def test_cubic_details_match_polyfit(oracle_lib, n):
    """On random maps the cubic details equal b - (tensor 4-point polynomial fit: rows
    first, then the column) to 1e-9, at every node where both axes have 4 coarse nodes."""
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    d, lv = oracle_lib.wavelet_details(n, b.ravel(), order=3)
    d = d.reshape(n, n)
    lv = lv.reshape(n, n)
    J = oracle_lib.max_level(n)
    checked = 0
    for r in range(n):
        for c in range(n):
            l = int(lv[r, c])
            if l == 0:
                continue
            h = 1 << (J - l)
            on_r, on_c = r % (2 * h) == 0, c % (2 * h) == 0
            fr = None if on_r else _lagrange_1d(None, r, h, n)
            fc = None if on_c else _lagrange_1d(None, c, h, n)
            if (not on_r and fr is None) or (not on_c and fc is None):
                continue
            rows = [r] if on_r else fr[1]
            cols = [c] if on_c else fc[1]
            t = [b[rr, c] if on_c else fc[0](b[rr, cols]) for rr in rows]
            pred = t[0] if on_r else fr[0](np.array(t))
            assert abs(d[r, c] - (b[r, c] - pred)) < 1e-9, (n, r, c)
            checked += 1
    assert checked > n * n // 4


def test_cubic_edge_weights_closed_form(oracle_lib):
    """One-sided 4-point weights (R19) at each edge of a 1-D-varying map: a single unit
    spike at coarse node p gives detail -w_p at the fine node (Lagrange basis values)."""
    n = 21   # J = 4; finest level h = 1, coarse stride 2
    cases = {  # fine node i -> {coarse node: weight}
        1: {0: 5 / 16, 2: 15 / 16, 4: -5 / 16, 6: 1 / 16},        # left edge {-1,1,3,5}
        9: {6: -1 / 16, 8: 9 / 16, 10: 9 / 16, 12: -1 / 16},      # interior
        19: {14: 1 / 16, 16: -5 / 16, 18: 15 / 16, 20: 5 / 16},   # right edge {-5,-3,-1,1}
    }
    for i, wts in cases.items():
        for p, w in wts.items():
            b = np.zeros((n, n))
            b[:, p] = 1.0                       # constant along rows: the row rule is exact
            d, _ = oracle_lib.wavelet_details(n, b.ravel(), order=3)
            assert d.reshape(n, n)[0, i] == -w, (i, p)
    # extrapolation past the last coarse node {-7,-5,-3,-1}: N = 20 -> node 19 (h = 1)
    n = 20
    for p, w in {12: -5 / 16, 14: 21 / 16, 16: -35 / 16, 18: 35 / 16}.items():
        b = np.zeros((n, n))
        b[:, p] = 1.0
        d, _ = oracle_lib.wavelet_details(n, b.ravel(), order=3)
        assert d.reshape(n, n)[0, 19] == -w, p


def test_cubic_keeps_fewer_points_on_smooth_maps(oracle_lib):
    """The point of a higher-order predictor: on a smooth beam-like map
    the cubic details are smaller, so the same relative eps keeps fewer nodes."""
    n = 81
    y, x = np.meshgrid(np.linspace(-1, 1, n), np.linspace(-1, 1, n), indexing="ij")
    b = np.exp(-((x - 0.2) ** 2 + y ** 2) / 0.08) + 0.5 * np.exp(-((x + 0.3) ** 2 + (y - 0.1) ** 2) / 0.05)
    k1, *_ = oracle_lib.compress(n, b.ravel(), 0.005, order=1)
    k3, *_ = oracle_lib.compress(n, b.ravel(), 0.005, order=3)
    assert len(k3) < len(k1)
    g0 = np.flatnonzero(oracle_lib.wavelet_details(n, b.ravel(), order=3)[1] == 0)
    assert set(g0) <= set(k3)
