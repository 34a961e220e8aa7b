"""Pins for the oracle's S7 Gauss-Seidel (Eq. 13-14) and the S0..S8 pipeline."""
import math

import numpy as np
import pytest

import synth


def test_gs_identity_and_scalar(oracle_lib):
    """A = I => x = max(b, 0) after one sweep; 1x1 => max(b/A11, 0)."""
    b = np.array([0.5, -1.0, 2.0, 0.0])
    assert np.array_equal(oracle_lib.gs(np.eye(4), b, 1), np.maximum(b, 0))
    assert oracle_lib.gs(np.array([[4.0]]), np.array([3.0]), 1)[0] == 0.75
    assert oracle_lib.gs(np.array([[4.0]]), np.array([-3.0]), 5)[0] == 0.0


def test_gs_2x2_by_hand(oracle_lib):
    """Eq. 13-14 by hand, A = [[2,1],[1,3]], b = [1,2], x0 = 0:
    sweep 1: x1 = 0 - (0 - 1)/2 = 0.5; x2 = 0 - (0.5 + 0 - 2)/3 = 0.5
    sweep 2: r1 = 1 + 0.5 - 1 = 0.5 -> x1 = 0.25; r2 = 0.25 + 1.5 - 2 = -0.25 -> x2 = 7/12."""
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    b = np.array([1.0, 2.0])
    assert np.allclose(oracle_lib.gs(A, b, 1), [0.5, 0.5], atol=1e-15)
    assert np.allclose(oracle_lib.gs(A, b, 2), [0.25, 7.0 / 12.0], atol=1e-15)
    assert np.allclose(oracle_lib.gs(A, b, 200), np.linalg.solve(A, b), atol=1e-13)


def test_gs_projection_active(oracle_lib):
    """Positivity: with A = [[1,0.9],[0.9,1]], b = [1, 0.1] the
    unconstrained solution has x2 < 0; the NNLS-type fixed point is x = (1, 0)."""
    A = np.array([[1.0, 0.9], [0.9, 1.0]])
    b = np.array([1.0, 0.1])
    x = oracle_lib.gs(A, b, 100)
    assert np.allclose(x, [1.0, 0.0], atol=1e-14)


def _pd_system(seed=0):
    """7x7 grid (49 pts), M=16, 4 kHz: dx/B ~ 0.8, A~ positive definite."""
    mic = synth.spiral_array(16, 0.5, 1)
    n, L, z0, f = 7, 1.0, 1.0, 4000.0
    return mic, n, L, z0, f


def test_gs_recovers_exact_sparse_solution(oracle_lib):
    """Brute force on a 49-point grid (north_star): b = A x_true with sparse x_true >= 0;
    numpy's dense solve returns x_true, and GS reaches it; objective 1/2 x'Ax - b'x is
    non-increasing sweep by sweep; x >= 0 throughout."""
    mic, n, L, z0, f = _pd_system()
    A = oracle_lib.psf(mic, 343.0, n, L, z0, 0, 0, f, np.arange(n * n))
    assert np.linalg.eigvalsh(A).min() > 0
    x_true = np.zeros(n * n)
    x_true[[3, 24, 30, 44]] = [1.0, 0.5, 0.25, 0.8]
    b = A @ x_true
    assert np.allclose(np.linalg.solve(A, b), x_true, atol=1e-8)
    obj_prev = 0.0
    for sw in [1, 2, 3, 5, 10, 20]:
        x = oracle_lib.gs(A, b, sw)
        assert x.min() >= 0
        obj = 0.5 * x @ A @ x - b @ x
        assert obj <= obj_prev + 1e-12
        obj_prev = obj
    x = oracle_lib.gs(A, b, 1000)
    assert np.max(np.abs(x - x_true)) < 1e-6


def test_gs_fixed_point(oracle_lib):
    """A fixed point x* >= 0 with A x* = b is unchanged by further sweeps."""
    mic, n, L, z0, f = _pd_system()
    A = oracle_lib.psf(mic, 343.0, n, L, z0, 0, 0, f, np.arange(n * n))
    x_true = np.zeros(n * n)
    x_true[[10, 11]] = [1.0, 2.0]
    b = A @ x_true
    x1 = oracle_lib.gs(A, b, 3000)
    x2 = oracle_lib.gs(A, b, 3001)
    assert np.max(np.abs(x2 - x1)) < 1e-12


def test_single_exact_source_recovered_at_its_node(oracle_lib):
    """north_star pin: a single exact-CSM source is recovered at its grid point, with the
    power descriptor x_s0 = q^2 ||g^P_s0||^2 / M (R1) on a PD 49-point grid."""
    mic, n, L, z0, f = _pd_system()
    s0 = 17
    src = synth.grid_node_xyz(n, L, z0, 0, 0, [s0])
    C = synth.csm_exact(mic, src, np.array([1.0]), f, 343.0)
    keep, x, b = oracle_lib.solve_bin(mic, 343.0, n, L, z0, 0, 0, f, C, 0.5, 0, 1000, full_grid=True)
    gp = synth.propagation_vectors(mic, src, f, 343.0)[:, 0]
    x0 = np.sum(np.abs(gp) ** 2) / 16
    assert np.argmax(x) == s0
    assert abs(x[s0] - x0) < 1e-6 * x0
    assert np.sum(np.abs(x)) - x[s0] < 1e-6


def test_gs_kkt_on_singular_grid(oracle_lib):
    """Larger grid, rank A <= M^2 < S: no unique solution, but after many
    sweeps the KKT conditions of min 1/2 x'Ax - b'x, x >= 0 hold."""
    mic = synth.spiral_array(4, 0.5, 1)
    n = 9
    A = oracle_lib.psf(mic, 343.0, n, 1.0, 1.0, 0, 0, 3000.0, np.arange(n * n))
    x_true = np.zeros(n * n)
    x_true[[20, 50]] = [1.0, 0.5]
    b = A @ x_true
    x = oracle_lib.gs(A, b, 5000)
    g = A @ x - b
    tol = 1e-6 * np.max(b)
    assert x.min() >= 0
    assert np.all(g[x == 0] >= -tol)
    assert np.all(np.abs(g[x > 0]) <= tol)


def test_gs_errors(oracle_lib):
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.gs(np.array([[0.0]]), np.array([1.0]), 1)      # A_ii <= 0
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.gs(np.eye(2), np.array([1.0, 1.0]), 0)        # sweeps < 1


def test_pipeline_cfg1(oracle_lib):
    """cfg1 (BASELINE configs[0]): two unit sources at (+-0.2, 0) m.  The compressed-grid
    DAMAS map peaks at the two source nodes, the keep set contains them and G^0, and the
    band driver equals the per-bin driver (threads do not change results)."""
    band = synth.make_band("cfg1")
    cfg = band.cfg
    nk, keep, x, b = oracle_lib.solve_band_cfg(band, n_threads=2)
    k1, x1, b1 = oracle_lib.solve_bin(band.mic_xyz, cfg.c0, cfg.n, cfg.side_len, cfg.z0, 0, 0,
                                      band.freqs[0], band.csm[0], cfg.epsilon, 0, cfg.sweeps)
    assert np.array_equal(keep[0, : nk[0]], k1) and np.array_equal(x[0], x1) and np.array_equal(b[0], b1)
    top2 = set(np.argsort(x[0])[::-1][:2].tolist())
    assert top2 == set(band.src_idx.tolist())
    assert set(band.src_idx.tolist()) <= set(k1.tolist())
    assert np.all(keep[0, nk[0]:] == -1)
    # total recovered power within 10% of the descriptors' sum (q^2 ||g||^2/M ~ 1)
    src = synth.grid_node_xyz(cfg.n, cfg.side_len, cfg.z0, 0, 0, band.src_idx)
    gp = synth.propagation_vectors(band.mic_xyz, src, band.freqs[0], cfg.c0)
    p0 = np.sum(band.src_pow * np.sum(np.abs(gp) ** 2, axis=0) / cfg.m)
    assert abs(x[0].sum() - p0) < 0.1 * p0


def test_pipeline_sigma_monotone_in_eps(oracle_lib):
    """Table 2 trend: sigma strictly increasing in eps."""
    band = synth.make_band("cfg1")
    cfg = band.cfg
    sig = []
    for eps in [0.01, 0.05, 0.1, 0.2]:
        nk, *_ = oracle_lib.solve_band_cfg(band, eps=eps, sweeps=1)
        sig.append(cfg.S / nk[0])
    assert all(a < b for a, b in zip(sig, sig[1:])), sig


def test_pipeline_deterministic(oracle_lib):
    band = synth.make_band("cfg2", bins=[0, 5])
    r1 = oracle_lib.solve_band_cfg(band, sweeps=20, n_threads=2)
    r2 = oracle_lib.solve_band_cfg(band, sweeps=20, n_threads=1)
    for a, b in zip(r1, r2):
        assert np.array_equal(a, b)


def test_config_eps_match_oracle_calibration():
    """The configs' relative eps are the oracle-calibrated values (scripts/calibrate_eps.py)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "eps_calibration.txt")
    for line in open(path):
        if line.startswith("#"):
            continue
        name, eps, fr, nb = [v.strip() for v in line.split(":")]
        assert synth.CONFIGS[name].epsilon == float(eps)
