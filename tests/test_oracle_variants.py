"""Pins for the NEXT-4 variants: alternating sweep directions (reading R21) and
the paper-literal asymmetric v/g beamformer/PSF of Eq. 4 / Eq. 7 (fidelity study of R1)."""
import numpy as np
import pytest

import synth


def _spd(n, seed):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    return M @ M.T / n + 0.5 * np.eye(n), rng


def test_backward_sweep_is_forward_sweep_on_reversed_system(oracle_lib):
    """A backward sweep on (A, b) is a forward sweep on (PAP, Pb), P the reversal: the second
    sweep of the alternating iteration equals forward-on-reversed started from sweep 1."""
    A, rng = _spd(9, 1)
    b = rng.standard_normal(9)
    x2 = oracle_lib.gs(A, b, 2, alt=True)
    # forward sweep 1, then one forward sweep on the reversed system from that start:
    x1 = oracle_lib.gs(A, b, 1)
    P = np.eye(9)[::-1]
    Ar, br = P @ A @ P, P @ b
    xr = P @ x1
    for i in range(9):                                    # one forward sweep (Eq. 13-14) by hand
        xr[i] = max(xr[i] - (Ar[i] @ xr - br[i]) / Ar[i, i], 0.0)
    assert np.max(np.abs(P @ xr - x2)) < 1e-13


def test_alternating_converges_to_the_same_solution(oracle_lib):
    """On an SPD system with a nonnegative solution both iterations reach x* = A^-1 b."""
    A, rng = _spd(12, 2)
    xs = np.abs(rng.standard_normal(12))
    b = A @ xs
    assert np.max(np.abs(oracle_lib.gs(A, b, 400, alt=True) - xs)) < 1e-9
    assert np.max(np.abs(oracle_lib.gs(A, b, 400) - xs)) < 1e-9


def test_alternating_objective_monotone_and_identity(oracle_lib):
    A, rng = _spd(10, 3)
    b = rng.standard_normal(10)
    f = lambda x: 0.5 * x @ A @ x - b @ x
    vals = [f(oracle_lib.gs(A, b, k, alt=True)) for k in range(1, 12)]
    assert all(vals[i + 1] <= vals[i] + 1e-14 for i in range(len(vals) - 1))
    bb = np.array([0.5, -1.0, 2.0])
    assert np.array_equal(oracle_lib.gs(np.eye(3), bb, 3, alt=True), np.maximum(bb, 0))


@pytest.fixture(scope="module")
def geom1():
    cfg = synth.CONFIGS["cfg1"]
    return cfg, cfg.mics()


def _g(cfg, mic):
    return (mic, cfg.c0, cfg.n, cfg.side_len, cfg.z0, cfg.cx, cfg.cy)


def test_paper_psf_unit_diagonal_and_asymmetric(oracle_lib, geom1):
    """Eq. 4 x Eq. 7: conj(v_m) g_m = 1 per microphone, so A_P[r][r] = 1; A_P is not symmetric
    (max |A - A^T| = 0.032 on cfg1), and differs from R1's symmetric PSF by a few %."""
    cfg, mic = geom1
    keep = np.arange(cfg.S, dtype=np.int32)
    AP = oracle_lib.psf_paper(*_g(cfg, mic), 4000.0, keep)
    A1 = oracle_lib.psf(*_g(cfg, mic), 4000.0, keep)
    assert np.max(np.abs(np.diag(AP) - 1.0)) < 1e-14
    asym = np.max(np.abs(AP - AP.T))
    assert 0.01 < asym < 0.1
    rel = np.linalg.norm(AP - A1) / np.linalg.norm(A1)
    assert 0.01 < rel < 0.1


def test_paper_das_of_model_csm_is_paper_psf_column(oracle_lib, geom1):
    """Eq. 9-12 with the paper's own vectors: C = q^2 g g^H (Eq. 8, synth's propagation model)
    gives b_P = q^2 A_P[:, s0] (the identity the paper derives)."""
    cfg, mic = geom1
    s0 = 150
    q2 = 0.8
    src = synth.grid_node_xyz(cfg.n, cfg.side_len, cfg.z0, cfg.cx, cfg.cy, np.array([s0]))
    C = synth.csm_exact(mic, src, np.array([q2]), 4000.0, cfg.c0)
    b = oracle_lib.das_paper(*_g(cfg, mic), 4000.0, C)
    AP = oracle_lib.psf_paper(*_g(cfg, mic), 4000.0, np.arange(cfg.S, dtype=np.int32))
    assert np.max(np.abs(b - q2 * AP[:, s0])) < 1e-12 * q2


def test_paper_mode_end_to_end_recovers_a_single_source(oracle_lib):
    """The paper-literal path end to end (Eq. 4 beamformer, Eq. 7 PSF, Eq. 13-14 sweeps): for the
    paper's own model CSM of one source at node s0, C = q^2 g g^H (Eq. 8), b_P = q^2 A_P[:, s0]
    (Eq. 9-12), so x = q^2 e_s0 is the fixed point of the sweeps.  On a coarse 7x7 grid (dx/B ~
    0.8) the sweeps reach it from x0 = 0; the R1 path on the same CSM returns a different power
    (its x is the array-averaged descriptor, reading R1/R14)."""
    m = 16
    mic = synth.spiral_array(m, 0.5, 1)
    n, L, z0, f = 7, 1.0, 1.0, 4000.0
    s0, q2 = 24, 0.7
    src = synth.grid_node_xyz(n, L, z0, 0.0, 0.0, np.array([s0]))
    C = synth.csm_exact(mic, src, np.array([q2]), f, 343.0)
    keep, x, b = oracle_lib.solve_bin(mic, 343.0, n, L, z0, 0.0, 0.0, f, C, 0.1, 0, 2000, full_grid=True,
                                      paper=True)
    assert len(keep) == n * n
    e = np.zeros(n * n)
    e[s0] = q2
    assert np.max(np.abs(x - e)) < 1e-6 * q2
    _, x1, _ = oracle_lib.solve_bin(mic, 343.0, n, L, z0, 0.0, 0.0, f, C, 0.1, 0, 2000, full_grid=True)
    assert abs(x1.sum() - q2) > 1e-3 * q2
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.solve_bin(mic, 343.0, n, L, z0, 0.0, 0.0, f, C, 0.1, 0, 5, dr=True, paper=True)
