"""Pins for the oracle's S2 DAS map (Eq. 2) and S5 PSF matrix (Eq. 9-12, 23)."""
import math

import numpy as np
import pytest

import synth


@pytest.fixture(scope="module")
def geom():
    mic = synth.spiral_array(24, 0.8, 3)
    return dict(mic=mic, c0=343.0, n=11, L=1.0, z0=1.0, cx=0.0, cy=0.0)


def _args(g):
    return (g["mic"], g["c0"], g["n"], g["L"], g["z0"], g["cx"], g["cy"])


def _nodes(g, idx=None):
    return synth.grid_node_xyz(g["n"], g["L"], g["z0"], g["cx"], g["cy"], idx)


def test_das_unit_source_is_psf_column(oracle_lib, geom):
    """Eq. 9-12: for the exact CSM of one source of strength q^2 at s0
    (Eq. 8, built by the scene generator from the paper's Eq. 7 vector g^P) the DAS map is
    b = A[:, s0] * x_s0 with x_s0 = q^2 ||g^P_s0||^2 / M (reading R1)."""
    g = geom
    f = 2500.0
    s0 = 37
    q2 = 0.7
    C = synth.csm_exact(g["mic"], _nodes(g, [s0]), np.array([q2]), f, g["c0"])
    b = oracle_lib.das(*_args(g), f, C)
    A = oracle_lib.psf(*_args(g), f, np.arange(g["n"] ** 2))
    gp = synth.propagation_vectors(g["mic"], _nodes(g, [s0]), f, g["c0"])[:, 0]
    x0 = q2 * np.sum(np.abs(gp) ** 2) / g["mic"].shape[0]
    assert np.max(np.abs(b - A[:, s0] * x0)) < 1e-12 * x0
    assert np.argmax(b) == s0


def test_das_two_sources_is_b_equals_Ax(oracle_lib, geom):
    """b = A x (Eq. 12) for an incoherent two-source exact CSM."""
    g = geom
    f = 4100.0
    idx = np.array([12, 90])
    q2 = np.array([1.0, 0.316])
    C = synth.csm_exact(g["mic"], _nodes(g, idx), q2, f, g["c0"])
    b = oracle_lib.das(*_args(g), f, C)
    A = oracle_lib.psf(*_args(g), f, np.arange(g["n"] ** 2))
    gp = synth.propagation_vectors(g["mic"], _nodes(g, idx), f, g["c0"])
    x = np.zeros(g["n"] ** 2)
    x[idx] = q2 * np.sum(np.abs(gp) ** 2, axis=0) / g["mic"].shape[0]
    assert np.max(np.abs(b - A @ x)) < 1e-12 * np.max(b)


def test_das_linear_zero_nonnegative(oracle_lib, geom):
    """C = 0 => b = 0; b is linear in C; b >= 0 for PSD C."""
    g = geom
    rng = np.random.default_rng(5)
    M = g["mic"].shape[0]
    f = 3300.0
    assert np.all(oracle_lib.das(*_args(g), f, np.zeros((M, M), complex)) == 0)
    C1 = synth.random_hermitian_psd(M, 6, rng)
    C2 = synth.random_hermitian_psd(M, 3, rng)
    b1 = oracle_lib.das(*_args(g), f, C1)
    b2 = oracle_lib.das(*_args(g), f, C2)
    b12 = oracle_lib.das(*_args(g), f, 2.5 * C1 + C2)
    assert np.max(np.abs(b12 - (2.5 * b1 + b2))) < 1e-12 * np.max(np.abs(b12))
    assert np.min(b1) >= 0 and np.min(b2) >= 0


def test_das_matches_eq2_with_paper_vector(oracle_lib, geom):
    """Eq. 2 evaluated independently with numpy from the paper's Eq. 7 vector g^P
    (different amplitude convention, normalised per column): b = Re(g^H C g) / (M ||g||^2)."""
    g = geom
    rng = np.random.default_rng(11)
    M = g["mic"].shape[0]
    f = 6000.0
    C = synth.random_hermitian_psd(M, 5, rng) + 0.1 * np.eye(M)
    b = oracle_lib.das(*_args(g), f, C)
    gp = synth.propagation_vectors(g["mic"], _nodes(g), f, g["c0"])
    ref = np.real(np.einsum("ms,mn,ns->s", gp.conj(), C, gp)) / (M * np.sum(np.abs(gp) ** 2, axis=0))
    assert np.max(np.abs(b - ref)) < 1e-12 * np.max(np.abs(ref))


def test_psf_invariants(oracle_lib, geom):
    """A_ii = 1, A = A^T, 0 <= A <= 1, A PSD (Schur product of Gram matrices),
    rank <= M^2 (north_star)."""
    g = geom
    f = 3700.0
    keep = np.arange(0, g["n"] ** 2, 2)
    A = oracle_lib.psf(*_args(g), f, keep)
    assert np.max(np.abs(np.diag(A) - 1.0)) < 1e-12
    assert np.max(np.abs(A - A.T)) < 1e-15
    assert A.min() >= 0 and A.max() <= 1 + 1e-12
    w = np.linalg.eigvalsh(A)
    assert w.min() > -1e-12


def test_psf_rank_and_single_mic(oracle_lib):
    """M = 1 => A all ones (no resolution); rank A <= M^2."""
    mic1 = np.array([[0.1, 0.2, 0.0]])
    A1 = oracle_lib.psf(mic1, 343.0, 6, 1.0, 1.0, 0, 0, 2000.0, np.arange(36))
    assert np.max(np.abs(A1 - 1.0)) < 1e-12
    mic = synth.spiral_array(4, 0.5, 1)
    A = oracle_lib.psf(mic, 343.0, 7, 1.0, 1.0, 0, 0, 3000.0, np.arange(49))
    assert np.linalg.matrix_rank(A, tol=1e-9) <= 16


def test_psf_restriction_is_submatrix(oracle_lib, geom):
    """Eq. 23: A~ = A[keep, keep]."""
    g = geom
    f = 5100.0
    full = oracle_lib.psf(*_args(g), f, np.arange(g["n"] ** 2))
    keep = np.array([3, 17, 18, 60, 119, 120])
    sub = oracle_lib.psf(*_args(g), f, keep)
    assert np.array_equal(sub, full[np.ix_(keep, keep)])


# ---------------------------------------------------------------------------- NEXT-2: diagonal removal
def test_dr_removes_uncorrelated_noise_exactly(oracle_lib, geom):
    """Diagonal removal (reading R20) drops the uncorrelated microphone noise of
    the CSM: the map of C + sigma^2 I equals the map of C; a pure noise CSM maps to 0."""
    g = geom
    f = 3100.0
    M = g["mic"].shape[0]
    C = synth.csm_exact(g["mic"], _nodes(g, [20, 77]), np.array([1.0, 0.3]), f, g["c0"])
    noisy = C + 0.8 * np.eye(M)
    b0 = oracle_lib.das(*_args(g), f, C, dr=True)
    b1 = oracle_lib.das(*_args(g), f, noisy, dr=True)
    assert np.max(np.abs(b1 - b0)) <= 1e-13 * np.max(b0)
    assert np.all(oracle_lib.das(*_args(g), f, 2.5 * np.eye(M), dr=True) == 0.0)
    assert np.any(oracle_lib.das(*_args(g), f, 2.5 * np.eye(M)) > 0.0)   # not without DR


def test_dr_single_source_is_dr_psf_column(oracle_lib, geom):
    """b = A_DR x for the exact single-source CSM (Eq. 9-12 with the diagonal removed):
    b_r = x (|e_r^H e_s|^2 - sum_q |e_qr|^2 |e_qs|^2) / (M^2 - M), clamped at 0 on both
    sides (clamp(x a) = x clamp(a) for x > 0).  The exact CSM is built from the normalised
    steering vector of s0 (oracle.steering), x = 1.7."""
    g = geom
    f = 2800.0
    s0 = 64
    x = 1.7
    e = oracle_lib.steering(*_args(g), f, np.array([s0], dtype=np.int32))[0]
    C = x * np.outer(e, e.conj())
    b = oracle_lib.das(*_args(g), f, C, dr=True)
    A = oracle_lib.psf(*_args(g), f, np.arange(g["n"] ** 2), dr=True)
    assert np.max(np.abs(b - x * A[:, s0])) <= 1e-12 * x
    assert np.argmax(b) == s0


def test_dr_psf_closed_forms(oracle_lib, geom):
    """A_DR diagonal = (M^2 - sum_q |e_q|^4) / (M^2 - M) (closed form from the steering
    vectors); symmetric; entries in [0, 1.0x] (clamped); equals the plain PSF minus the
    fourth-moment term where the plain entry is large."""
    g = geom
    f = 4200.0
    keep = np.arange(0, g["n"] ** 2, 3, dtype=np.int32)
    M = g["mic"].shape[0]
    A = oracle_lib.psf(*_args(g), f, keep, dr=True)
    A0 = oracle_lib.psf(*_args(g), f, keep)
    E = oracle_lib.steering(*_args(g), f, keep)
    w = np.abs(E) ** 2                                     # [nk, M]
    diag = (M * M - np.sum(w ** 2, axis=1)) / (M * M - M)
    assert np.max(np.abs(np.diag(A) - diag)) < 1e-12
    assert np.array_equal(A, A.T)
    assert A.min() >= 0.0
    ref = np.maximum((A0 * M * M - w @ w.T) / (M * M - M), 0.0)
    assert np.max(np.abs(A - ref)) < 1e-12
