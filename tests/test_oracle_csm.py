"""Pins for the oracle's Eq. 1: C = (1/I) sum_i p_i p_i^H, the step before
the path."""
import numpy as np
import pytest
from scipy.linalg import hadamard

import synth


def _geom():
    mic = synth.spiral_array(16, 0.5, 2)
    src = synth.grid_node_xyz(21, 1.0, 1.0, 0.0, 0.0, np.array([50, 137, 220, 301]))
    return mic, src


def test_orthogonal_design_reproduces_exact_csm(oracle_lib):
    """Snapshots p_i = sum_s sqrt(x_s) h_si g_s with the rows of a Hadamard matrix
    ((1/I) sum_i h_si h_ti = delta_st) average to the exact model CSM of Eq. 8,
    C = sum_s x_s g_s g_s^H (computed independently by synth.csm_exact)."""
    mic, src = _geom()
    x = np.array([1.0, 0.5, 0.25, 2.0])
    for f in (1000.0, 4000.0):
        g = synth.propagation_vectors(mic, src, f, 343.0)
        H = hadamard(8)[: len(x)].astype(float)            # 4 orthogonal +-1 rows of length 8
        p = (g * np.sqrt(x)[None, :]) @ H
        C = oracle_lib.csm(p)
        ref = synth.csm_exact(mic, src, x, f, 343.0)
        assert np.abs(C - ref).max() <= 1e-13 * np.abs(ref).max()


def test_single_snapshot_is_outer_product(oracle_lib):
    rng = np.random.default_rng(3)
    p = rng.standard_normal((9, 1)) + 1j * rng.standard_normal((9, 1))
    C = oracle_lib.csm(p)
    R = np.outer(p[:, 0], p[:, 0].conj())
    assert np.abs(C - R).max() <= 4e-16 * np.abs(R).max()


def test_hermitian_psd_trace_scaling(oracle_lib):
    rng = np.random.default_rng(4)
    p = rng.standard_normal((12, 37)) + 1j * rng.standard_normal((12, 37))
    C = oracle_lib.csm(p)
    assert np.array_equal(C, C.conj().T)                   # exact: same products, mirrored signs
    ev = np.linalg.eigvalsh(C)
    assert ev.min() >= -1e-12 * ev.max()
    assert np.linalg.matrix_rank(oracle_lib.csm(p[:, :5]), tol=1e-10) == 5   # rank <= I
    assert abs(np.trace(C).real - np.sum(np.abs(p) ** 2) / 37) < 1e-12 * np.trace(C).real
    assert np.allclose(oracle_lib.csm(2j * p), 4 * C, rtol=1e-14, atol=0)


def test_sampled_config_snapshots_match_the_csm_input(oracle_lib):
    """The snapshot generator and the CSM generator are the same draws: Eq. 1 on cfg2's
    snapshots equals the CSM the CSM-in path is fed (to rounding)."""
    band = synth.make_band("cfg2", bins=[0, 5])
    snap = synth.make_snapshots("cfg2", bins=[0, 5])
    C = oracle_lib.csm(snap)
    assert np.abs(C - band.csm).max() <= 1e-12 * np.abs(band.csm).max()
    with pytest.raises(ValueError):
        synth.make_snapshots("cfg1")
