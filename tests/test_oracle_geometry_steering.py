"""Pins for the oracle's geometry, Eq. 24 helper and S1 steering vectors.

Each pin is something the paper or the mathematics fixes, independent of the
oracle's own code path (values printed in PAPER.md, closed forms, invariants,
or the paper's *other* formula for the same quantity)."""
import math
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _table1():
    vals = {}
    for line in open(os.path.join(GOLD, "paper_table1.txt")):
        line = line.split("#")[0].strip()
        if line:
            k, v = line.split("=")
            vals[k.strip()] = float(v)
    return vals


def test_table1_geometry(oracle_lib):
    """Table 1, Eq. 24 (:291-294): L, B, S, dx/B, k, lambda."""
    t = _table1()
    z0, alpha = t["z0"], math.radians(t["alpha_deg"])
    L = 2 * z0 * math.tan(alpha / 2)
    assert abs(L - t["L"]) < 0.01
    n = int(t["N"])
    assert n * n == t["S"]
    # grid spacing from the oracle's own node positions (reading R17: dx = L/(N-1))
    p0 = oracle_lib.grid_point(n, L, z0, 0.0, 0.0, 0)
    p1 = oracle_lib.grid_point(n, L, z0, 0.0, 0.0, 1)
    pn = oracle_lib.grid_point(n, L, z0, 0.0, 0.0, n)
    dx = p1[0] - p0[0]
    assert abs((pn[1] - p0[1]) - dx) < 1e-12 and abs(p0[0] + L / 2) < 1e-12 and p0[2] == z0
    B = oracle_lib.rayleigh_beamwidth(z0, t["c0"], math.radians(t["phi_deg"]), t["D"], t["f"])
    assert abs(B - t["B"]) < 0.01
    assert abs(dx / B - t["dx_over_B"]) < 0.005
    lam = t["c0"] / t["f"]
    assert abs(lam - t["lambda"]) < 0.001
    k = 2 * math.pi * t["f"] / t["c0"]
    assert abs(k - 55.44) < 0.01                           # SPEC.md:210 (derived from :289-290)


def test_beamwidth_closed_forms(oracle_lib):
    """phi=0 collapses; B is proportional to 1/f."""
    assert abs(oracle_lib.rayleigh_beamwidth(1.0, 340.0, 0.0, 1.0, 340.0) - 1.22) < 1e-12
    b1 = oracle_lib.rayleigh_beamwidth(2.0, 343.0, 0.3, 1.5, 1000.0)
    b2 = oracle_lib.rayleigh_beamwidth(2.0, 343.0, 0.3, 1.5, 2000.0)
    assert abs(b1 / b2 - 2.0) < 1e-12


def test_spacing_warning_boundary(oracle_lib):
    """dx/B <= 0.2 recommended: the flag rises above 0.2 only."""
    mic = synth.spiral_array(16, 1.0, 1)
    # cfg3-like geometry: L=1, z0=1, N=101 -> dx = 0.01; B ~ 1/f, so high f -> small B
    assert oracle_lib.spacing_warning(mic, 343.0, 101, 1.0, 1.0, 500.0) == 0
    rmax = np.max(np.hypot(mic[:, 0], mic[:, 1]))
    phi = math.atan(1.0 / 2.0)
    # frequency at which dx/B == 0.2 exactly
    f_star = 0.2 * 1.22 * 1.0 * 343.0 / (math.cos(phi) ** 3 * 2 * rmax * 0.01)
    assert oracle_lib.spacing_warning(mic, 343.0, 101, 1.0, 1.0, f_star * 0.999) == 0
    assert oracle_lib.spacing_warning(mic, 343.0, 101, 1.0, 1.0, f_star * 1.001) == 1


@pytest.fixture(scope="module")
def small_geom():
    mic = synth.spiral_array(16, 0.5, 2)
    return dict(mic=mic, c0=343.0, n=9, L=1.2, z0=0.8, cx=0.05, cy=-0.1)


def _nodes(g):
    return synth.grid_node_xyz(g["n"], g["L"], g["z0"], g["cx"], g["cy"])


def test_steering_norm_amplitude_phase(oracle_lib, small_geom):
    """R1: e_s = sqrt(M) g_s/||g_s||, g_m = exp(-jkd)/d  =>  ||e_s||^2 = M,
    |e_ms| d_ms constant over m, arg e_ms = -k d_ms (mod 2 pi)."""
    g = small_geom
    f = 3000.0
    idx = np.arange(g["n"] ** 2)
    E = oracle_lib.steering(g["mic"], g["c0"], g["n"], g["L"], g["z0"], g["cx"], g["cy"], f, idx)
    M = g["mic"].shape[0]
    assert np.allclose(np.sum(np.abs(E) ** 2, axis=1), M, rtol=0, atol=1e-12)
    nodes = _nodes(g)
    d = np.linalg.norm(nodes[:, None, :] - g["mic"][None, :, :], axis=-1)
    ad = np.abs(E) * d
    assert np.allclose(ad / ad[:, :1], 1.0, atol=1e-12)
    k = 2 * math.pi * f / g["c0"]
    ph = np.angle(E * np.exp(1j * k * d))
    assert np.max(np.abs(ph)) < 1e-9


def test_steering_zero_frequency_real_positive(oracle_lib, small_geom):
    """k = 0 => all phases zero, e real positive."""
    g = small_geom
    E = oracle_lib.steering(g["mic"], g["c0"], g["n"], g["L"], g["z0"], g["cx"], g["cy"], 0.0,
                            np.arange(10))
    assert np.all(E.real > 0) and np.all(E.imag == 0)


def test_steering_equals_normalised_eq7_vector(oracle_lib, small_geom):
    """The paper's Eq. 7 vector g^P_m = |r_s|/|r_s-r_m| e^{-jk|r_s-r_m|} (with the |r_s|
    factor, computed by the scene generator) normalised to norm sqrt(M) is the oracle's e."""
    g = small_geom
    f = 5200.0
    idx = np.array([0, 7, 40, 80])
    E = oracle_lib.steering(g["mic"], g["c0"], g["n"], g["L"], g["z0"], g["cx"], g["cy"], f, idx)
    gp = synth.propagation_vectors(g["mic"], _nodes(g)[idx], f, g["c0"])   # (M, pts)
    M = g["mic"].shape[0]
    ref = (math.sqrt(M) * gp / np.linalg.norm(gp, axis=0)).T
    assert np.max(np.abs(E - ref)) < 1e-12


def test_steering_singular_point(oracle_lib):
    """A grid node on a microphone is a singularity error."""
    mic = np.array([[0.0, 0.0, 1.0], [0.3, 0.0, 0.0]])
    with pytest.raises(oracle_lib.OracleError) as ei:
        oracle_lib.steering(mic, 343.0, 3, 1.0, 1.0, 0.0, 0.0, 1000.0, [4])  # node 4 = (0,0,1)
    assert ei.value.code == -2
