"""Seeded synthetic inputs for the DAMAS-on-compressed-grid hot path.

This module is the ONLY code shared by the oracle (`oracle/`) and the CUDA
path (`paper_1608_05179_b200/`).  It produces *inputs*: microphone-array
geometry, scan-grid parameters, frequency bins, source scenes and the
cross-spectral matrices (CSMs) a measurement would deliver.  It contains none
of the method's arithmetic (no steering normalisation, no DAS map, no wavelet
threshold, no PSF, no Gauss-Seidel): the hot path starts from the CSM.

Forward model (the measurement the paper simulates, §3 Eq. 5-8 and
§2 Eq. 1):
  * a source at grid node r_s with mean-square pressure amplitude q_s^2 "in
    terms of the pressure produced at the array centre"
    produces at microphone m the pressure q_s * g_m(r_s) with the paper's
    normalised propagation vector (Eq. 7, exponent typo
    r -> r_s fixed):  g_m(r_s) = |r_s|/|r_s - r_m| * exp(-j k |r_s - r_m|)
  * exact CSM (Eq. 8): C = sum_s q_s^2 g_s g_s^H
  * sampled CSM (Eq. 1, PAPER.md:88-95 + "Gaussian white noise ... at the
    microphone array"): C = (1/I) sum_i p_i p_i^H with
    p_i = sum_s q_s xi_{s,i} g_s + n_i,  xi ~ CN(0,1) iid (incoherent sources),
    n_i ~ CN(0, sigma^2 I), sigma^2 = mean_m E|signal_m|^2 / 10^(SNR/10).

Config values follow SURVEY.md §8(d) / BASELINE.json `configs`.  Every random
draw comes from numpy's PCG64 seeded by SeedSequence([cfg_id, seed]) (scene)
and SeedSequence([cfg_id, seed, k]) (bin k's snapshots), so any subset of bins
(e.g. one GPU's shard) is generated identically.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

C0_DEFAULT = 343.0


# ----------------------------------------------------------------------------
# geometry
# ----------------------------------------------------------------------------
def spiral_array(m: int, aperture: float, arms: int, psi_deg: float = 30.0,
                 r_in_frac: float = 0.1) -> np.ndarray:
    """Multi-arm logarithmic spiral in the plane z=0 (stand-in for the paper's
    unpublished 60-mic layout).  Returns (m,3) fp64."""
    if m < 2 or m % arms:
        raise ValueError("m must be >= 2 and a multiple of arms")
    per = m // arms
    big_r = aperture / 2.0
    r_in = r_in_frac * big_r
    tpsi = math.tan(math.radians(psi_deg))
    xyz = np.zeros((m, 3), dtype=np.float64)
    idx = 0
    for a in range(arms):
        for i in range(per):
            frac = i / (per - 1) if per > 1 else 1.0
            r = r_in * (big_r / r_in) ** frac
            th = math.log(r / r_in) / tpsi + 2.0 * math.pi * a / arms
            xyz[idx] = (r * math.cos(th), r * math.sin(th), 0.0)
            idx += 1
    return xyz


def grid_node_xyz(n: int, side_len: float, z0: float, cx: float = 0.0,
                  cy: float = 0.0, s: Optional[np.ndarray] = None) -> np.ndarray:
    """Positions of scan-grid nodes: x_c = cx - L/2 + c*dx, y_r = cy - L/2 + r*dx,
    z = z0, dx = L/(n-1), s = r*n + c."""
    if s is None:
        s = np.arange(n * n)
    s = np.asarray(s)
    r, c = np.divmod(s, n)
    dx = side_len / (n - 1)
    out = np.empty(s.shape + (3,), dtype=np.float64)
    out[..., 0] = cx - side_len / 2.0 + c * dx
    out[..., 1] = cy - side_len / 2.0 + r * dx
    out[..., 2] = z0
    return out


def nearest_node(n: int, side_len: float, x: float, y: float,
                 cx: float = 0.0, cy: float = 0.0) -> int:
    dx = side_len / (n - 1)
    c = int(round((x - (cx - side_len / 2.0)) / dx))
    r = int(round((y - (cy - side_len / 2.0)) / dx))
    c = min(max(c, 0), n - 1)
    r = min(max(r, 0), n - 1)
    return r * n + c


def propagation_vectors(mic_xyz: np.ndarray, src_xyz: np.ndarray, freq: float,
                        c0: float) -> np.ndarray:
    """The paper's normalised propagation matrix G (Eq. 5-7): columns g(r_s),
    g_m = |r_s|/|r_s - r_m| exp(-j k |r_s - r_m|).  Returns (M, n_src) complex128.
    Scene synthesis only (the forward model that produces the data)."""
    k = 2.0 * math.pi * freq / c0
    diff = src_xyz[None, :, :] - mic_xyz[:, None, :]
    dist = np.sqrt(np.sum(diff * diff, axis=-1))
    rs = np.sqrt(np.sum(src_xyz * src_xyz, axis=-1))[None, :]
    return (rs / dist) * np.exp(-1j * k * dist)


# ----------------------------------------------------------------------------
# configs (BASELINE.json configs[0..4])
# ----------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    cfg_id: int
    m: int
    aperture: float
    arms: int
    n: int
    side_len: float
    z0: float
    f_lo: float
    f_hi: float
    n_bins: int
    scene: str
    csm: str            # "exact" | "sampled"
    snapshots: int
    snr_db: float
    sweeps: int
    epsilon: float
    eps_mode: int = 0   # 0 relative, 1 absolute
    full_grid: bool = False
    c0: float = C0_DEFAULT
    cx: float = 0.0
    cy: float = 0.0

    @property
    def S(self) -> int:
        return self.n * self.n

    def freqs(self) -> np.ndarray:
        if self.n_bins == 1:
            return np.array([self.f_lo], dtype=np.float64)
        return np.linspace(self.f_lo, self.f_hi, self.n_bins, dtype=np.float64)

    def mics(self) -> np.ndarray:
        return spiral_array(self.m, self.aperture, self.arms)


# epsilon values are relative thresholds calibrated once with the ORACLE on
# seed 0 to hit the kept fraction BASELINE.json names (scripts/calibrate_eps.py
# writes tests/golden/eps_calibration.txt); cfg1 uses the paper's case-1 value.
CONFIGS: Dict[str, Config] = {
    "cfg1": Config("cfg1", 1, 16, 0.5, 1, 21, 1.0, 1.0, 4000.0, 4000.0, 1,
                   "cfg1", "exact", 1, math.inf, 100, 0.1),
    "cfg2": Config("cfg2", 2, 64, 1.0, 8, 81, 2.0, 1.5, 1000.0, 8000.0, 8,
                   "cfg2", "sampled", 1000, 20.0, 1000, 0.0078),
    "cfg3": Config("cfg3", 3, 64, 1.0, 8, 101, 1.0, 1.0, 500.0, 10000.0, 256,
                   "cfg3", "sampled", 2000, 20.0, 1000, 0.00703),
    "cfg4": Config("cfg4", 4, 128, 1.5, 8, 101, 1.0, 1.0, 1000.0, 8000.0, 64,
                   "cfg4", "exact", 1, math.inf, 500, 0.01, full_grid=True),
    "cfg5": Config("cfg5", 5, 128, 1.5, 8, 201, 2.0, 2.0, 500.0, 12000.0, 1024,
                   "cfg5", "sampled", 4000, 10.0, 200, 0.00224),
}


def scene_sources(cfg: Config, seed: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(node indices int64, powers q^2 fp64) of the config's scene."""
    rng = np.random.default_rng(np.random.SeedSequence([cfg.cfg_id, seed]))
    n = cfg.n
    if cfg.scene == "cfg1":
        idx = [nearest_node(n, cfg.side_len, -0.2, 0.0), nearest_node(n, cfg.side_len, 0.2, 0.0)]
        pw = [1.0, 1.0]
    elif cfg.scene in ("cfg2", "cfg4"):
        frac = 0.6 if cfg.scene == "cfg2" else 0.5
        count = 3 if cfg.scene == "cfg2" else 4
        lo = int(round((0.5 - frac / 2) * (n - 1)))
        hi = int(round((0.5 + frac / 2) * (n - 1)))
        idx = []
        while len(idx) < count:
            r, c = rng.integers(lo, hi + 1, size=2)
            s = int(r) * n + int(c)
            if s not in idx:
                idx.append(s)
        pw = [1.0, 0.5, 0.25] if cfg.scene == "cfg2" else [1.0] * 4
    elif cfg.scene == "cfg3":
        idx = []
        while len(idx) < 5:
            x = 0.1 + rng.uniform(-0.1, 0.1)
            y = 0.0 + rng.uniform(-0.1, 0.1)
            s = nearest_node(n, cfg.side_len, x, y)
            if s not in idx:
                idx.append(s)
        mid = 10.0 ** (-rng.uniform(0.0, 1.0, size=3))
        pw = [1.0] + list(mid) + [0.1]
    elif cfg.scene == "cfg5":
        idx = [100 * n + c for c in range(76, 126)]
        pw = [1.0] * 50
        extra = []
        while len(extra) < 10:
            s = int(rng.integers(0, n * n))
            if s not in idx and s not in extra:
                extra.append(s)
        idx += extra
        pw += list(rng.uniform(0.1, 1.0, size=10))
    else:
        raise ValueError(cfg.scene)
    return np.asarray(idx, dtype=np.int64), np.asarray(pw, dtype=np.float64)


def csm_exact(mic_xyz: np.ndarray, src_xyz: np.ndarray, powers: np.ndarray,
              freq: float, c0: float) -> np.ndarray:
    """Eq. 8: C = sum_s q_s^2 g_s g_s^H."""
    g = propagation_vectors(mic_xyz, src_xyz, freq, c0)
    return (g * powers[None, :]) @ g.conj().T


def snapshots_sampled(mic_xyz: np.ndarray, src_xyz: np.ndarray, powers: np.ndarray,
                      freq: float, c0: float, snapshots: int, snr_db: float,
                      rng: np.random.Generator) -> np.ndarray:
    """The I snapshot spectra p_i (M x I complex128) of incoherent CN(0,1) source phasors
    propagated by Eq. 5-7 plus white microphone noise at the given SNR.
    Input of the on-device Eq. 1 path (NEXT-3); csm_sampled averages the same draws."""
    g = propagation_vectors(mic_xyz, src_xyz, freq, c0)
    m = g.shape[0]
    ns = g.shape[1]
    xi = (rng.standard_normal((ns, snapshots)) + 1j * rng.standard_normal((ns, snapshots))) / math.sqrt(2.0)
    p = (g * np.sqrt(powers)[None, :]) @ xi
    sig_pow = float(np.sum(powers * np.sum(np.abs(g) ** 2, axis=0)) / m)
    if math.isfinite(snr_db):
        sigma2 = sig_pow / (10.0 ** (snr_db / 10.0))
        noise = (rng.standard_normal((m, snapshots)) + 1j * rng.standard_normal((m, snapshots))) * math.sqrt(sigma2 / 2.0)
        p = p + noise
    return p


def csm_sampled(mic_xyz: np.ndarray, src_xyz: np.ndarray, powers: np.ndarray,
                freq: float, c0: float, snapshots: int, snr_db: float,
                rng: np.random.Generator) -> np.ndarray:
    """Eq. 1 averaged over I snapshots (the CSM input of the CSM-in path)."""
    p = snapshots_sampled(mic_xyz, src_xyz, powers, freq, c0, snapshots, snr_db, rng)
    return (p @ p.conj().T) / snapshots


def make_snapshots(cfg: "Config | str", seed: int = 0, bins: Optional[Sequence[int]] = None) -> np.ndarray:
    """Snapshot spectra [K, M, I] of a sampled-CSM config, the same draws make_band averages."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.csm == "exact":
        raise ValueError(f"{cfg.name} has an exact CSM (no snapshots)")
    mics = cfg.mics()
    allf = cfg.freqs()
    bins = np.arange(cfg.n_bins) if bins is None else np.asarray(bins, dtype=np.int64)
    src_idx, src_pow = scene_sources(cfg, seed)
    src_xyz = grid_node_xyz(cfg.n, cfg.side_len, cfg.z0, cfg.cx, cfg.cy, src_idx)
    out = np.empty((len(bins), cfg.m, cfg.snapshots), dtype=np.complex128)
    for j, k in enumerate(bins):
        rng = np.random.default_rng(np.random.SeedSequence([cfg.cfg_id, seed, int(k)]))
        out[j] = snapshots_sampled(mics, src_xyz, src_pow, float(allf[k]), cfg.c0, cfg.snapshots, cfg.snr_db, rng)
    return out


@dataclasses.dataclass
class Band:
    """All inputs of one band: what the C-ABI's dwc_solve_band takes."""
    cfg: Config
    mic_xyz: np.ndarray        # (M,3) fp64
    freqs: np.ndarray          # (K,) fp64
    csm: np.ndarray            # (K,M,M) complex128, row-major
    src_idx: np.ndarray
    src_pow: np.ndarray
    bins: np.ndarray           # which bins of the config these are


def make_band(cfg: Config | str, seed: int = 0, bins: Optional[Sequence[int]] = None, block: int = 0) -> Band:
    """The config's band of bins.  block > 0: another measurement block of the same scene (new
    snapshot and noise draws; the exact-CSM configs have no draws, so their block is the band
    itself)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    mics = cfg.mics()
    allf = cfg.freqs()
    bins = np.arange(cfg.n_bins) if bins is None else np.asarray(bins, dtype=np.int64)
    src_idx, src_pow = scene_sources(cfg, seed)
    src_xyz = grid_node_xyz(cfg.n, cfg.side_len, cfg.z0, cfg.cx, cfg.cy, src_idx)
    csm = np.empty((len(bins), cfg.m, cfg.m), dtype=np.complex128)
    for j, k in enumerate(bins):
        f = float(allf[k])
        if cfg.csm == "exact":
            csm[j] = csm_exact(mics, src_xyz, src_pow, f, cfg.c0)
        else:
            key = [cfg.cfg_id, seed, int(k)] + ([int(block)] if block else [])
            rng = np.random.default_rng(np.random.SeedSequence(key))
            csm[j] = csm_sampled(mics, src_xyz, src_pow, f, cfg.c0, cfg.snapshots, cfg.snr_db, rng)
    return Band(cfg, mics, allf[bins].copy(), csm, src_idx, src_pow, bins)


def random_hermitian_psd(m: int, rank: int, rng: np.random.Generator) -> np.ndarray:
    """A random PSD Hermitian matrix (generic CSM-shaped test input)."""
    z = (rng.standard_normal((m, rank)) + 1j * rng.standard_normal((m, rank))) / math.sqrt(2 * rank)
    return z @ z.conj().T


def strided_bins(n_bins: int, count: int) -> List[int]:
    """A strided subset of bins spanning the whole band (used for bounded
    oracle samples and full-size parity checks)."""
    if count >= n_bins:
        return list(range(n_bins))
    step = n_bins / count
    return sorted({int(i * step + step / 2) for i in range(count)})
