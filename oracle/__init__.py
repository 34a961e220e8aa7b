"""ctypes shim over the fp64 CPU ORACLE (oracle/dwc_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` leg.  The product package
(paper_1608_05179_b200) never imports this module and shares no code with it.

Every function is a thin marshalling wrapper; the arithmetic lives in the C
file, each function there citing the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dwc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread", "-std=c11",
          "-D_GNU_SOURCE"]


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _P = C.c_void_p
        d, i = C.c_double, C.c_int
        geo = [i, _P, d, i, d, d, d, d]  # m, mic, c0, n, L, z0, cx, cy
        _lib.or_grid_point.argtypes = [i, d, d, d, d, i, _P]
        _lib.or_rayleigh_beamwidth.argtypes = [d, d, d, d, d]
        _lib.or_rayleigh_beamwidth.restype = d
        _lib.or_spacing_warning.argtypes = [i, _P, d, i, d, d, d]
        _lib.or_steering.argtypes = geo + [d, i, _P, _P]
        _lib.or_das.argtypes = geo + [d, _P, _P, i]
        _lib.or_max_level.argtypes = [i]
        _lib.or_wavelet_details.argtypes = [i, _P, _P, _P, i]
        _lib.or_compress.argtypes = [i, _P, d, i, i, _P, _P, _P, _P, i]
        _lib.or_psf.argtypes = geo + [d, i, _P, _P, i]
        _lib.or_gs.argtypes = [i, _P, _P, i, _P, i]
        _lib.or_das_paper.argtypes = geo + [d, _P, _P]
        _lib.or_psf_paper.argtypes = geo + [d, i, _P, _P]
        _lib.or_csm.argtypes = [i, i, _P, _P]
        _lib.or_solve_bin.argtypes = geo + [d, _P, d, i, i, i, _P, _P, _P, _P]
        _lib.or_solve_band.argtypes = geo + [i, _P, _P, d, i, i, i, _P, _P, _P, _P, i]
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"oracle {where} failed with code {code}")
        self.code = code


def _chk(rc: int, where: str) -> int:
    if rc < 0:
        raise OracleError(rc, where)
    return rc


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _geo(mic, c0, n, L, z0, cx, cy):
    mic = _f64(mic).reshape(-1, 3)
    return mic, [mic.shape[0], _p(mic), float(c0), int(n), float(L), float(z0), float(cx), float(cy)]


def grid_point(n, L, z0, cx, cy, s) -> np.ndarray:
    out = np.zeros(3)
    lib().or_grid_point(n, L, z0, cx, cy, s, _p(out))
    return out


def rayleigh_beamwidth(z0, c0, phi, D, f) -> float:
    return lib().or_rayleigh_beamwidth(float(z0), float(c0), float(phi), float(D), float(f))


def spacing_warning(mic, c0, n, L, z0, freq) -> int:
    mic = _f64(mic).reshape(-1, 3)
    return lib().or_spacing_warning(mic.shape[0], _p(mic), float(c0), int(n), float(L), float(z0),
                                    float(freq))


def steering(mic, c0, n, L, z0, cx, cy, freq, idx) -> np.ndarray:
    """E[pt, m] complex128: the normalised steering vectors of the given nodes."""
    mic, g = _geo(mic, c0, n, L, z0, cx, cy)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    E = np.zeros((len(idx), mic.shape[0], 2))
    _chk(lib().or_steering(*g, float(freq), len(idx), _p(idx), _p(E)), "steering")
    return E[..., 0] + 1j * E[..., 1]


def das(mic, c0, n, L, z0, cx, cy, freq, csm, dr: bool = False) -> np.ndarray:
    """Eq. 2; dr: diagonal removal (R20)."""
    mic, g = _geo(mic, c0, n, L, z0, cx, cy)
    csm = np.ascontiguousarray(csm, dtype=np.complex128)
    b = np.zeros(n * n)
    _chk(lib().or_das(*g, float(freq), _p(csm), _p(b), int(bool(dr))), "das")
    return b


def max_level(n: int) -> int:
    return lib().or_max_level(int(n))


def wavelet_details(n: int, b, order: int = 1) -> Tuple[np.ndarray, np.ndarray]:
    """order 1: linear predictor (R7); 3: 4-point cubic predictor (R19)."""
    b = _f64(b)
    d = np.zeros(n * n)
    lv = np.zeros(n * n, dtype=np.uint8)
    _chk(lib().or_wavelet_details(int(n), _p(b), _p(d), _p(lv), int(order)), "wavelet_details")
    return d, lv


def compress(n: int, b, eps: float, eps_mode: int = 0, full_grid: bool = False, order: int = 1):
    """-> (keep int32 ascending, level uint8[S], d fp64[S], eps_eff)."""
    b = _f64(b)
    keep = np.zeros(n * n, dtype=np.int32)
    lv = np.zeros(n * n, dtype=np.uint8)
    d = np.zeros(n * n)
    ee = np.zeros(1)
    nk = _chk(lib().or_compress(int(n), _p(b), float(eps), int(eps_mode), int(full_grid),
                                _p(keep), _p(lv), _p(d), _p(ee), int(order)), "compress")
    return keep[:nk].copy(), lv, d, float(ee[0])


def psf(mic, c0, n, L, z0, cx, cy, freq, keep, dr: bool = False) -> np.ndarray:
    """Eq. 10 restricted to keep; dr: the diagonal-removal PSF (R20)."""
    mic, g = _geo(mic, c0, n, L, z0, cx, cy)
    keep = np.ascontiguousarray(keep, dtype=np.int32)
    A = np.zeros((len(keep), len(keep)))
    _chk(lib().or_psf(*g, float(freq), len(keep), _p(keep), _p(A), int(bool(dr))), "psf")
    return A


def das_paper(mic, c0, n, L, z0, cx, cy, freq, csm) -> np.ndarray:
    """Eq. 2 with the paper's Eq. 4 focus vector (fidelity variant, not the GPU path)."""
    mic, g = _geo(mic, c0, n, L, z0, cx, cy)
    csm = np.ascontiguousarray(csm, dtype=np.complex128)
    b = np.zeros(n * n)
    _chk(lib().or_das_paper(*g, float(freq), _p(csm), _p(b)), "das_paper")
    return b


def psf_paper(mic, c0, n, L, z0, cx, cy, freq, keep) -> np.ndarray:
    """Eq. 10 with the paper's v (Eq. 4) and g (Eq. 7): asymmetric (fidelity variant)."""
    mic, g = _geo(mic, c0, n, L, z0, cx, cy)
    keep = np.ascontiguousarray(keep, dtype=np.int32)
    A = np.zeros((len(keep), len(keep)))
    _chk(lib().or_psf_paper(*g, float(freq), len(keep), _p(keep), _p(A)), "psf_paper")
    return A


def csm(snap) -> np.ndarray:
    """Eq. 1: snap complex128 [M, I] (or [K, M, I]) -> C complex128 [M, M] ([K, M, M])."""
    snap = np.ascontiguousarray(snap, dtype=np.complex128)
    if snap.ndim == 3:
        return np.stack([csm(s) for s in snap])
    M, I = snap.shape
    C = np.zeros((M, M), dtype=np.complex128)
    _chk(lib().or_csm(int(M), int(I), _p(snap), _p(C)), "csm")
    return C


def gs(A, b, sweeps: int, alt: bool = False) -> np.ndarray:
    """Eq. 13-14 forward sweeps; alt: alternating directions (R21)."""
    A = _f64(A)
    b = _f64(b)
    x = np.zeros(len(b))
    _chk(lib().or_gs(len(b), _p(A), _p(b), int(sweeps), _p(x), int(bool(alt))), "gs")
    return x


def _flags(full_grid, order, dr=False, alt=False, paper=False):
    return (1 if full_grid else 0) | (2 if order == 3 else 0) | (4 if dr else 0) | (8 if alt else 0) | \
        (16 if paper else 0)


def solve_bin(mic, c0, n, L, z0, cx, cy, freq, csm, eps, eps_mode, sweeps, full_grid=False, order=1, dr=False,
              alt=False, paper=False):
    """-> (keep, x_map fp64[S], b fp64[S])."""
    mic, g = _geo(mic, c0, n, L, z0, cx, cy)
    csm = np.ascontiguousarray(csm, dtype=np.complex128)
    S = n * n
    nk = np.zeros(1, dtype=np.int32)
    keep = np.zeros(S, dtype=np.int32)
    x = np.zeros(S)
    b = np.zeros(S)
    _chk(lib().or_solve_bin(*g, float(freq), _p(csm), float(eps), int(eps_mode), int(sweeps),
                            _flags(full_grid, order, dr, alt, paper), _p(nk), _p(keep), _p(x), _p(b)), "solve_bin")
    return keep[: nk[0]].copy(), x, b


def solve_band(mic, c0, n, L, z0, cx, cy, freqs, csm, eps, eps_mode, sweeps,
               full_grid=False, n_threads: Optional[int] = None, order: int = 1, dr: bool = False,
               alt: bool = False, paper: bool = False):
    """Batched S0..S8 over K bins on a pthread pool.
    -> (n_keep int32[K], keep int32[K,S] (-1 padded), x_map fp64[K,S], b fp64[K,S])."""
    mic, g = _geo(mic, c0, n, L, z0, cx, cy)
    freqs = _f64(freqs)
    csm = np.ascontiguousarray(csm, dtype=np.complex128)
    K = len(freqs)
    S = n * n
    nk = np.zeros(K, dtype=np.int32)
    keep = np.full((K, S), -1, dtype=np.int32)
    x = np.zeros((K, S))
    b = np.zeros((K, S))
    if n_threads is None:
        n_threads = os.cpu_count() or 1
    _chk(lib().or_solve_band(*g, K, _p(freqs), _p(csm), float(eps), int(eps_mode), int(sweeps),
                             _flags(full_grid, order, dr, alt, paper), _p(nk), _p(keep), _p(x), _p(b), int(n_threads)),
         "solve_band")
    return nk, keep, x, b


def solve_band_cfg(band, n_threads: Optional[int] = None, sweeps: Optional[int] = None,
                   full_grid: Optional[bool] = None, eps: Optional[float] = None, order: int = 1,
                   dr: bool = False, alt: bool = False, paper: bool = False):
    """Convenience: run the oracle on a synth.Band."""
    cfg = band.cfg
    return solve_band(band.mic_xyz, cfg.c0, cfg.n, cfg.side_len, cfg.z0, cfg.cx, cfg.cy,
                      band.freqs, band.csm, cfg.epsilon if eps is None else eps, cfg.eps_mode,
                      cfg.sweeps if sweeps is None else sweeps,
                      cfg.full_grid if full_grid is None else full_grid, n_threads, order, dr, alt, paper)
