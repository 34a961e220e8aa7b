"""Thin ctypes binding over the C ABI in include/dwc.h (libdwc.so, built in-tree for
sm_100a).  Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no fallback: if the library is missing or the device is not a
B200 the calls raise."""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DWC_LIB", os.path.join(_HERE, "libdwc.so"))   # override: experiments only

DWC_FULL_GRID = 1
DWC_CUBIC = 2
DWC_DIAG_REMOVAL = 4
DWC_ALT_SWEEPS = 8
DWC_GS_DENSE_STREAM = 16
DWC_GS_RESIDUAL = 32
DWC_PAPER_PSF = 64
DWC_THROUGHPUT = 128
GS_KERNELS = {0: "none", 1: "cluster", 2: "cluster_xtra", 3: "alternating", 4: "residual"}
STATUS = {0: "DWC_OK", -1: "DWC_EINVAL", -2: "DWC_ESINGULAR", -3: "DWC_ENUMERIC",
          -4: "DWC_ENOMEM", -5: "DWC_ECUDA", -6: "DWC_ESTATE"}


class DwcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Array(C.Structure):
    _fields_ = [("m", C.c_int32), ("mic_xyz", C.c_void_p), ("c0", C.c_double)]


class Grid(C.Structure):
    _fields_ = [("n", C.c_int32), ("side_len", C.c_double), ("z0", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double)]


class Params(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("eps_mode", C.c_int32), ("sweeps", C.c_int32),
                ("flags", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("n_bins", C.c_int32), ("sum_keep", C.c_int64), ("sum_keep_sq", C.c_double),
                ("gs_bytes", C.c_double), ("psf_flops", C.c_double), ("das_flops", C.c_double),
                ("launches", C.c_int32), ("ms_total", C.c_float), ("ms_das", C.c_float),
                ("ms_compress", C.c_float), ("ms_psf", C.c_float), ("ms_gs", C.c_float),
                ("gs_kernel", C.c_int32), ("gs_xtra_tiles", C.c_int32), ("gs_ctas", C.c_int32),
                ("gs_max_group", C.c_int32), ("gs_updates", C.c_int64), ("gs_row_bytes", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_1608_05179_b200.build`")
        L = C.CDLL(LIB_PATH)
        P, i32, d = C.c_void_p, C.c_int32, C.c_double
        ap, gp, pp = C.POINTER(Array), C.POINTER(Grid), C.POINTER(Params)
        L.dwc_create.argtypes = [C.c_int, C.POINTER(P)]
        L.dwc_destroy.argtypes = [P]
        band = [P, ap, gp, pp, i32, P, P, P, P, P, P, P, P]
        L.dwc_solve_band.argtypes = band
        L.dwc_solve_band_host.argtypes = band
        L.dwc_steer.argtypes = [P, ap, gp, d, i32, P, P, P]
        L.dwc_das.argtypes = [P, ap, gp, i32, P, P, i32, P, P]
        L.dwc_compress.argtypes = [P, gp, pp, i32, P, P, P, P, P]
        L.dwc_psf.argtypes = [P, ap, gp, d, i32, P, i32, P, P]
        L.dwc_gs.argtypes = [P, i32, P, P, i32, i32, P, P]
        L.dwc_keep_mask.argtypes = [P, i32, i32, P, P, P, P]
        L.dwc_solve_band_snapshots.argtypes = [P, ap, gp, pp, i32, P, i32, P, P, P, P, P, P, P]
        L.dwc_csm.argtypes = [P, i32, i32, i32, P, P, P]
        L.dwc_keep_unmask.argtypes = [P, i32, i32, P, P, P, P]
        L.dwc_set_timing.argtypes = [P, C.c_int]
        L.dwc_get_stats.argtypes = [P, C.POINTER(Stats)]
        L.dwc_last_error.restype = C.c_char_p
        L.dwc_version.restype = C.c_char_p
        L.dwc_workspace_bytes.argtypes = [P]
        L.dwc_workspace_bytes.restype = C.c_size_t
        for name in ("dwc_create", "dwc_destroy", "dwc_solve_band", "dwc_solve_band_host", "dwc_steer",
                     "dwc_das", "dwc_compress", "dwc_psf", "dwc_gs", "dwc_keep_mask", "dwc_keep_unmask",
                     "dwc_solve_band_snapshots", "dwc_csm",
                     "dwc_set_timing", "dwc_get_stats"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise DwcError(rc, lib().dwc_last_error().decode())


@dataclasses.dataclass
class Geometry:
    """Array + scan grid."""
    mic_xyz: np.ndarray      # (M,3) metres
    n: int
    side_len: float
    z0: float
    c0: float = 343.0
    cx: float = 0.0
    cy: float = 0.0

    def __post_init__(self):
        self.mic_xyz = np.ascontiguousarray(self.mic_xyz, dtype=np.float64).reshape(-1, 3)

    @property
    def m(self) -> int:
        return self.mic_xyz.shape[0]

    @property
    def S(self) -> int:
        return self.n * self.n

    def c_array(self) -> Array:
        return Array(self.m, self.mic_xyz.ctypes.data, float(self.c0))

    def c_grid(self) -> Grid:
        return Grid(int(self.n), float(self.side_len), float(self.z0), float(self.cx), float(self.cy))


def _gs_kernel_flag(dense_stream) -> int:
    """dense_stream: None = automatic (by system size), True = dense-stream kernel, False = residual."""
    if dense_stream is None:
        return 0
    return DWC_GS_DENSE_STREAM if dense_stream else DWC_GS_RESIDUAL


def _flags(full_grid: bool, order: int, dr: bool = False, alt: bool = False, dense_stream=None,
           paper: bool = False, throughput: bool = False) -> int:
    if order not in (1, 3):
        raise ValueError("order must be 1 (linear predictor) or 3 (cubic)")
    return ((DWC_FULL_GRID if full_grid else 0) | (DWC_CUBIC if order == 3 else 0) |
            (DWC_DIAG_REMOVAL if dr else 0) | (DWC_ALT_SWEEPS if alt else 0) |
            (0 if paper else _gs_kernel_flag(dense_stream)) | (DWC_PAPER_PSF if paper else 0) |
            (DWC_THROUGHPUT if throughput else 0))


def _stream(stream, device=None) -> int:
    """The cudaStream_t to enqueue on: `stream`, else the current stream of the context's device."""
    import torch
    s = torch.cuda.current_stream(device) if stream is None else stream
    return int(s.cuda_stream)


def _rec(stream, *tensors):
    """A call enqueued on `stream` reads and writes these device tensors: the caching allocator
    allocated them on (or for) another stream -- the current one -- and would otherwise hand their
    blocks out again as soon as the Python objects die, while the call's kernels still run on
    `stream` (found with consecutive bands on several contexts, each on its own stream: an output
    dropped before its stream synchronised was reallocated to another band's call).
    record_stream delays the reuse until `stream`'s work queued at free time is done."""
    if stream is None:
        return
    for t in tensors:
        if t is not None and getattr(t, "is_cuda", False):
            t.record_stream(stream)


def _check_out(out: dict, K: int, S: int, want_b: bool, host: bool, device=None):
    """Caller-supplied output buffers: shape, dtype, contiguity and residency (the C call writes
    K*S elements through raw pointers)."""
    import torch
    spec = {"n_keep": ((K,), torch.int32), "keep_idx": ((K, S), torch.int32), "x_map": ((K, S), torch.float32)}
    if want_b or out.get("b_map") is not None:
        spec["b_map"] = ((K, S), torch.float64)
    for key, (shape, dtype) in spec.items():
        t = out.get(key)
        if t is None:
            raise ValueError(f"out[{key!r}] is missing")
        if not isinstance(t, torch.Tensor) or tuple(t.shape) != shape or t.dtype != dtype or not t.is_contiguous():
            raise ValueError(f"out[{key!r}] must be a contiguous {dtype} tensor of shape {shape}")
        if host and t.is_cuda:
            raise ValueError(f"out[{key!r}] must be a host tensor")
        if not host and (not t.is_cuda or (device is not None and t.device != device)):
            raise ValueError(f"out[{key!r}] must be a CUDA tensor on {device}")


def _dev(t, dtype, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


class Context:
    """One dwc_ctx on one CUDA device."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _check(lib().dwc_create(int(device), C.byref(self._h)))
        self.device = device

    def close(self):
        if self._h:
            lib().dwc_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- hot path ---------------------------------------------------------------
    def solve_band(self, geom: Geometry, freqs: Sequence[float], csm, epsilon: float, sweeps: int,
                   eps_mode: int = 0, full_grid: bool = False, want_b: bool = False, out=None, order: int = 1,
                   stream=None, dr: bool = False, alt: bool = False, dense_stream=None, paper: bool = False,
                   throughput: bool = False):
        """Batched S0..S8 on device tensors.  csm: cuda complex128 [K,M,M].
        Returns dict(n_keep int32[K], keep_idx int32[K,S], x_map float32[K,S], b_map, warn)."""
        import torch
        freqs = np.ascontiguousarray(freqs, dtype=np.float64)
        K, S = len(freqs), geom.S
        if tuple(csm.shape) != (K, geom.m, geom.m):
            raise ValueError(f"csm shape {tuple(csm.shape)} != {(K, geom.m, geom.m)}")
        dev = csm.device
        if out is None:
            out = {"n_keep": torch.empty(K, dtype=torch.int32, device=dev),
                   "keep_idx": torch.empty((K, S), dtype=torch.int32, device=dev),
                   "x_map": torch.empty((K, S), dtype=torch.float32, device=dev),
                   "b_map": torch.empty((K, S), dtype=torch.float64, device=dev) if want_b else None}
        else:
            _check_out(out, K, S, want_b, host=False, device=dev)
        warn = np.zeros(K, dtype=np.uint32)
        arr, grid = geom.c_array(), geom.c_grid()
        prm = Params(float(epsilon), int(eps_mode), int(sweeps), _flags(full_grid, order, dr, alt, dense_stream, paper, throughput))
        _check(lib().dwc_solve_band(
            self._h, C.byref(arr), C.byref(grid), C.byref(prm), K, freqs.ctypes.data,
            _dev(csm, torch.complex128, "csm"), _dev(out["n_keep"], torch.int32, "n_keep"),
            _dev(out["keep_idx"], torch.int32, "keep_idx"), _dev(out["x_map"], torch.float32, "x_map"),
            _dev(out["b_map"], torch.float64, "b_map") if out.get("b_map") is not None else None,
            warn.ctypes.data, _stream(stream, self.device)))
        _rec(stream, csm, out["n_keep"], out["keep_idx"], out["x_map"], out.get("b_map"))
        out["warn"] = warn
        return out

    def solve_band_host(self, geom: Geometry, freqs, csm, epsilon: float, sweeps: int, eps_mode: int = 0,
                        full_grid: bool = False, want_b: bool = False, out=None, stream=None, order: int = 1,
                        dr: bool = False, alt: bool = False, dense_stream=None, paper: bool = False,
                   throughput: bool = False):
        """Same as solve_band with host buffers (numpy or CPU tensors, pinned or not); the
        host<->device copies happen inside the C call, which returns when results are on the host."""
        import torch
        freqs = np.ascontiguousarray(freqs, dtype=np.float64)
        K, S = len(freqs), geom.S
        if isinstance(csm, np.ndarray):
            csm = torch.from_numpy(np.ascontiguousarray(csm, dtype=np.complex128))
        if tuple(csm.shape) != (K, geom.m, geom.m) or csm.dtype != torch.complex128 or csm.is_cuda:
            raise ValueError("csm must be a host complex128 [K,M,M] array")
        if out is None:
            out = {"n_keep": torch.empty(K, dtype=torch.int32), "keep_idx": torch.empty((K, S), dtype=torch.int32),
                   "x_map": torch.empty((K, S), dtype=torch.float32),
                   "b_map": torch.empty((K, S), dtype=torch.float64) if want_b else None}
        else:
            _check_out(out, K, S, want_b, host=True)
        warn = np.zeros(K, dtype=np.uint32)
        arr, grid = geom.c_array(), geom.c_grid()
        prm = Params(float(epsilon), int(eps_mode), int(sweeps), _flags(full_grid, order, dr, alt, dense_stream, paper, throughput))
        csm = csm.contiguous()
        _check(lib().dwc_solve_band_host(
            self._h, C.byref(arr), C.byref(grid), C.byref(prm), K, freqs.ctypes.data, csm.data_ptr(),
            out["n_keep"].data_ptr(), out["keep_idx"].data_ptr(), out["x_map"].data_ptr(),
            out["b_map"].data_ptr() if out.get("b_map") is not None else None,
            warn.ctypes.data, _stream(stream, self.device)))
        out["warn"] = warn
        return out

    # ---- stage entry points ---------------------------------------------------------
    def solve_band_snapshots(self, geom: Geometry, freqs: Sequence[float], snap, epsilon: float, sweeps: int,
                             eps_mode: int = 0, full_grid: bool = False, want_b: bool = False, order: int = 1,
                             stream=None, dr: bool = False, alt: bool = False, dense_stream=None, paper: bool = False,
                   throughput: bool = False):
        """The path from snapshot spectra (Eq. 1 on the device).  snap: cuda complex128 [K,M,I]."""
        import torch
        freqs = np.ascontiguousarray(freqs, dtype=np.float64)
        K, S = len(freqs), geom.S
        if snap.dim() != 3 or tuple(snap.shape[:2]) != (K, geom.m):
            raise ValueError(f"snap shape {tuple(snap.shape)} != {(K, geom.m, 'I')}")
        dev = snap.device
        out = {"n_keep": torch.empty(K, dtype=torch.int32, device=dev),
               "keep_idx": torch.empty((K, S), dtype=torch.int32, device=dev),
               "x_map": torch.empty((K, S), dtype=torch.float32, device=dev),
               "b_map": torch.empty((K, S), dtype=torch.float64, device=dev) if want_b else None}
        warn = np.zeros(K, dtype=np.uint32)
        arr, grid = geom.c_array(), geom.c_grid()
        prm = Params(float(epsilon), int(eps_mode), int(sweeps), _flags(full_grid, order, dr, alt, dense_stream, paper, throughput))
        _check(lib().dwc_solve_band_snapshots(
            self._h, C.byref(arr), C.byref(grid), C.byref(prm), K, freqs.ctypes.data, int(snap.shape[2]),
            _dev(snap, torch.complex128, "snap"), _dev(out["n_keep"], torch.int32, "n_keep"),
            _dev(out["keep_idx"], torch.int32, "keep_idx"), _dev(out["x_map"], torch.float32, "x_map"),
            _dev(out["b_map"], torch.float64, "b_map") if out["b_map"] is not None else None,
            warn.ctypes.data, _stream(stream, self.device)))
        _rec(stream, snap, out["n_keep"], out["keep_idx"], out["x_map"], out["b_map"])
        out["warn"] = warn
        return out

    def csm(self, snap, stream=None):
        """Eq. 1 on the device: snap cuda complex128 [K,M,I] -> C complex128 [K,M,M]."""
        import torch
        K, M, I = snap.shape
        out = torch.empty((K, M, M), dtype=torch.complex128, device=snap.device)
        _check(lib().dwc_csm(self._h, M, K, I, _dev(snap, torch.complex128, "snap"),
                             _dev(out, torch.complex128, "csm"), _stream(stream, self.device)))
        _rec(stream, snap, out)
        return out

    def steer(self, geom: Geometry, freq: float, idx, stream=None):
        import torch
        idx = idx.to(torch.int32).contiguous()
        E = torch.empty((idx.numel(), geom.m), dtype=torch.complex128, device=idx.device)
        arr, grid = geom.c_array(), geom.c_grid()
        _check(lib().dwc_steer(self._h, C.byref(arr), C.byref(grid), float(freq), idx.numel(),
                               _dev(idx, torch.int32, "idx"), _dev(E, torch.complex128, "E"), _stream(stream, self.device)))
        _rec(stream, idx, E)
        return E

    def das(self, geom: Geometry, freqs, csm, stream=None, dr: bool = False, paper: bool = False):
        import torch
        freqs = np.ascontiguousarray(freqs, dtype=np.float64)
        b = torch.empty((len(freqs), geom.S), dtype=torch.float64, device=csm.device)
        arr, grid = geom.c_array(), geom.c_grid()
        _check(lib().dwc_das(self._h, C.byref(arr), C.byref(grid), len(freqs), freqs.ctypes.data,
                             _dev(csm, torch.complex128, "csm"),
                             (DWC_DIAG_REMOVAL if dr else 0) | (DWC_PAPER_PSF if paper else 0),
                             _dev(b, torch.float64, "b"), _stream(stream, self.device)))
        _rec(stream, csm, b)
        return b

    def compress(self, geom: Geometry, b_map, epsilon: float, eps_mode: int = 0, full_grid: bool = False, order: int = 1,
                 want_level: bool = False, stream=None):
        import torch
        K = b_map.shape[0]
        nk = torch.empty(K, dtype=torch.int32, device=b_map.device)
        keep = torch.empty((K, geom.S), dtype=torch.int32, device=b_map.device)
        lev = torch.empty((K, geom.S), dtype=torch.uint8, device=b_map.device) if want_level else None
        grid = geom.c_grid()
        prm = Params(float(epsilon), int(eps_mode), 1, _flags(full_grid, order))
        _check(lib().dwc_compress(self._h, C.byref(grid), C.byref(prm), K, _dev(b_map, torch.float64, "b_map"),
                                  _dev(nk, torch.int32, "n_keep"), _dev(keep, torch.int32, "keep_idx"),
                                  _dev(lev, torch.uint8, "level") if lev is not None else None, _stream(stream, self.device)))
        _rec(stream, b_map, nk, keep, lev)
        return nk, keep, lev

    def psf(self, geom: Geometry, freq: float, keep_idx, stream=None, dr: bool = False, paper: bool = False):
        import torch
        keep_idx = keep_idx.to(torch.int32).contiguous()
        n = keep_idx.numel()
        A = torch.empty((n, n), dtype=torch.float32, device=keep_idx.device)
        arr, grid = geom.c_array(), geom.c_grid()
        _check(lib().dwc_psf(self._h, C.byref(arr), C.byref(grid), float(freq), n,
                             _dev(keep_idx, torch.int32, "keep_idx"),
                             (DWC_DIAG_REMOVAL if dr else 0) | (DWC_PAPER_PSF if paper else 0),
                             _dev(A, torch.float32, "A"), _stream(stream, self.device)))
        _rec(stream, keep_idx, A)
        return A

    def gs(self, A, b, sweeps: int, stream=None, alt: bool = False, dense_stream=None, general: bool = False):
        import torch
        n = A.shape[0]
        x = torch.empty(n, dtype=torch.float32, device=A.device)
        fl = DWC_PAPER_PSF if general else ((DWC_ALT_SWEEPS if alt else 0) | _gs_kernel_flag(dense_stream))
        _check(lib().dwc_gs(self._h, n, _dev(A, torch.float32, "A"), _dev(b, torch.float64, "b"), int(sweeps),
                            fl, _dev(x, torch.float32, "x"), _stream(stream, self.device)))
        _rec(stream, A, b, x)
        return x

    # ---- multi-GPU gather helpers ----------------------------------------------------------
    def keep_mask(self, n_keep, keep_idx, stream=None):
        """Keep lists [K, S] (ascending, -1 padded) -> bitmask words [K, ceil(S/32)] (int32
        tensor holding the uint32 bit patterns: bit s%32 of word s/32)."""
        import torch
        K, S = keep_idx.shape
        mask = torch.empty((K, (S + 31) // 32), dtype=torch.int32, device=keep_idx.device)
        _check(lib().dwc_keep_mask(self._h, K, S, _dev(n_keep, torch.int32, "n_keep"),
                                   _dev(keep_idx, torch.int32, "keep_idx"), _dev(mask, torch.int32, "mask"),
                                   _stream(stream, self.device)))
        _rec(stream, n_keep, keep_idx, mask)
        return mask

    def keep_unmask(self, mask, S: int, stream=None):
        """Inverse of keep_mask: (n_keep [K], keep_idx [K, S] ascending, -1 padded)."""
        import torch
        K = mask.shape[0]
        n_keep = torch.empty(K, dtype=torch.int32, device=mask.device)
        keep_idx = torch.empty((K, S), dtype=torch.int32, device=mask.device)
        _check(lib().dwc_keep_unmask(self._h, K, int(S), _dev(mask, torch.int32, "mask"),
                                     _dev(n_keep, torch.int32, "n_keep"), _dev(keep_idx, torch.int32, "keep_idx"),
                                     _stream(stream, self.device)))
        _rec(stream, mask, n_keep, keep_idx)
        return n_keep, keep_idx

    # ---- diagnostics --------------------------------------------------------------------
    def set_timing(self, enable: bool = True):
        _check(lib().dwc_set_timing(self._h, 1 if enable else 0))

    def stats(self) -> dict:
        s = Stats()
        _check(lib().dwc_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def workspace_bytes(self) -> int:
        return int(lib().dwc_workspace_bytes(self._h))


def exported_symbols_from_header(header: Optional[str] = None):
    """Function names declared with DWC_API in include/dwc.h."""
    import re
    header = header or os.path.join(_HERE, "..", "include", "dwc.h")
    return re.findall(r"DWC_API\s+[\w\s\*]*?\b(dwc_\w+)\s*\(", open(header).read())
