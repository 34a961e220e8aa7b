"""GPU parity on the large systems: the Gauss-Seidel kernel configurations that only the big
configs reach (cfg4's full grid, cfg5's S~ up to ~9k), compared with the fp64 oracle element
by element (north_star tolerances: keep set bit-exact, map within 1e-3 relative L2, integrated
power within 1e-3).

On the residual kernel these sizes run its cluster mode (r split over 2-4 CTAs per bin,
dwc_stats.gs_max_group); on the dense-stream cluster kernel the instantiation with extra ring
tiles behind the dynamic tables (dwc_stats.gs_kernel == DWC_GS_KERNEL_CLUSTER_XTRA).  The tests
assert which kernel and cluster size ran, so a change of the selection cannot silently drop the
coverage."""
import dataclasses
import os
import subprocess
import sys

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

TOL_X = 1e-3
TOL_P = 1e-3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def ctx(torch_cuda):
    from paper_1608_05179_b200 import Context
    c = Context(0)
    yield c
    c.close()


def geom_of(band):
    from paper_1608_05179_b200 import Geometry
    cfg = band.cfg
    return Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)


def oracle_args(g):
    return (g.mic_xyz, g.c0, g.n, g.side_len, g.z0, g.cx, g.cy)


_SYS = {}
_ORACLE = {}


def resid_ctas(nk, wide):
    """CTAs per bin of the residual kernel: one CTA up to 5120 padded points (r in registers, 8
    chunks per stream warp above 2560), else a cluster -- wide (5120 points per CTA, the
    compressed grid and dwc_gs) or narrow (2560, the full grid)."""
    sp = (int(nk) + 31) // 32 * 32
    return 1 if sp <= 5120 else -(-sp // (5120 if wide else 2560))


def cfg5_system(oracle_lib, nk):
    """The oracle's PSF and DAS on the nk strongest nodes of cfg5's top bin (12 kHz, M = 128,
    201x201 grid): an S~ = nk system in cfg5's own geometry."""
    if nk not in _SYS:
        band = synth.make_band("cfg5", bins=[1023])
        g = geom_of(band)
        f = band.freqs[0]
        b = oracle_lib.das(*oracle_args(g), f, band.csm[0])
        keep = np.sort(np.argsort(-b)[:nk]).astype(np.int32)
        A = oracle_lib.psf(*oracle_args(g), f, keep)
        _SYS[nk] = (A, b[keep])
    return _SYS[nk]


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
@pytest.mark.parametrize("nk,sweeps", [(2100, 20), (4500, 20), (9150, 20)])
def test_gs_large_systems(ctx, torch_cuda, oracle_lib, nk, sweeps, dense):
    """dwc_gs on S~ = 2100 / 4500 / 9150 (T = 66 / 141 / 286 row blocks: ownership tables,
    y strides and segment runs far beyond the cfg3 sizes; on the dense-stream kernel the
    extra-ring instantiation)."""
    torch = torch_cuda
    A, bt = cfg5_system(oracle_lib, nk)
    ref = oracle_lib.gs(A, bt, sweeps)
    x = ctx.gs(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(bt).cuda(), sweeps,
               dense_stream=dense).cpu().numpy()
    st = ctx.stats()
    if dense:
        assert st["gs_kernel"] == 2 and st["gs_xtra_tiles"] > 0 and st["gs_max_group"] == 4
    else:   # CTAs per bin: one up to 5120 points, else wide clusters of 5120 points per CTA
        assert st["gs_kernel"] == 4 and st["gs_updates"] > 0 and st["gs_max_group"] == resid_ctas(nk, wide=True)
    assert x.min() >= 0
    assert rel_l2(x, ref) < TOL_X, rel_l2(x, ref)
    assert abs(x.sum() - ref.sum()) < TOL_P * ref.sum()


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_gs_large_system_bitwise_deterministic(ctx, torch_cuda, oracle_lib, dense):
    """Repeated runs of an S~ = 4500 system are bit-identical (every summation order is fixed, so
    a difference would be an ordering race in the ring / partial-sum / x-forwarding protocol)."""
    torch = torch_cuda
    A, bt = cfg5_system(oracle_lib, 4500)
    Ad = torch.from_numpy(A.astype(np.float32)).cuda()
    bd = torch.from_numpy(bt).cuda()
    ref = ctx.gs(Ad, bd, 30, dense_stream=dense).cpu().numpy()
    for _ in range(3):
        assert np.array_equal(ctx.gs(Ad, bd, 30, dense_stream=dense).cpu().numpy(), ref)


_XTRA_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1608_05179_b200 import Context
A = np.load({a!r}); b = np.load({b!r})
c = Context(0)
x = c.gs(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), 25, dense_stream=True).cpu().numpy()
st = c.stats()
np.save({out!r}, x)
print(st["gs_kernel"], st["gs_xtra_tiles"])
"""


def test_gs_extra_ring_tiles_do_not_change_results(ctx, torch_cuda, oracle_lib, tmp_path):
    """The extra ring slots only change buffering: DWC_GS_XTRA=0 (the fixed ring) gives the
    bitwise-identical solution of an S~ = 2100 system (separate process: the knob is read once)."""
    torch = torch_cuda
    A, bt = cfg5_system(oracle_lib, 2100)
    A32 = A.astype(np.float32)
    x_default = ctx.gs(torch.from_numpy(A32).cuda(), torch.from_numpy(bt).cuda(), 25, dense_stream=True).cpu().numpy()
    kern_default = ctx.stats()["gs_kernel"]
    pa, pb, po = tmp_path / "A.npy", tmp_path / "b.npy", tmp_path / "x.npy"
    np.save(pa, A32)
    np.save(pb, bt)
    script = _XTRA_SCRIPT.format(root=ROOT, a=str(pa), b=str(pb), out=str(po))
    env = dict(os.environ, DWC_GS_XTRA="0")
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    kern, xt = (int(v) for v in r.stdout.split()[-2:])
    if kern_default == 2:
        assert xt == 0 and kern == 1   # the knob really selected the fixed ring
    assert np.array_equal(np.load(po), x_default)


def _e2e(ctx, torch, oracle_lib, band, sweeps, full=False, dense=False):
    cfg = band.cfg
    g = geom_of(band)
    out = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, sweeps, cfg.eps_mode,
                         full_grid=full, want_b=True, dense_stream=dense)
    st = ctx.stats()
    nk = out["n_keep"].cpu().numpy()
    keep = out["keep_idx"].cpu().numpy()
    x = out["x_map"].cpu().numpy()
    key = (cfg.name, cfg.n, tuple(int(b) for b in band.bins), sweeps, full)
    if key not in _ORACLE:   # one oracle run serves both kernels
        _ORACLE[key] = oracle_lib.solve_band_cfg(band, sweeps=sweeps, full_grid=full)
    rnk, rkeep, rx, rb = _ORACLE[key]
    for k in range(len(band.freqs)):
        assert rel_l2(out["b_map"][k].cpu().numpy(), rb[k]) < 1e-5
        assert nk[k] == rnk[k], (k, nk[k], rnk[k])
        assert np.array_equal(keep[k], rkeep[k])
        assert rel_l2(x[k], rx[k]) < TOL_X, (k, rel_l2(x[k], rx[k]))
        assert abs(x[k].sum() - rx[k].sum()) <= TOL_P * rx[k].sum()
        assert x[k].min() >= 0
    return st, nk


def test_gs_residual_cluster_of_3(ctx, torch_cuda, oracle_lib):
    """S~ = 12000 (12000 padded points: a wide cluster of 3 CTAs, 3 x 4000 columns of r) on the
    residual kernel against the oracle."""
    torch = torch_cuda
    A, bt = cfg5_system(oracle_lib, 12000)
    ref = oracle_lib.gs(A, bt, 12)
    x = ctx.gs(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(bt).cuda(), 12,
               dense_stream=False).cpu().numpy()
    st = ctx.stats()
    assert st["gs_kernel"] == 4 and st["gs_max_group"] == 3
    assert x.min() >= 0
    assert rel_l2(x, ref) < TOL_X, rel_l2(x, ref)
    assert abs(x.sum() - ref.sum()) < TOL_P * ref.sum()


def test_e2e_cfg5_mixed_cluster_classes(ctx, torch_cuda, oracle_lib):
    """One cfg5 band with three residual launch classes (S~ ~ 1.6k: one CTA; 3.3k: one CTA with
    wide registers; 8.6k: a wide cluster of 2), the classes concurrently on forked streams, 20
    sweeps."""
    band = synth.make_band("cfg5", bins=[300, 600, 1023])
    st, nk = _e2e(ctx, torch_cuda, oracle_lib, band, 20)
    assert st["gs_kernel"] == 4 and st["gs_max_group"] == 2
    sps = sorted((int(v) + 31) // 32 * 32 for v in nk)
    assert sps[0] <= 2560 < sps[1] <= 5120 < sps[2] and resid_ctas(nk.max(), wide=True) == 2


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_e2e_cfg5_largest_bins(ctx, torch_cuda, oracle_lib, dense):
    """cfg5's three largest bins (11.2-12 kHz, S~ ~ 8-9k of 40401) at 20 sweeps, in one call."""
    band = synth.make_band("cfg5", bins=[1000, 1012, 1023])
    st, nk = _e2e(ctx, torch_cuda, oracle_lib, band, 20, dense=dense)
    assert nk.min() > 6000
    assert st["gs_kernel"] == (2 if dense else 4)
    assert dense or st["gs_max_group"] == 2   # (the residual kernel's wide cluster mode)


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_e2e_cfg4_full_grid_n47(ctx, torch_cuda, oracle_lib, dense):
    """Full-grid mode on cfg4's array at n = 47 (S = 2209, T = 70 row blocks): three bins."""
    cfg = dataclasses.replace(synth.CONFIGS["cfg4"], n=47, n_bins=3)
    band = synth.make_band(cfg)
    st, nk = _e2e(ctx, torch_cuda, oracle_lib, band, 30, full=True, dense=dense)
    assert np.all(nk == 47 * 47)


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_e2e_cfg4_full_grid_defining_size(ctx, torch_cuda, oracle_lib, dense):
    """Full-grid mode at cfg4's own size (n = 101, S = 10201, A~ 416 MB per bin): one bin of the
    band (8 kHz), 10 sweeps; the oracle builds the dense 10201 x 10201 PSF."""
    band = synth.make_band("cfg4", bins=[63])
    st, nk = _e2e(ctx, torch_cuda, oracle_lib, band, 10, full=True, dense=dense)
    assert nk[0] == 10201
    assert st["gs_kernel"] == (2 if dense else 4)
    assert dense or st["gs_max_group"] == 4


def test_automatic_kernel_choice(ctx, torch_cuda, tmp_path):
    """Without a kernel flag the band's largest system picks the GS kernel: the residual kernel up
    to 20480 padded points -- cfg3's compressed bins on one CTA each, a full-grid band of S = 6400
    on (narrow) clusters of 3 -- and above that the dense-stream cluster kernel (checked in a subprocess
    with the threshold lowered to 2048 by DWC_RGS_AUTO_MAX_SP: a full-grid band of S = 2209);
    both flags at once are rejected."""
    torch = torch_cuda
    from paper_1608_05179_b200 import DwcError  # noqa: F401
    band = synth.make_band("cfg3", bins=[0, 255])
    cfg = band.cfg
    ctx.solve_band(geom_of(band), band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, 5)
    assert ctx.stats()["gs_kernel"] == 4 and ctx.stats()["gs_max_group"] == 1
    cfg4 = dataclasses.replace(synth.CONFIGS["cfg4"], n=80, n_bins=1)
    b4 = synth.make_band(cfg4)
    ctx.solve_band(geom_of(b4), b4.freqs, torch.from_numpy(b4.csm).cuda(), cfg4.epsilon, 3, full_grid=True)
    assert ctx.stats()["gs_kernel"] == 4 and ctx.stats()["gs_max_group"] == 3
    script = _AUTO_SCRIPT.format(root=ROOT)
    env = dict(os.environ, DWC_RGS_AUTO_MAX_SP="2048")
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert int(r.stdout.split()[-1]) in (1, 2)
    import ctypes as C

    from paper_1608_05179_b200.dwc import Params, lib
    g = geom_of(band)
    arr, grid = g.c_array(), g.c_grid()
    nk = torch.empty(2, dtype=torch.int32, device="cuda")
    keep = torch.empty((2, g.S), dtype=torch.int32, device="cuda")
    x = torch.empty((2, g.S), dtype=torch.float32, device="cuda")
    f = np.array(band.freqs, dtype=np.float64)
    csm = torch.from_numpy(band.csm).cuda()
    rc = lib().dwc_solve_band(ctx._h, C.byref(arr), C.byref(grid), C.byref(Params(cfg.epsilon, 0, 5, 16 | 32)), 2,
                              f.ctypes.data, csm.data_ptr(), nk.data_ptr(), keep.data_ptr(), x.data_ptr(), None, None,
                              torch.cuda.current_stream().cuda_stream)
    assert rc == -1
    A8 = torch.eye(8, dtype=torch.float32).cuda()
    b8 = torch.ones(8, dtype=torch.float64).cuda()
    x8 = torch.empty(8, dtype=torch.float32).cuda()
    assert lib().dwc_gs(ctx._h, 8, A8.data_ptr(), b8.data_ptr(), 1, 16 | 32, x8.data_ptr(), None) == -1


_AUTO_SCRIPT = r"""
import dataclasses, sys, torch
sys.path.insert(0, {root!r})
import synth
from paper_1608_05179_b200 import Context, Geometry
cfg4 = dataclasses.replace(synth.CONFIGS["cfg4"], n=47, n_bins=1)
b4 = synth.make_band(cfg4)
g = Geometry(b4.mic_xyz, cfg4.n, cfg4.side_len, cfg4.z0, cfg4.c0, cfg4.cx, cfg4.cy)
c = Context(0)
c.solve_band(g, b4.freqs, torch.from_numpy(b4.csm).cuda(), cfg4.epsilon, 3, full_grid=True)
print(c.stats()["gs_kernel"])
"""


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "alt_kernel"])
def test_gs_large_alternating(ctx, torch_cuda, oracle_lib, dense):
    """Alternating sweep directions (R21) on an S~ = 4500 system: the residual kernel's cluster
    mode (2 CTAs, the alternating visit sequence across CTAs) and the one-CTA-per-bin kernel."""
    torch = torch_cuda
    A, bt = cfg5_system(oracle_lib, 4500)
    ref = oracle_lib.gs(A, bt, 21, alt=True)
    x = ctx.gs(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(bt).cuda(), 21, alt=True,
               dense_stream=dense).cpu().numpy()
    st = ctx.stats()
    assert st["gs_kernel"] == (3 if dense else 4) and (dense or st["gs_max_group"] == 1)
    assert x.min() >= 0
    assert rel_l2(x, ref) < TOL_X, rel_l2(x, ref)
    assert abs(x.sum() - ref.sum()) < TOL_P * ref.sum()


def test_gs_large_general_matrix(ctx, torch_cuda, oracle_lib):
    """The paper-literal (asymmetric) PSF of an S~ = 3000 system in cfg5's geometry: the residual
    kernel's cluster mode on the transposed store, against the oracle's Eq. 13-14 loop."""
    torch = torch_cuda
    band = synth.make_band("cfg5", bins=[1023])
    g = geom_of(band)
    f = band.freqs[0]
    b_full = oracle_lib.das_paper(*oracle_args(g), f, band.csm[0])
    keep = np.sort(np.argsort(-b_full)[:3000]).astype(np.int32)
    A = oracle_lib.psf_paper(*oracle_args(g), f, keep)
    bt = b_full[keep]
    ref = oracle_lib.gs(A, bt, 20)
    x = ctx.gs(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(bt).cuda(), 20,
               general=True).cpu().numpy()
    st = ctx.stats()
    assert st["gs_kernel"] == 4 and st["gs_max_group"] == 1   # (one CTA, wide registers)
    assert x.min() >= 0
    assert rel_l2(x, ref) < TOL_X, rel_l2(x, ref)
    assert abs(x.sum() - ref.sum()) < TOL_P * ref.sum()


_SMEM_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1608_05179_b200 import Context
c = Context(0)
out = {{}}
for name, alt in (("fwd", False), ("alt", True)):
    A = np.load({a!r}); b = np.load({b!r})
    x = c.gs(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), 15, alt=alt, dense_stream=False).cpu().numpy()
    out[name] = x
    out[name + "_k"] = np.array([c.stats()["gs_kernel"], c.stats()["gs_max_group"]])
np.savez({o!r}, **out)
"""


def test_gs_residual_shared_memory_path(oracle_lib, tmp_path):
    """The residual kernel with r in shared memory (the path for systems whose rows do not fit a
    ring slot; forced here by DWC_RGS_NO_REGR in a separate process): an S~ = 2100 system,
    forward and alternating sweeps, against the oracle."""
    A, bt = cfg5_system(oracle_lib, 2100)
    pa, pb, po = tmp_path / "A.npy", tmp_path / "b.npy", tmp_path / "x.npz"
    np.save(pa, A.astype(np.float32))
    np.save(pb, bt)
    script = _SMEM_SCRIPT.format(root=ROOT, a=str(pa), b=str(pb), o=str(po))
    env = dict(os.environ, DWC_RGS_NO_REGR="1")
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = np.load(po)
    for name, alt in (("fwd", False), ("alt", True)):
        assert list(res[name + "_k"]) == [4, 1]
        ref = oracle_lib.gs(A, bt, 15, alt=alt)
        x = res[name]
        assert x.min() >= 0
        assert rel_l2(x, ref) < TOL_X, (name, rel_l2(x, ref))
        assert abs(x.sum() - ref.sum()) < TOL_P * ref.sum()
