"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by
element on the same seeded inputs (north_star tolerances):
  keep set bit-exact; b and A within 1e-5 relative L2; x_map within 1e-3 relative L2;
  integrated power within 1e-3."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

TOL_B = 1e-5
TOL_A = 1e-5
TOL_X = 1e-3
TOL_P = 1e-3


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


def small_geom(m=16, n=13, arms=2):
    from paper_1608_05179_b200 import Geometry
    return Geometry(synth.spiral_array(m, 0.6, arms), n, 1.2, 0.9, 343.0, 0.03, -0.02)


# ---------------------------------------------------------------------------- S1
def test_steer_parity(ctx, torch_cuda, oracle_lib):
    torch = torch_cuda
    g = small_geom()
    idx = np.array([0, 1, 5, 77, g.S - 1], dtype=np.int32)
    E = ctx.steer(g, 4321.0, torch.from_numpy(idx).cuda()).cpu().numpy()
    ref = oracle_lib.steering(*oracle_args(g), 4321.0, idx)
    assert np.max(np.abs(E - ref)) < 1e-12


# ---------------------------------------------------------------------------- S2
@pytest.mark.parametrize("cfgname", ["cfg1", "cfg2"])
def test_das_parity(ctx, torch_cuda, oracle_lib, cfgname):
    torch = torch_cuda
    band = synth.make_band(cfgname)
    g = geom_of(band)
    b = ctx.das(g, band.freqs, torch.from_numpy(band.csm).cuda()).cpu().numpy()
    for k in range(len(band.freqs)):
        ref = oracle_lib.das(*oracle_args(g), band.freqs[k], band.csm[k])
        assert rel_l2(b[k], ref) < 1e-12          # fp64 both sides (<< the 1e-5 bar)
        assert rel_l2(b[k], ref) < TOL_B


@pytest.mark.parametrize("m", [2, 13, 64, 128, 208, 216, 300, 512])
def test_das_odd_sizes_and_non_hermitian(ctx, torch_cuda, oracle_lib, m):
    """Ragged mic counts (chunk tails) and a non-Hermitian CSM: only its Hermitian part
    matters (reading R3), so GPU == oracle's full quadratic form."""
    torch = torch_cuda
    from paper_1608_05179_b200 import Geometry
    rng = np.random.default_rng(m)
    g = Geometry(rng.uniform(-0.4, 0.4, size=(m, 3)) * [1, 1, 0], 9, 1.0, 1.0, 343.0)
    C = rng.standard_normal((2, m, m)) + 1j * rng.standard_normal((2, m, m))
    freqs = np.array([900.0, 7300.0])
    b = ctx.das(g, freqs, torch.from_numpy(C).cuda()).cpu().numpy()
    for k in range(2):
        ref = oracle_lib.das(*oracle_args(g), freqs[k], C[k])
        assert np.max(np.abs(b[k] - ref)) < 1e-12 * np.max(np.abs(ref))


# ---------------------------------------------------------------------------- S3/S4
def _compress_both(ctx, torch, g, bmaps, eps, mode=0, full=False, order=1):
    nk, keep, lev = ctx.compress(g, torch.from_numpy(np.ascontiguousarray(bmaps)).cuda(), eps, mode, full,
                                 order=order, want_level=True)
    nk, keep, lev = nk.cpu().numpy(), keep.cpu().numpy(), lev.cpu().numpy()
    import oracle as orc
    for k in range(bmaps.shape[0]):
        rk, rlev, _, _ = orc.compress(g.n, bmaps[k], eps, mode, full, order=order)
        assert nk[k] == len(rk)
        assert np.array_equal(keep[k, : nk[k]], rk)
        assert np.all(keep[k, nk[k]:] == -1)
        assert np.array_equal(lev[k], rlev)
    return nk


def test_compress_bit_exact_on_oracle_maps(ctx, torch_cuda, oracle_lib):
    """Stage test (i): the same fp64 b into both compressors -> identical keep sets."""
    torch = torch_cuda
    band = synth.make_band("cfg2")
    g = geom_of(band)
    bm = np.stack([oracle_lib.das(*oracle_args(g), f, c) for f, c in zip(band.freqs, band.csm)])
    for eps in [band.cfg.epsilon, 0.001, 0.05, 0.3]:
        _compress_both(ctx, torch, g, bm, eps)
    # absolute mode, full grid
    _compress_both(ctx, torch, g, bm, 0.01 * bm.max(), mode=1)
    nk = _compress_both(ctx, torch, g, bm, 0.5, full=True)
    assert np.all(nk == g.S)


@pytest.mark.parametrize("order", [1, 3])
def test_compress_cubic_bit_exact_on_oracle_maps(ctx, torch_cuda, oracle_lib, order):
    """NEXT-1: the cubic (4-point) predictor, same stage protocol (bit-exact keep sets)."""
    torch = torch_cuda
    for cfgname in ("cfg1", "cfg2"):
        band = synth.make_band(cfgname)
        g = geom_of(band)
        bm = np.stack([oracle_lib.das(*oracle_args(g), f, c) for f, c in zip(band.freqs, band.csm)])
        for eps in [band.cfg.epsilon, 0.002, 0.05]:
            _compress_both(ctx, torch, g, bm, eps, order=order)


@pytest.mark.parametrize("order", [1, 3])
@pytest.mark.parametrize("n", [2, 3, 5, 6, 8, 17, 20, 33, 64, 101])
def test_compress_edge_grids(ctx, torch_cuda, n, order):
    """Dyadic and non-dyadic N, tiny grids, random maps with ties, constant and zero maps."""
    torch = torch_cuda
    from paper_1608_05179_b200 import Geometry
    g = Geometry(np.zeros((2, 3)), n, 1.0, 1.0)
    rng = np.random.default_rng(n)
    maps = [rng.random(n * n), np.full(n * n, 2.5), np.zeros(n * n),
            np.round(rng.random(n * n) * 4) / 4]          # many exact ties at |d| == eps_eff
    bm = np.stack(maps)
    for eps in [0.125, 0.25, 0.01]:
        _compress_both(ctx, torch, g, bm, eps, order=order)
    _compress_both(ctx, torch, g, bm, 0.25, mode=1, order=order)


# ---------------------------------------------------------------------------- S5
@pytest.mark.parametrize("cfgname,bin_", [("cfg1", 0), ("cfg2", 0), ("cfg2", 7), ("cfg3", 200)])
def test_psf_parity_on_oracle_keep(ctx, torch_cuda, oracle_lib, cfgname, bin_):
    torch = torch_cuda
    band = synth.make_band(cfgname, bins=[bin_])
    g = geom_of(band)
    f = band.freqs[0]
    b = oracle_lib.das(*oracle_args(g), f, band.csm[0])
    keep, *_ = oracle_lib.compress(g.n, b, band.cfg.epsilon)
    A = ctx.psf(g, f, torch.from_numpy(keep).cuda()).cpu().numpy()
    ref = oracle_lib.psf(*oracle_args(g), f, keep)
    assert rel_l2(A, ref) < TOL_A
    assert rel_l2(A, ref) < 1e-7          # fp32-accurate (the fp64 PSF rounded to fp32)
    assert np.max(np.abs(A - A.T)) == 0.0
    assert np.max(np.abs(np.diag(A) - 1)) < 1e-6


@pytest.mark.parametrize("m,n,nk", [(24, 15, 1), (24, 15, 2), (24, 15, 31), (24, 15, 32), (24, 15, 33),
                                    (24, 15, 64), (24, 15, 65), (24, 15, 127), (24, 15, 128), (24, 15, 129),
                                    (24, 15, 200), (13, 15, 100), (5, 15, 40), (128, 21, 300), (128, 21, 441),
                                    (200, 15, 150), (512, 21, 300), (64, 47, 2000)])
def test_psf_ragged_sizes(ctx, torch_cuda, oracle_lib, m, n, nk):
    """Ragged S~ (one tile, tile edges, several 128x32 tiles + tail), odd M (K padding), K
    steps wrapping the operand ring inside a tile (M = 200: 13 steps; M = 512 = DWC_MAX_MICS:
    32 steps, the largest int32 level sums), and more tiles than CTAs (nk = 2000: every CTA
    of the persistent kernel runs several tiles through both TMEM buffers)."""
    torch = torch_cuda
    g = small_geom(m, n, 3 if m % 3 == 0 else 1)
    keep = np.sort(np.random.default_rng(nk).choice(g.S, size=nk, replace=False)).astype(np.int32)
    A = ctx.psf(g, 5100.0, torch.from_numpy(keep).cuda()).cpu().numpy()
    ref = oracle_lib.psf(*oracle_args(g), 5100.0, keep)
    assert rel_l2(A, ref) < TOL_A
    # the int8-digit tensor-core Gram is exact to ~1e-9: A is the fp64 PSF rounded to fp32
    assert rel_l2(A, ref) < 1e-7
    assert np.max(np.abs(A - ref)) <= 2.0 ** -23
    assert np.array_equal(A, A.T)


# ---------------------------------------------------------------------------- S7
def test_gs_identity_and_scalar(ctx, torch_cuda):
    torch = torch_cuda
    b = np.array([0.5, -1.0, 2.0, 0.0, 3.0])
    x = ctx.gs(torch.eye(5, dtype=torch.float32).cuda(), torch.from_numpy(b).cuda(), 1).cpu().numpy()
    assert np.array_equal(x, np.maximum(b, 0).astype(np.float32))
    x = ctx.gs(torch.tensor([[4.0]]).cuda(), torch.tensor([3.0], dtype=torch.float64).cuda(), 3).cpu().numpy()
    assert x[0] == 0.75


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
@pytest.mark.parametrize("nk,sweeps", [(1, 5), (2, 7), (31, 50), (32, 50), (33, 50), (64, 40), (65, 40), (97, 200),
                                       (300, 1000), (447, 80), (448, 80), (640, 80), (831, 60), (832, 60),
                                       (1000, 100), (1190, 60)])
def test_gs_parity_on_oracle_system(ctx, torch_cuda, oracle_lib, nk, sweeps, dense):
    """GS on the oracle's own A~ (rounded to fp32) and b~: ragged sizes around the 32-row
    block and multi-block systems, both sides of the CTAs-per-bin thresholds (g = 1 below 448
    kept points, 2 from 448, 4 from 832) and a g = 4 system whose T = 38 blocks end inside the
    18-block column-ownership period."""
    torch = torch_cuda
    band = synth.make_band("cfg3", bins=[150])
    g = geom_of(band)
    f = band.freqs[0]
    b = oracle_lib.das(*oracle_args(g), f, band.csm[0])
    order = np.argsort(-b)[:nk]
    keep = np.sort(order).astype(np.int32)
    A = oracle_lib.psf(*oracle_args(g), f, keep)
    bt = b[keep]
    ref = oracle_lib.gs(A, bt, sweeps)
    x = ctx.gs(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(bt).cuda(), sweeps,
               dense_stream=dense).cpu().numpy()
    assert ctx.stats()["gs_kernel"] == (1 if dense else 4) or (dense and ctx.stats()["gs_kernel"] == 2)
    assert x.min() >= 0
    assert rel_l2(x, ref) < TOL_X
    assert abs(x.sum() - ref.sum()) < TOL_P * ref.sum()


@pytest.mark.parametrize("nk", [2, 300, 1086])
def test_gs_nonneg_widening_is_bitwise_exact(ctx, torch_cuda, oracle_lib, nk):
    """The residual kernel widens a non-negative A~ by bit placement (f * 2^-896, the 2^896 in
    dx) instead of F2F; a -0.0 in the lower triangle (never read by the symmetric solve, but seen
    by dwc_gs's sign scan) forces the F2F path on the same system: the iterates must be
    bitwise identical."""
    torch = torch_cuda
    band = synth.make_band("cfg3", bins=[249])
    g = geom_of(band)
    f = band.freqs[0]
    b = oracle_lib.das(*oracle_args(g), f, band.csm[0])
    keep = np.sort(np.argsort(-b)[:nk]).astype(np.int32)
    A = oracle_lib.psf(*oracle_args(g), f, keep).astype(np.float32)
    bt = torch.from_numpy(b[keep]).cuda()
    x_nn = ctx.gs(torch.from_numpy(A).cuda(), bt, 200, dense_stream=False).cpu().numpy()
    A2 = A.copy()
    A2[nk - 1, 0] = -0.0
    x_f2f = ctx.gs(torch.from_numpy(A2).cuda(), bt, 200, dense_stream=False).cpu().numpy()
    assert np.array_equal(x_nn, x_f2f)


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
@pytest.mark.parametrize("n", [40, 333])
def test_gs_signed_matrix_parity(ctx, torch_cuda, oracle_lib, n, dense):
    """A symmetric positive-definite matrix with negative off-diagonal entries (dwc_gs accepts
    any A with A_ii > 0): the residual kernel's F2F widening path, against the oracle."""
    torch = torch_cuda
    rng = np.random.default_rng(n)
    B = rng.standard_normal((n, n // 2))
    A = B @ B.T / n + np.diag(1.0 + rng.random(n))
    A /= np.sqrt(np.outer(np.diag(A), np.diag(A)))   # unit diagonal, like the PSF
    A = A.astype(np.float32).astype(np.float64)
    assert A.min() < 0
    bt = A @ np.abs(rng.standard_normal(n)) - 0.05
    ref = oracle_lib.gs(A, bt, 150)
    x = ctx.gs(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(bt).cuda(), 150,
               dense_stream=dense).cpu().numpy()
    assert x.min() >= 0
    assert rel_l2(x, ref) < TOL_X, rel_l2(x, ref)


# ---------------------------------------------------------------------------- end to end
def _e2e(ctx, torch, oracle_lib, band, sweeps=None, full=False, check_b=True, order=1, dr=False, alt=False,
         dense=False):
    cfg = band.cfg
    g = geom_of(band)
    sw = sweeps or cfg.sweeps
    out = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, sw, cfg.eps_mode,
                         full_grid=full, want_b=True, order=order, dr=dr, alt=alt, dense_stream=dense)
    kern = ctx.stats()["gs_kernel"]
    assert kern == ((3 if dense else 4) if alt else (4 if not dense else kern)) and kern != 0
    nk = out["n_keep"].cpu().numpy()
    keep = out["keep_idx"].cpu().numpy()
    x = out["x_map"].cpu().numpy()
    bm = out["b_map"].cpu().numpy()
    rnk, rkeep, rx, rb = oracle_lib.solve_band_cfg(band, sweeps=sw, full_grid=full, order=order, dr=dr, alt=alt)
    for k in range(len(band.freqs)):
        assert rel_l2(bm[k], rb[k]) < TOL_B
        assert nk[k] == rnk[k], (k, nk[k], rnk[k])
        assert np.array_equal(keep[k], rkeep[k])
        assert rel_l2(x[k], rx[k]) < TOL_X, (k, rel_l2(x[k], rx[k]))
        assert abs(x[k].sum() - rx[k].sum()) <= TOL_P * rx[k].sum()
        assert x[k].min() >= 0
    return out


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_e2e_cfg1_compressed_and_full(ctx, torch_cuda, oracle_lib, dense):
    band = synth.make_band("cfg1")
    _e2e(ctx, torch_cuda, oracle_lib, band, dense=dense)
    _e2e(ctx, torch_cuda, oracle_lib, band, full=True, dense=dense)


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_e2e_cfg2_all_bins(ctx, torch_cuda, oracle_lib, dense):
    _e2e(ctx, torch_cuda, oracle_lib, synth.make_band("cfg2"), dense=dense)


def test_e2e_cfg2_cubic_predictor(ctx, torch_cuda, oracle_lib):
    """NEXT-1 end to end: the cubic predictor changes the kept set; every tolerance holds."""
    _e2e(ctx, torch_cuda, oracle_lib, synth.make_band("cfg2"), order=3)


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_e2e_cfg3_strided_bins(ctx, torch_cuda, oracle_lib, dense):
    band = synth.make_band("cfg3", bins=synth.strided_bins(256, 6))
    _e2e(ctx, torch_cuda, oracle_lib, band, dense=dense)


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_e2e_full_grid_m128(ctx, torch_cuda, oracle_lib, dense):
    """Full-grid mode (cfg4's 128-mic array, exact CSM) on a 31x31 grid the oracle can
    build the dense S x S PSF for; several 32-row blocks and a ragged tail (961 = 30*32+1)."""
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["cfg4"], n=31, n_bins=3)
    band = synth.make_band(cfg)
    _e2e(ctx, torch_cuda, oracle_lib, band, sweeps=60, full=True, dense=dense)


def test_e2e_max_mics(ctx, torch_cuda, oracle_lib):
    """The whole path at DWC_MAX_MICS = 512 microphones (the DAS form with 16 points per CTA, the
    PSF with 32 K steps of int8 digits): two bins on a 15 x 15 grid, 60 sweeps."""
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"], m=512, arms=8, n=15, n_bins=2, snapshots=600)
    band = synth.make_band(cfg)
    _e2e(ctx, torch_cuda, oracle_lib, band, sweeps=60)


def test_e2e_cfg5_strided_bins_few_sweeps(ctx, torch_cuda, oracle_lib):
    """cfg5 geometry (M=128, 201x201 grid, 10 dB SNR) on two low bins, 20 sweeps."""
    band = synth.make_band("cfg5", bins=[10, 120])
    _e2e(ctx, torch_cuda, oracle_lib, band, sweeps=20)


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_full_size_cfg3_sampled(ctx, torch_cuda, oracle_lib, dense):
    """BASELINE configs[2] at full size in the bench's launch configuration (all 256 bins in
    one call); the oracle recomputes a strided sample of 8 bins one by one."""
    torch = torch_cuda
    cfg = synth.CONFIGS["cfg3"]
    band = synth.make_band(cfg)
    g = geom_of(band)
    out = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, cfg.sweeps,
                         dense_stream=dense)
    if not dense:   # more bins than SMs: the systems of at most half the largest size ran two per SM
        assert ctx.stats()["gs_kernel"] == 4 and ctx.stats()["gs_ctas"] > 148
    nk = out["n_keep"].cpu().numpy()
    keep = out["keep_idx"].cpu().numpy()
    x = out["x_map"].cpu().numpy()
    sample = synth.strided_bins(256, 8)
    sub = synth.make_band(cfg, bins=sample)
    rnk, rkeep, rx, _ = oracle_lib.solve_band_cfg(sub)
    for j, k in enumerate(sample):
        assert nk[k] == rnk[j] and np.array_equal(keep[k], rkeep[j])
        assert rel_l2(x[k], rx[j]) < TOL_X
        assert abs(x[k].sum() - rx[j].sum()) <= TOL_P * rx[j].sum()


def test_host_api_equals_device_api_and_deterministic(ctx, torch_cuda):
    torch = torch_cuda
    band = synth.make_band("cfg2", bins=[1, 4, 6])
    g = geom_of(band)
    cfg = band.cfg
    d1 = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, 200, want_b=True)
    d2 = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, 200, want_b=True)
    h = ctx.solve_band_host(g, band.freqs, torch.from_numpy(band.csm).pin_memory(), cfg.epsilon, 200, want_b=True)
    # pinned outputs take the early keep-set readback (on a copy stream, overlapping S5-S7)
    K, S = len(band.freqs), g.S
    pin = {"n_keep": torch.full((K,), -7, dtype=torch.int32).pin_memory(),
           "keep_idx": torch.full((K, S), -7, dtype=torch.int32).pin_memory(),
           "x_map": torch.empty((K, S), dtype=torch.float32).pin_memory(),
           "b_map": torch.empty((K, S), dtype=torch.float64).pin_memory()}
    hp = ctx.solve_band_host(g, band.freqs, torch.from_numpy(band.csm).pin_memory(), cfg.epsilon, 200,
                             want_b=True, out=pin)
    for key in ["n_keep", "keep_idx", "x_map", "b_map"]:
        a = d1[key].cpu()
        assert torch.equal(a, d2[key].cpu())
        assert torch.equal(a, h[key])
        assert torch.equal(a, hp[key])


def test_shard_invariance(ctx, torch_cuda):
    """Per-bin outputs do not depend on which other bins share the call (the property the
    multi-GPU strided sharding relies on): bins solved in a batch == bins solved alone."""
    torch = torch_cuda
    band = synth.make_band("cfg2")
    g = geom_of(band)
    cfg = band.cfg
    full = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, 300)
    for k in [0, 3, 7]:
        one = ctx.solve_band(g, band.freqs[k:k + 1], torch.from_numpy(band.csm[k:k + 1]).cuda(), cfg.epsilon, 300)
        assert torch.equal(one["x_map"][0], full["x_map"][k])
        assert torch.equal(one["keep_idx"][0], full["keep_idx"][k])


def test_errors(ctx, torch_cuda):
    torch = torch_cuda
    from paper_1608_05179_b200 import DwcError, Geometry
    band = synth.make_band("cfg1")
    g = geom_of(band)
    csm = torch.from_numpy(band.csm).cuda()
    with pytest.raises(DwcError) as e:
        ctx.solve_band(g, band.freqs, csm, -1.0, 10)
    assert e.value.code == -1
    with pytest.raises(DwcError) as e:
        ctx.solve_band(g, band.freqs, csm, 0.1, 0)
    assert e.value.code == -1
    with pytest.raises(DwcError) as e:
        ctx.solve_band(g, -band.freqs, csm, 0.1, 10)
    assert e.value.code == -1
    bad = Geometry(g.mic_xyz, 1, 1.0, 1.0)
    with pytest.raises(DwcError):
        ctx.solve_band(bad, band.freqs, torch.zeros((1, 16, 16), dtype=torch.complex128).cuda(), 0.1, 10)
    nan = csm.clone()
    nan[0, 0, 0] = float("nan")
    with pytest.raises(DwcError) as e:
        ctx.solve_band(g, band.freqs, nan, 0.1, 10)
    assert e.value.code == -3
    # a grid node on a microphone -> singular
    mic = np.array([[0.0, 0.0, 1.0], [0.2, 0.1, 0.0]])
    gs = Geometry(mic, 3, 1.0, 1.0)
    with pytest.raises(DwcError) as e:
        ctx.solve_band(gs, [1000.0], torch.eye(2, dtype=torch.complex128).reshape(1, 2, 2).cuda(), 0.1, 5)
    assert e.value.code == -2
    # the context still works after errors
    ctx.solve_band(g, band.freqs, csm, 0.1, 5)


# ---------------------------------------------------------------------------- NEXT-3: Eq. 1 on device
@pytest.mark.parametrize("m,I", [(16, 1), (13, 37), (64, 1000), (128, 100)])
def test_csm_parity(ctx, torch_cuda, oracle_lib, m, I):
    """C = (1/I) sum_i p_i p_i^H in fp64 on the GPU vs the oracle's loops (odd M, ragged I)."""
    torch = torch_cuda
    rng = np.random.default_rng(m * 1000 + I)
    snap = rng.standard_normal((3, m, I)) + 1j * rng.standard_normal((3, m, I))
    C = ctx.csm(torch.from_numpy(snap).cuda()).cpu().numpy()
    ref = oracle_lib.csm(snap)
    assert np.abs(C - ref).max() <= 1e-13 * np.abs(ref).max()


def test_e2e_from_snapshots_cfg2(ctx, torch_cuda, oracle_lib):
    """The whole path from snapshot spectra (Eq. 1 on device) vs the oracle's Eq. 1 + path."""
    torch = torch_cuda
    bins = [0, 3, 7]
    band = synth.make_band("cfg2", bins=bins)
    snap = synth.make_snapshots("cfg2", bins=bins)
    cfg = band.cfg
    g = geom_of(band)
    out = ctx.solve_band_snapshots(g, band.freqs, torch.from_numpy(snap).cuda(), cfg.epsilon, cfg.sweeps,
                                   want_b=True)
    import dataclasses
    ob = dataclasses.replace(band, csm=oracle_lib.csm(snap))
    rnk, rkeep, rx, rb = oracle_lib.solve_band_cfg(ob)
    for k in range(len(bins)):
        assert rel_l2(out["b_map"][k].cpu().numpy(), rb[k]) < TOL_B
        assert np.array_equal(out["keep_idx"][k].cpu().numpy(), rkeep[k])
        x = out["x_map"][k].cpu().numpy()
        assert rel_l2(x, rx[k]) < TOL_X
        assert abs(x.sum() - rx[k].sum()) <= TOL_P * rx[k].sum()


# ---------------------------------------------------------------------------- NEXT-2: diagonal removal
@pytest.mark.parametrize("cfgname", ["cfg1", "cfg2"])
def test_das_dr_parity(ctx, torch_cuda, oracle_lib, cfgname):
    torch = torch_cuda
    band = synth.make_band(cfgname)
    g = geom_of(band)
    b = ctx.das(g, band.freqs, torch.from_numpy(band.csm).cuda(), dr=True).cpu().numpy()
    for k, (f, c) in enumerate(zip(band.freqs, band.csm)):
        ref = oracle_lib.das(*oracle_args(g), f, c, dr=True)
        assert rel_l2(b[k], ref) < TOL_B
        assert b[k].min() >= 0.0


@pytest.mark.parametrize("m,n,nk", [(24, 15, 65), (24, 15, 200), (128, 21, 300), (13, 15, 100)])
def test_psf_dr_parity(ctx, torch_cuda, oracle_lib, m, n, nk):
    torch = torch_cuda
    g = small_geom(m, n, 3 if m % 3 == 0 else 1)
    keep = np.sort(np.random.default_rng(nk).choice(g.S, size=nk, replace=False)).astype(np.int32)
    A = ctx.psf(g, 5100.0, torch.from_numpy(keep).cuda(), dr=True).cpu().numpy()
    ref = oracle_lib.psf(*oracle_args(g), 5100.0, keep, dr=True)
    assert rel_l2(A, ref) < TOL_A
    assert np.max(np.abs(A - ref)) <= 2.0 ** -22
    assert np.array_equal(A, A.T) and A.min() >= 0.0


def test_e2e_cfg2_diag_removal(ctx, torch_cuda, oracle_lib):
    """NEXT-2 end to end: cfg2's 20 dB noisy CSMs with the diagonal removed."""
    _e2e(ctx, torch_cuda, oracle_lib, synth.make_band("cfg2"), dr=True)


# ---------------------------------------------------------------------------- NEXT-4: alternating sweeps
@pytest.mark.parametrize("dense", [False, True], ids=["residual", "alt_kernel"])
@pytest.mark.parametrize("nk,sweeps", [(1, 3), (31, 40), (33, 41), (64, 30), (97, 31), (130, 100), (257, 61),
                                       (300, 200)])
def test_gs_alternating_parity(ctx, torch_cuda, oracle_lib, nk, sweeps, dense):
    """Alternating forward/backward sweeps (R21) on oracle PSF systems (odd sweep counts end on
    a forward sweep, even ones on a backward sweep): the residual kernel's visit sequence (T = 1,
    2, 3, 4, 5, 9, 10 blocks: turns inside and beyond its 7-block carry window) and the
    one-CTA-per-bin alternating kernel."""
    torch = torch_cuda
    g = small_geom(24, 19, 3)
    rng = np.random.default_rng(nk)
    keep = np.sort(rng.choice(g.S, size=nk, replace=False)).astype(np.int32)
    A = oracle_lib.psf(*oracle_args(g), 3000.0, keep)
    b = A @ np.abs(rng.standard_normal(nk)) + 0.01 * rng.standard_normal(nk)
    ref = oracle_lib.gs(A, b, sweeps, alt=True)
    x = ctx.gs(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(b).cuda(), sweeps,
               alt=True, dense_stream=dense).cpu().numpy()
    assert ctx.stats()["gs_kernel"] == (3 if dense else 4)
    assert x.min() >= 0
    assert rel_l2(x, ref) < TOL_X
    assert abs(x.sum() - ref.sum()) < TOL_P * ref.sum()


@pytest.mark.parametrize("dense", [False, True], ids=["residual", "alt_kernel"])
def test_e2e_cfg2_alternating_sweeps(ctx, torch_cuda, oracle_lib, dense):
    _e2e(ctx, torch_cuda, oracle_lib, synth.make_band("cfg2", bins=[0, 4, 7]), alt=True, dense=dense)


def test_e2e_cfg3_alternating_paper_mode(ctx, torch_cuda, oracle_lib):
    """Alternating sweeps with the paper-literal PSF (both NEXT-4 variants at once) on cfg3 bins."""
    torch = torch_cuda
    band = synth.make_band("cfg3", bins=[40, 160, 250])
    cfg = band.cfg
    g = geom_of(band)
    out = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, 200, cfg.eps_mode,
                         alt=True, paper=True)
    assert ctx.stats()["gs_kernel"] == 4
    rnk, rkeep, rx, _ = oracle_lib.solve_band_cfg(band, sweeps=200, alt=True, paper=True)
    for k in range(3):
        assert np.array_equal(out["keep_idx"][k].cpu().numpy(), rkeep[k])
        x = out["x_map"][k].cpu().numpy()
        assert rel_l2(x, rx[k]) < TOL_X, (k, rel_l2(x, rx[k]))
        assert abs(x.sum() - rx[k].sum()) <= TOL_P * rx[k].sum()


def test_errors_flags_and_new_entry_points(ctx, torch_cuda):
    """Unknown flag bits, bad snapshot counts, sizes over the on-chip capacity, bad stage flags."""
    torch = torch_cuda
    import ctypes as C

    from paper_1608_05179_b200 import DwcError
    from paper_1608_05179_b200.dwc import Array, Grid, Params, lib
    band = synth.make_band("cfg1")
    g = geom_of(band)
    csm = torch.from_numpy(band.csm).cuda()
    arr, grid = g.c_array(), g.c_grid()
    nk = torch.empty(1, dtype=torch.int32, device="cuda")
    keep = torch.empty((1, g.S), dtype=torch.int32, device="cuda")
    x = torch.empty((1, g.S), dtype=torch.float32, device="cuda")
    f = np.array(band.freqs, dtype=np.float64)
    prm = Params(0.1, 0, 5, 1 << 20)   # unknown flag bit
    rc = lib().dwc_solve_band(ctx._h, C.byref(arr), C.byref(grid), C.byref(prm), 1, f.ctypes.data,
                              csm.data_ptr(), nk.data_ptr(), keep.data_ptr(), x.data_ptr(), None, None,
                              torch.cuda.current_stream().cuda_stream)
    assert rc == -1 and b"flags" in lib().dwc_last_error()
    with pytest.raises(DwcError):
        ctx.solve_band_snapshots(g, band.freqs, torch.zeros((1, 16, 0), dtype=torch.complex128).cuda(), 0.1, 5)
    with pytest.raises(DwcError):   # S~ beyond the GS kernel's on-chip x capacity (rejected before any launch)
        n = 20000
        ctx.gs(torch.zeros((n, n), dtype=torch.float32).cuda(), torch.zeros(n, dtype=torch.float64).cuda(), 1)
    # A_ii <= 0 -> DWC_ENUMERIC, detected on the device before any sweep
    Abad = torch.eye(40, dtype=torch.float32).cuda()
    Abad[17, 17] = 0.0
    with pytest.raises(DwcError) as ei:
        ctx.gs(Abad, torch.ones(40, dtype=torch.float64).cuda(), 3)
    assert ei.value.code == -3
    Abad[17, 17] = float("nan")
    with pytest.raises(DwcError):
        ctx.gs(Abad, torch.ones(40, dtype=torch.float64).cuda(), 3)
    # keep masks: n_bins 0 is a no-op, S < 1 rejected
    assert lib().dwc_keep_mask(ctx._h, 0, 10, None, None, None, None) == 0
    assert lib().dwc_keep_mask(ctx._h, 1, 0, nk.data_ptr(), keep.data_ptr(), x.data_ptr(), None) == -1
    # the context still works
    ctx.solve_band(g, band.freqs, csm, 0.1, 5, dr=True, order=3)


# ---------------------------------------------------------------------------- degenerate inputs
@pytest.mark.gpu
def test_zero_csm_bin_in_a_batch(ctx, torch_cuda, oracle_lib):
    """A bin with C = 0 (max|b| = 0, reading R6): b = 0, only the coarsest level G^0 is kept and
    x = 0; the other bins of the same batch are bit-identical to solving them alone."""
    torch = torch_cuda
    band = synth.make_band("cfg2", bins=[0, 3, 6])
    cfg = band.cfg
    g = geom_of(band)
    csm = band.csm.copy()
    csm[1] = 0.0
    out = ctx.solve_band(g, band.freqs, torch.from_numpy(csm).cuda(), cfg.epsilon, 200, cfg.eps_mode, want_b=True)
    nk = out["n_keep"].cpu().numpy()
    keep = out["keep_idx"].cpu().numpy()
    n = cfg.n
    J = int(np.floor(np.log2(n)))
    h = 2 ** J
    g0 = sorted(r * n + c for r in range(0, n, h) for c in range(0, n, h))
    assert nk[1] == len(g0) == 4
    assert list(keep[1][:4]) == g0 and np.all(keep[1][4:] == -1)
    assert np.all(out["x_map"].cpu().numpy()[1] == 0.0)
    assert np.all(out["b_map"].cpu().numpy()[1] == 0.0)
    for k in (0, 2):
        solo = ctx.solve_band(g, band.freqs[k:k + 1], torch.from_numpy(band.csm[k:k + 1]).cuda(), cfg.epsilon, 200,
                              cfg.eps_mode)
        assert nk[k] == solo["n_keep"].cpu().numpy()[0]
        assert np.array_equal(out["x_map"].cpu().numpy()[k], solo["x_map"].cpu().numpy()[0])


@pytest.mark.gpu
def test_absolute_threshold_mode_matches_relative(ctx, torch_cuda):
    """eps_mode = 1 (absolute) with eps_abs = eps * max|b| selects the same kept set and map as
    the relative mode (reading R6: eps_eff = eps * max_s |b_s|)."""
    torch = torch_cuda
    band = synth.make_band("cfg2", bins=[2])
    cfg = band.cfg
    g = geom_of(band)
    csm = torch.from_numpy(band.csm).cuda()
    rel = ctx.solve_band(g, band.freqs, csm, cfg.epsilon, 100, 0, want_b=True)
    bmax = float(np.max(np.abs(rel["b_map"].cpu().numpy()[0])))
    ab = ctx.solve_band(g, band.freqs, csm, cfg.epsilon * bmax, 100, 1)
    assert np.array_equal(rel["n_keep"].cpu().numpy(), ab["n_keep"].cpu().numpy())
    assert np.array_equal(rel["keep_idx"].cpu().numpy(), ab["keep_idx"].cpu().numpy())
    assert np.array_equal(rel["x_map"].cpu().numpy(), ab["x_map"].cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("dense", [False, True], ids=["residual", "dense_stream"])
def test_batched_path_bitwise_deterministic_cfg3(dense):
    """The whole 256-bin cfg3 band, three calls: every map bit-identical (all summation orders are
    fixed, so any difference is a race -- this test caught one in the GS solver's staging)."""
    import torch
    from paper_1608_05179_b200 import Context
    cfg = synth.CONFIGS["cfg3"]
    band = synth.make_band(cfg)
    g = geom_of(band)
    ctx = Context(0)
    csm = torch.from_numpy(band.csm).cuda()
    ref = None
    for _ in range(3):
        x = ctx.solve_band(g, band.freqs, csm, cfg.epsilon, 300, cfg.eps_mode, dense_stream=dense)["x_map"].cpu().numpy()
        if ref is None:
            ref = x
        else:
            assert np.array_equal(x, ref)
    ctx.close()


# ---------------------------------------------------------------------------- NEXT-4: paper-literal PSF
@pytest.mark.parametrize("cfgname", ["cfg1", "cfg2"])
def test_das_paper_parity(ctx, torch_cuda, oracle_lib, cfgname):
    """The DAS map with Eq. 4's focus vector v against the oracle's or_das_paper."""
    torch = torch_cuda
    band = synth.make_band(cfgname)
    g = geom_of(band)
    b = ctx.das(g, band.freqs, torch.from_numpy(band.csm).cuda(), paper=True).cpu().numpy()
    for k in range(len(band.freqs)):
        ref = oracle_lib.das_paper(*oracle_args(g), band.freqs[k], band.csm[k])
        assert rel_l2(b[k], ref) < 1e-12


@pytest.mark.parametrize("m,n,nk", [(16, 21, 441), (24, 15, 33), (24, 15, 129), (13, 15, 100), (128, 21, 300)])
def test_psf_paper_parity(ctx, torch_cuda, oracle_lib, m, n, nk):
    """The asymmetric paper-literal PSF A_P = |V^H G|^2 / M^2 (Eq. 4 x Eq. 7) on every tile: the
    exact int8-digit Gram with v on the A side and g on the B side, each with its own scales."""
    torch = torch_cuda
    g = small_geom(m, n, 3 if m % 3 == 0 else 1)
    keep = np.sort(np.random.default_rng(nk).choice(g.S, size=nk, replace=False)).astype(np.int32)
    A = ctx.psf(g, 5100.0, torch.from_numpy(keep).cuda(), paper=True).cpu().numpy()
    ref = oracle_lib.psf_paper(*oracle_args(g), 5100.0, keep)
    assert rel_l2(A, ref) < 1e-7
    assert np.max(np.abs(A - ref)) <= 2.0 ** -23 * max(1.0, np.abs(ref).max())
    if nk > 1:
        assert np.max(np.abs(A - A.T)) > 1e-4          # really asymmetric
    assert np.max(np.abs(np.diag(A) - 1.0)) < 1e-6


@pytest.mark.parametrize("nk,sweeps", [(1, 3), (33, 40), (130, 60), (441, 40)])
def test_gs_general_matrix_parity(ctx, torch_cuda, oracle_lib, nk, sweeps):
    """Forward sweeps on a general (paper-literal, asymmetric) matrix: the residual kernel on the
    transpose, against the oracle's Eq. 13-14 loop."""
    torch = torch_cuda
    band = synth.make_band("cfg1")
    g = geom_of(band)
    f = band.freqs[0]
    b_full = oracle_lib.das_paper(*oracle_args(g), f, band.csm[0])
    keep = np.sort(np.argsort(-b_full)[:nk]).astype(np.int32)
    A = oracle_lib.psf_paper(*oracle_args(g), f, keep)
    bt = b_full[keep]
    ref = oracle_lib.gs(A, bt, sweeps)
    x = ctx.gs(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(bt).cuda(), sweeps,
               general=True).cpu().numpy()
    assert ctx.stats()["gs_kernel"] == 4
    assert x.min() >= 0
    assert rel_l2(x, ref) < TOL_X, rel_l2(x, ref)
    assert abs(x.sum() - ref.sum()) < TOL_P * ref.sum()


@pytest.mark.parametrize("cfgname,bins,sweeps", [("cfg1", None, 100), ("cfg2", [0, 3, 7], 300)])
def test_e2e_paper_mode(ctx, torch_cuda, oracle_lib, cfgname, bins, sweeps):
    """NEXT-4 end to end: Eq. 4 beamformer, Alg. 1 on its map, the asymmetric Eq. 4 x Eq. 7 PSF,
    forward sweeps -- keep sets bit-exact, maps within the north_star tolerances."""
    torch = torch_cuda
    band = synth.make_band(cfgname, bins=bins)
    cfg = band.cfg
    g = geom_of(band)
    out = ctx.solve_band(g, band.freqs, torch.from_numpy(band.csm).cuda(), cfg.epsilon, sweeps, cfg.eps_mode,
                         want_b=True, paper=True)
    assert ctx.stats()["gs_kernel"] == 4
    rnk, rkeep, rx, rb = oracle_lib.solve_band_cfg(band, sweeps=sweeps, paper=True)
    for k in range(len(band.freqs)):
        assert rel_l2(out["b_map"][k].cpu().numpy(), rb[k]) < 1e-12
        assert np.array_equal(out["keep_idx"][k].cpu().numpy(), rkeep[k])
        x = out["x_map"][k].cpu().numpy()
        assert rel_l2(x, rx[k]) < TOL_X, (k, rel_l2(x, rx[k]))
        assert abs(x.sum() - rx[k].sum()) <= TOL_P * rx[k].sum()
