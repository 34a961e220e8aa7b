"""Two contexts driven from two host threads on two streams (bench.py's pipelined measurement):
every band's outputs are bit-identical to the same band solved alone.

Regressions this guards: a kernel's dynamic shared-memory limit is per function and device, so a
thread setting it for a small launch lowered it under the other thread's larger launch
(cudaErrorInvalidValue: raise_smem_limit only raises it); outputs read before the band's own
stream finished."""
import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_two_contexts_two_threads_match_alone(torch_cuda):
    torch = torch_cuda
    from paper_1608_05179_b200 import Context, Geometry
    cfg = synth.CONFIGS["cfg3"]
    b0 = synth.make_band(cfg)
    g = Geometry(b0.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
    # bands of different sizes (different launch classes and shared-memory needs) on each context
    subsets = [list(range(0, 40)), list(range(200, 256)), list(range(90, 150)), list(range(230, 256))]
    bands = [synth.make_band(cfg, seed=0, bins=s_, block=i + 1) for i, s_ in enumerate(subsets)]
    csm = [torch.from_numpy(b.csm).cuda() for b in bands]
    ctxs = [Context(0), Context(0)]
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    try:
        ref = []
        for b, c in zip(bands, csm):
            o = ctxs[0].solve_band(g, b.freqs, c, cfg.epsilon, cfg.sweeps, cfg.eps_mode)
            torch.cuda.synchronize()
            ref.append({k: o[k].cpu().numpy() for k in ("n_keep", "keep_idx", "x_map")})
        errors, got = [], {}

        def worker(j):
            try:
                for rep in range(3):
                    for i in range(j, len(bands), 2):
                        o = ctxs[j].solve_band(g, bands[i].freqs, csm[i], cfg.epsilon, cfg.sweeps, cfg.eps_mode,
                                               stream=sts[j])
                        sts[j].synchronize()
                        got[(rep, i)] = {k: o[k].cpu().numpy() for k in ("n_keep", "keep_idx", "x_map")}
            except Exception as e:   # noqa: BLE001 -- reported by the main thread
                errors.append(repr(e))
        ths = [threading.Thread(target=worker, args=(j,)) for j in range(2)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert not errors, errors
        assert len(got) == 3 * len(bands)
        for (rep, i), o in got.items():
            np.testing.assert_array_equal(o["n_keep"], ref[i]["n_keep"])
            for k in range(len(bands[i].freqs)):
                nk = int(ref[i]["n_keep"][k])
                np.testing.assert_array_equal(o["keep_idx"][k, :nk], ref[i]["keep_idx"][k, :nk])
            np.testing.assert_array_equal(o["x_map"], ref[i]["x_map"], err_msg=f"rep {rep} band {i}")
    finally:
        for c in ctxs:
            c.close()


def test_four_contexts_dropped_outputs_on_side_streams(torch_cuda):
    """Four contexts on four threads and streams, each call's outputs allocated by the binding and
    dropped before the stream synchronises (every other call's kept): the binding records the
    call's stream on every tensor it hands the library, so the caching allocator does not give a
    dropped output's block to another thread's allocation while the kernels still write it.
    (Regression: consecutive shard-sized bands on four contexts faulted with illegal-address and
    invalid-address-space errors; CUDA_LAUNCH_BLOCKING=1 hid it.)"""
    torch = torch_cuda
    from paper_1608_05179_b200 import Context, Geometry
    cfg = synth.CONFIGS["cfg3"]
    bins = list(range(1, 256, 8))   # a 32-bin strided shard (8-way sharding)
    bands = [synth.make_band(cfg, seed=0, bins=bins, block=i + 1) for i in range(4)]
    g = Geometry(bands[0].mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
    csm = [torch.from_numpy(b.csm).cuda() for b in bands]
    nc = 4
    ctxs = [Context(0) for _ in range(nc)]
    sts = [torch.cuda.Stream() for _ in range(nc)]
    sweeps = 300
    try:
        ref = []
        for b, c in zip(bands, csm):
            o = ctxs[0].solve_band(g, b.freqs, c, cfg.epsilon, sweeps, cfg.eps_mode)
            torch.cuda.synchronize()
            ref.append({k: o[k].cpu().numpy() for k in ("n_keep", "x_map")})
        errors, got = [], {}

        def worker(j):
            try:
                for rep in range(4):
                    i = (j + rep) % len(bands)
                    ctxs[j].solve_band(g, bands[i].freqs, csm[i], cfg.epsilon, sweeps, cfg.eps_mode, stream=sts[j])
                    junk = [torch.full((len(bins), cfg.S), -7, dtype=torch.int32, device="cuda") for _ in range(3)]
                    o = ctxs[j].solve_band(g, bands[i].freqs, csm[i], cfg.epsilon, sweeps, cfg.eps_mode, stream=sts[j])
                    junk += [torch.full((len(bins), cfg.S), 1e30, dtype=torch.float32, device="cuda") for _ in range(3)]
                    sts[j].synchronize()
                    got[(j, rep)] = (i, {k: o[k].cpu().numpy() for k in ("n_keep", "x_map")})
                    del junk
            except Exception as e:   # noqa: BLE001 -- reported by the main thread
                errors.append(repr(e))
        ths = [threading.Thread(target=worker, args=(j,)) for j in range(nc)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        torch.cuda.synchronize()
        assert not errors, errors
        for (j, rep), (i, o) in got.items():
            np.testing.assert_array_equal(o["n_keep"], ref[i]["n_keep"])
            np.testing.assert_array_equal(o["x_map"], ref[i]["x_map"], err_msg=f"context {j} rep {rep} band {i}")
    finally:
        for c in ctxs:
            c.close()


def test_throughput_hint_is_bitwise_neutral(torch_cuda):
    """DWC_THROUGHPUT only moves systems into the two-CTAs-per-SM class: the full cfg3 band's
    outputs are bitwise identical with and without it (also on a 32-bin shard, where the hint
    pairs bins the default leaves one per SM)."""
    torch = torch_cuda
    from paper_1608_05179_b200 import Context, Geometry
    cfg = synth.CONFIGS["cfg3"]
    ctx = Context(0)
    try:
        for bins in (None, list(range(1, 256, 8))):
            band = synth.make_band(cfg, bins=bins)
            g = Geometry(band.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
            csm = torch.from_numpy(band.csm).cuda()
            outs = []
            for tp in (False, True):
                o = ctx.solve_band(g, band.freqs, csm, cfg.epsilon, cfg.sweeps, cfg.eps_mode, throughput=tp)
                torch.cuda.synchronize()
                outs.append({k: o[k].cpu().numpy() for k in ("n_keep", "keep_idx", "x_map")})
            for k in ("n_keep", "keep_idx", "x_map"):
                np.testing.assert_array_equal(outs[0][k], outs[1][k], err_msg=k)
    finally:
        ctx.close()


def test_results_independent_of_timing_small_systems_and_alternating(torch_cuda):
    """The panel producer's prediction mask is read only from a visit that is certainly complete,
    so which carries take the staged-panel path (and so the fp32 summation order) never depends
    on timing: bins of < 4 blocks and alternating sweeps (whose turn revisits a block at once)
    give bitwise the same maps alone and while another context's band loads the GPU."""
    torch = torch_cuda
    from paper_1608_05179_b200 import Context, Geometry
    cfg = synth.CONFIGS["cfg3"]
    small = synth.make_band(cfg, bins=list(range(0, 24)))   # the smallest systems of the band (S~ < 200)
    load = synth.make_band(cfg, bins=list(range(128, 256)), block=1)
    g = Geometry(small.mic_xyz, cfg.n, cfg.side_len, cfg.z0, cfg.c0, cfg.cx, cfg.cy)
    cs, cl = torch.from_numpy(small.csm).cuda(), torch.from_numpy(load.csm).cuda()
    ctxs = [Context(0), Context(0)]
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    try:
        for alt in (False, True):
            ref = ctxs[0].solve_band(g, small.freqs, cs, cfg.epsilon, 400, cfg.eps_mode, alt=alt)
            torch.cuda.synchronize()
            assert int(ref["n_keep"].min()) < 128   # (some system of fewer than 4 blocks)
            ref = ref["x_map"].cpu().numpy()
            for rep in range(3):
                ctxs[1].solve_band(g, load.freqs, cl, cfg.epsilon, 300, cfg.eps_mode, stream=sts[1])
                o = ctxs[0].solve_band(g, small.freqs, cs, cfg.epsilon, 400, cfg.eps_mode, alt=alt, stream=sts[0])
                torch.cuda.synchronize()
                np.testing.assert_array_equal(o["x_map"].cpu().numpy(), ref, err_msg=f"alt={alt} rep {rep}")
    finally:
        for c in ctxs:
            c.close()
