"""Multi-GPU plumbing: bins sharded k -> rank k mod G, one all-gather of
x_map / keep bitmask / n_keep at the end.  The collective logic runs here on CPU with the
gloo backend (world sizes 2 and 3, ragged shards); the bitmask kernels are checked on the
GPU against numpy's packbits."""
import os
import socket

import numpy as np
import pytest

from paper_1608_05179_b200.band_parallel import owner_of, rows_per_rank, shard_bins


def test_shard_partition_and_balance():
    for n_bins in (1, 2, 7, 8, 64, 256, 1024):
        for world in (1, 2, 3, 4, 8):
            shards = [shard_bins(n_bins, r, world) for r in range(world)]
            flat = sorted(k for s in shards for k in s)
            assert flat == list(range(n_bins))
            assert max(map(len, shards)) - min(map(len, shards)) <= 1
            assert max(map(len, shards)) == (rows_per_rank(n_bins, world) if n_bins else 0) or n_bins < world
            for r, s in enumerate(shards):
                for i, k in enumerate(s):
                    assert owner_of(k, world) == (r, i)
    with pytest.raises(ValueError):
        shard_bins(8, 2, 2)


def test_strided_shards_balance_work():
    # S~ grows with frequency; strided shards keep sum S~^2 within a few %
    nk = np.linspace(93, 1170, 256) ** 2
    for world in (2, 4, 8):
        loads = [nk[shard_bins(256, r, world)].sum() for r in range(world)]
        assert max(loads) / np.mean(loads) < 1.05


def keep_sets(n_bins, S, seed):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n_bins):
        nk = min(S, int(rng.integers(1, S + 1)) if k % 3 else int(rng.integers(1, 8)))
        out.append(np.sort(rng.choice(S, size=nk, replace=False)).astype(np.int32))
    return out


def pack_words(keep, S):
    bits = np.zeros(((S + 31) // 32) * 32, dtype=np.uint8)
    bits[keep] = 1
    return np.packbits(bits, bitorder="little").view("<u4").astype(np.int64).astype(np.uint32).view(np.int32)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, n_bins, S):
    import torch
    import torch.distributed as dist

    from paper_1608_05179_b200.band_parallel import gather_band

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        keeps = keep_sets(n_bins, S, 7)
        mine = shard_bins(n_bins, rank, world)
        x = torch.tensor(np.array([k * 1000.0 + np.arange(S) for k in mine]).reshape(len(mine), S), dtype=torch.float32)
        nk = torch.tensor([len(keeps[k]) for k in mine], dtype=torch.int32)
        m = torch.tensor(np.array([pack_words(keeps[k], S) for k in mine]).reshape(len(mine), -1))
        calls = []
        real = dist.all_gather_into_tensor

        def counting(*a, **kw):
            calls.append(1)
            return real(*a, **kw)
        dist.all_gather_into_tensor = counting
        try:
            gx, gn, gm = gather_band(x, nk, m, n_bins)
        finally:
            dist.all_gather_into_tensor = real
        assert len(calls) == 1   # exactly one all_gather_into_tensor
        ref_x = np.array([k * 1000.0 + np.arange(S) for k in range(n_bins)], dtype=np.float32)
        assert np.array_equal(gx.numpy(), ref_x)
        assert np.array_equal(gn.numpy(), [len(kk) for kk in keeps])
        for k in range(n_bins):
            assert np.array_equal(gm[k].numpy(), pack_words(keeps[k], S))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_bins,S", [(2, 8, 441), (2, 7, 100), (3, 8, 37)])
def test_gather_band_gloo(world, n_bins, S):
    import torch.multiprocessing as mp
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    mp.spawn(_gather_worker, args=(world, _free_port(), n_bins, S), nprocs=world, join=True)


@pytest.mark.gpu
@pytest.mark.parametrize("S", [1, 31, 32, 33, 441, 10201])
def test_keep_mask_roundtrip_gpu(S):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_05179_b200 import Context
    ctx = Context(0)
    keeps = keep_sets(5, S, S)
    keep_idx = np.full((5, S), -1, dtype=np.int32)
    for k, kk in enumerate(keeps):
        keep_idx[k, :len(kk)] = kk
    nk = torch.tensor([len(kk) for kk in keeps], dtype=torch.int32, device="cuda")
    ki = torch.from_numpy(keep_idx).cuda()
    mask = ctx.keep_mask(nk, ki)
    torch.cuda.synchronize()
    for k, kk in enumerate(keeps):
        assert np.array_equal(mask[k].cpu().numpy(), pack_words(kk, S))
    n2, k2 = ctx.keep_unmask(mask, S)
    assert np.array_equal(n2.cpu().numpy(), nk.cpu().numpy())
    assert np.array_equal(k2.cpu().numpy(), keep_idx)
    ctx.close()
