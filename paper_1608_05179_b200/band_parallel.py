"""Frequency bins of one band sharded over the GPUs of a node.

Bins are independent problems (the paper processes a band of frequencies one by one,
PAPER.md:22, :545-547), so the hot path has no inter-GPU traffic: bin k is solved on rank
k mod G (strided, so every rank gets the same spread of frequencies and about the same
sum of S~_k^2).  The only collective is one gather of the results at the end:
x_map [K_r, S] fp32, the keep sets as bitmask words [K_r, ceil(S/32)] (dwc_keep_mask) and
n_keep [K_r], each padded to ceil(K/G) rows per rank, moved with all_gather_into_tensor
(NCCL over NVLink on the GPU box; the same code runs on gloo in the CPU tests).

This module is plumbing: it moves and reorders bytes; every computation on the path runs
in the library's kernels.
"""
from __future__ import annotations

import math
from typing import List, Tuple


def shard_bins(n_bins: int, rank: int, world: int) -> List[int]:
    """Bins solved by `rank`: k = rank, rank + G, ... (ascending)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return list(range(rank, n_bins, world))


def rows_per_rank(n_bins: int, world: int) -> int:
    return max(1, math.ceil(n_bins / world))


def owner_of(k: int, world: int) -> Tuple[int, int]:
    """(rank, local row) of global bin k."""
    return k % world, k // world


def gather_band(x_local, n_keep_local, mask_local, n_bins: int, group=None):
    """All-gather the per-rank results into global bin order on every rank.

    x_local [K_r, S] float32, n_keep_local [K_r] int32, mask_local [K_r, W] int32 (bitmask
    words); all on the process group's device.  Returns (x_map [n_bins, S],
    n_keep [n_bins], mask [n_bins, W]) in global bin order.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    kmax = rows_per_rank(n_bins, world)
    k_r = len(shard_bins(n_bins, rank, world))
    if x_local.shape[0] != k_r or n_keep_local.shape[0] != k_r or mask_local.shape[0] != k_r:
        raise ValueError(f"rank {rank} holds {x_local.shape[0]} bins, expected {k_r}")
    S, W = x_local.shape[1], mask_local.shape[1]
    dev = x_local.device

    def padded(t, shape_tail, dtype):
        out = torch.zeros((kmax,) + shape_tail, dtype=dtype, device=dev)
        out[:k_r].copy_(t)
        return out

    xs = torch.empty((world * kmax, S), dtype=x_local.dtype, device=dev)
    ms = torch.empty((world * kmax, W), dtype=mask_local.dtype, device=dev)
    ns = torch.empty((world * kmax,), dtype=n_keep_local.dtype, device=dev)
    dist.all_gather_into_tensor(xs, padded(x_local, (S,), x_local.dtype), group=group)
    dist.all_gather_into_tensor(ms, padded(mask_local, (W,), mask_local.dtype), group=group)
    dist.all_gather_into_tensor(ns, padded(n_keep_local, (), n_keep_local.dtype), group=group)
    # global bin k lives at [k % world, k // world]: a transpose of the (world, kmax) grid
    order = torch.arange(n_bins, device=dev)
    src = (order % world) * kmax + order // world
    return xs.index_select(0, src), ns.index_select(0, src), ms.index_select(0, src)
