"""Frequency bins of one band sharded over the GPUs of a node.

Bins are independent problems (the paper processes a band of frequencies one by one,
PAPER.md:22, :545-547), so the hot path has no inter-GPU traffic: bin k is solved on rank
k mod G (strided, so every rank gets the same spread of frequencies and about the same
sum of S~_k^2).  The only collective is ONE all_gather_into_tensor of the results at the end:
each rank packs, per bin row, x_map [S] fp32 (as its 32-bit words), the keep set as bitmask
words [ceil(S/32)] (dwc_keep_mask) and n_keep into one int32 row of S + ceil(S/32) + 1 words,
padded to ceil(K/G) rows (NCCL over NVLink on the GPU box; the same code runs on gloo in the
CPU tests).

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
    if x_local.dtype != torch.float32 or mask_local.dtype != torch.int32 or n_keep_local.dtype != torch.int32:
        raise TypeError("x_map float32, mask int32 and n_keep int32 expected")
    row = S + W + 1
    # one packed send buffer: [x_map bits | mask words | n_keep] per bin row (zero padded rows)
    send = torch.zeros((kmax, row), dtype=torch.int32, device=dev)
    send[:k_r, :S].copy_(x_local.contiguous().view(torch.int32))
    send[:k_r, S:S + W].copy_(mask_local)
    send[:k_r, S + W].copy_(n_keep_local)
    recv = torch.empty((world * kmax, row), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    # global bin k lives at [k % world, k // world]: a transpose of the (world, kmax) grid
    order = torch.arange(n_bins, device=dev)
    src = (order % world) * kmax + order // world
    g = recv.index_select(0, src)
    return g[:, :S].contiguous().view(torch.float32), g[:, S + W].contiguous(), g[:, S:S + W].contiguous()
