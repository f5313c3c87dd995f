# SPDX-License-Identifier: Apache-2.0
"""Multi-GPU plumbing for the batch-sharded path (BASELINE config 5a).

One process per GPU.  Ciphertext batches are independent, so they are split
across ranks with no data-path collective; the only collective is the timing
reduction (device time = max over ranks).
"""
from __future__ import annotations

import os
from typing import Tuple


def env() -> Tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous block partition of n_items across world ranks (sizes differ by <= 1)."""
    base, rem = divmod(n_items, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (e.g. device milliseconds)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def chunk_shards(n_items: int, world: int, chunks: int):
    """Row blocks of a chunked, rank-sharded output: entry [c][r] is the range of global
    rows rank r produces in its chunk c (rank r's shard split into `chunks` contiguous
    pieces), so chunk c of every rank can be gathered while chunk c + 1 is computed."""
    out = []
    for c in range(chunks):
        row = []
        for r in range(world):
            blk = shard(n_items, r, world)
            sub = shard(len(blk), c, chunks)
            row.append(range(blk.start + sub.start, blk.start + sub.stop))
        out.append(row)
    return out
