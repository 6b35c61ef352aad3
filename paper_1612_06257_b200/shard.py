"""Multi-GPU sharding of a batch by message index.

Every message is hashed independently (S/_highway_np.py:1-6), so a batch
shards into contiguous message-index ranges with no data-path collective:
one process per GPU, the key passed to each device as a kernel argument, and
the digests gathered once at the end (``gather_digests``).

* fixed-length batches: equal message counts per rank;
* ragged batches: byte-balanced ranges, cut at the byte quantiles of the
  offsets' prefix sum (cfg2 is sorted by length, so equal counts would differ
  ~15x in bytes);
* PRF counter ranges: equal counts.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np


def fixed_shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, stop) of rank's messages; sizes differ by at most one."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def ragged_cuts(offsets: np.ndarray, lengths: Optional[np.ndarray], world: int) -> np.ndarray:
    """world+1 message-index cut points that balance payload bytes.

    offsets: u64[n+1] (lengths None) or u64[n] with u32 lengths[n]."""
    if lengths is None:
        sizes = np.diff(np.asarray(offsets, dtype=np.uint64)).astype(np.int64)
    else:
        sizes = np.asarray(lengths, dtype=np.int64)
    n = len(sizes)
    csum = np.concatenate([[0], np.cumsum(sizes)])
    total = int(csum[-1])
    cuts = np.zeros(world + 1, np.int64)
    cuts[-1] = n
    for r in range(1, world):
        # first message whose start is at or past the r-th byte quantile
        cuts[r] = int(np.searchsorted(csum, (total * r) // world, side="left"))
        cuts[r] = max(cuts[r], cuts[r - 1])
    return cuts


def ragged_shard(offsets, lengths, world: int, rank: int) -> Tuple[int, int]:
    cuts = ragged_cuts(offsets, lengths, world)
    return int(cuts[rank]), int(cuts[rank + 1])


def gather_digests(local, n_total: int, lanes: int = 1, group=None):
    """All-gather per-rank digest tensors (contiguous shards in rank order)
    into one (n_total[, lanes]) tensor on every rank.  Works with NCCL (CUDA
    tensors) and gloo (CPU tensors).  Called once, after hashing."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    counts = [int(s.item()) for s in all_sizes]
    if sum(counts) != n_total:
        raise ValueError("shard sizes do not add up to the batch")
    mx = max(counts) if counts else 0
    shape = (mx,) if lanes == 1 else (mx, lanes)
    pad = torch.zeros(shape, dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
