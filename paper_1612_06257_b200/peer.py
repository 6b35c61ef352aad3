"""Digests gathered by peer stores instead of a collective.

The batch shards by message index with no exchange in the hot loop; the only
communication is the end-of-run gather of the digests.  On one node of
NVLink-connected GPUs that gather need not be a separate step: the root rank
allocates the full (n_total[, lanes]) digest tensor, shares it with every
rank through CUDA IPC (the same mechanism ``torch.multiprocessing`` uses for
CUDA tensors, opened with lazy peer access), and each rank passes its slice
of that buffer as ``out=`` to the hashing call.  Every kernel then stores its
digests straight into the root's HBM over NVLink while it hashes -- the
"compute followed by a collective" fused into the compute kernel itself,
with no kernel change (the engine's kernels store digests through a plain
device pointer; ``engine`` accepts an ``out`` on a peer-accessible device).

The digests are 8 bytes per message (1/128 of a 1 KiB batch's input bytes),
so the peer stores are a negligible share of the NVLink bandwidth and are
hidden under the hashing.  ``shard.gather_digests`` (NCCL all-gather after
the kernels) remains the portable alternative.

Usage, in every rank (one process per GPU, torch.distributed initialised):

    buf = peer.shared_digest_buffer(n_total, lanes, root=0)   # root's memory
    a, b = shard.fixed_shard(n_total, world, rank)
    engine.highway_batch(key, my_msgs, 64, out=buf[a:b])
    peer.fence()            # every rank's stores are complete and visible
    if rank == root: use(buf)

The shared view stays valid while the root's tensor is alive: call
``fence()`` before the root frees or reads it.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shared_digest_buffer(n_total: int, lanes: int = 1, root: int = 0, group=None):
    """The root's (n_total[, lanes]) int64 CUDA tensor, allocated on the
    root's current device and mapped into every rank by CUDA IPC.  Returns
    the local view (the root: the tensor itself)."""
    from torch.multiprocessing.reductions import reduce_tensor

    rank = dist.get_rank(group)
    shape = (n_total,) if lanes == 1 else (n_total, lanes)
    payload = [None]
    if rank == root:
        buf = torch.empty(shape, dtype=torch.int64, device=torch.cuda.current_device())
        payload = [reduce_tensor(buf)]
    dist.broadcast_object_list(payload, src=root, group=group)
    if rank == root:
        return buf
    fn, args = payload[0]
    return fn(*args)


def fence(group=None) -> None:
    """Wait for this rank's kernels (its peer stores), then for every rank:
    after it returns, the root's buffer holds all digests."""
    torch.cuda.synchronize()
    dist.barrier(group=group)
