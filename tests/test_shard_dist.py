"""Multi-process (gloo, world_size 2, CPU) coverage of the N>1 path: shard
ranges, byte balancing for ragged batches, and the end-of-run digest gather.
Per-rank digests come from the CPU oracle here (the GPU kernels are covered by
the -m gpu tests); what is under test is the host-side sharding/gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1612_06257_b200 import shard, synth


def test_fixed_shard_covers_exactly_once():
    for n in (0, 1, 7, 1000, 1 << 24):
        for world in (1, 2, 3, 8):
            ranges = [shard.fixed_shard(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.fixed_shard(10, 2, 2)


def test_ragged_cuts_balance_bytes_on_sorted_sweep():
    lens, off, _ = synth.remainder_sweep_layout(1024, 64)
    for world in (2, 4, 8):
        cuts = shard.ragged_cuts(off, None, world)
        assert cuts[0] == 0 and cuts[-1] == len(lens)
        assert np.all(np.diff(cuts) >= 0)
        per = [int(off[cuts[r + 1]] - off[cuts[r]]) for r in range(world)]
        total = int(off[-1])
        assert max(per) - min(per) <= 2 * 1023 + 1, per  # within one message of ideal
        assert sum(per) == total
        # equal-count shards would be badly unbalanced on this sorted layout
        eq = [shard.fixed_shard(len(lens), world, r) for r in range(world)]
        eq_bytes = [int(off[b] - off[a]) for a, b in eq]
        assert max(eq_bytes) / max(1, min(eq_bytes)) > 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle

        key = synth.key256()
        # ragged batch, byte-balanced shards
        lens = synth.lengths(3, 5000, 0, 300)
        off = np.zeros(5001, np.uint64)
        off[1:] = np.cumsum(lens)
        buf = synth.counter_bytes(4, int(off[-1]))
        a, b = shard.ragged_shard(off, None, world, rank)
        local = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off[a:b + 1], None, 256, 4)
        local_t = torch.from_numpy(local.view(np.int64).reshape(-1, 4).copy())
        full = shard.gather_digests(local_t, 5000, lanes=4)
        # fixed batch (weak-scaling layout of bench.py), counter bytes by global index
        n_per, L = 300, 64
        s0, s1 = shard.fixed_shard(n_per * world, world, rank)
        mine = synth.counter_bytes(1, (s1 - s0) * L, word_offset=s0 * L // 8).reshape(-1, L)
        d = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, mine, 64, 4)
        full2 = shard.gather_digests(torch.from_numpy(d.view(np.int64).copy()), n_per * world)
        if rank == 0:
            np.save(os.path.join(result_dir, "ragged.npy"), full.numpy().view(np.uint64))
            np.save(os.path.join(result_dir, "fixed.npy"), full2.numpy().view(np.uint64))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_equals_whole_batch(tmp_path, oracle):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    key = synth.key256()
    lens = synth.lengths(3, 5000, 0, 300)
    off = np.zeros(5001, np.uint64)
    off[1:] = np.cumsum(lens)
    buf = synth.counter_bytes(4, int(off[-1]))
    whole = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, None, 256, 4)
    assert np.array_equal(np.load(tmp_path / "ragged.npy"), whole)
    allm = synth.counter_bytes(1, 600 * 64).reshape(600, 64)
    assert np.array_equal(np.load(tmp_path / "fixed.npy"),
                          oracle.batch_fixed(oracle.ALG_HIGHWAY, key, allm, 64, 4))
