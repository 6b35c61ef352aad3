"""Gather by peer stores (peer.py): two processes share the root's digest
buffer through CUDA IPC, each hashes its shard with ``out=`` its slice of
that buffer, and after ``fence()`` the root holds every digest, equal to the
oracle's.  Both processes use cuda:0 here (the box has one GPU): this checks
the IPC mapping and the engine's store path, not NVLink bandwidth."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1612_06257_b200 import engine, peer, shard, synth

        torch.cuda.set_device(0)
        n, L = 50_001, 1024
        a, b = shard.fixed_shard(n, world, rank)
        msgs = torch.empty((b - a) * L, dtype=torch.uint8, device="cuda")
        synth.fill_device(msgs, 31, word_offset=a * L // 8)
        buf = peer.shared_digest_buffer(n, 4, root=0)
        engine.highway_batch(synth.key256(), msgs.view(b - a, L), 256, out=buf[a:b])
        # a ragged call into a second shared buffer
        sbuf = peer.shared_digest_buffer(n, 1, root=0)
        off = torch.arange(b - a + 1, dtype=torch.int64, device="cuda") * L
        engine.sip_ragged(synth.key128(), msgs, off, None, 2, 4, out=sbuf[a:b])
        peer.fence()
        if rank == 0:
            from oracle import oracle

            host = synth.counter_bytes(31, n * L).reshape(n, L)
            want = oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(), host, 256, 4)
            want_s = oracle.batch_fixed(oracle.ALG_SIPHASH, synth.key128(), host, 2, 4)
            ok = (np.array_equal(engine.to_u64(buf), want) and
                  np.array_equal(engine.to_u64(sbuf), want_s))
            with open(result, "w") as f:
                f.write("ok" if ok else "mismatch")
        peer.fence()
    finally:
        dist.destroy_process_group()


def test_peer_store_gather(tmp_path):
    result = str(tmp_path / "r")
    mp.start_processes(_worker, args=(2, _free_port(), result), nprocs=2, start_method="spawn")
    assert open(result).read() == "ok"


def test_out_on_other_device_rejected_without_peer_access():
    """A single-GPU box has no peer device: an out on a CPU tensor is still
    rejected (the peer relaxation only admits peer-accessible GPUs)."""
    from paper_1612_06257_b200 import engine, synth

    m = torch.zeros((4, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        engine.highway_batch(synth.key256(), m, 64, out=torch.empty(4, dtype=torch.int64))
