"""The engine's launches are CUDA-graph capturable: no host synchronisation,
allocation or device query on the launch path once a shape has run, so a
launch-bound batch loop can be captured once and replayed.  Each case
captures a call, refills the (same) input buffer with new bytes, replays
and compares with the oracle."""
import numpy as np
import pytest
import torch

from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import (KERNEL_AUTO, KERNEL_RING, KERNEL_SPLIT, KERNEL_STAGED,
                                          KERNEL_TMA, to_u64)

pytestmark = pytest.mark.gpu


def _capture(fn):
    fn()  # warm-up: per-kernel setup happens outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


@pytest.mark.parametrize("n,L,kernel", [(4096, 1024, KERNEL_AUTO), (4096, 1024, KERNEL_SPLIT),
                                        (70000, 256, KERNEL_TMA), (5000, 1000, KERNEL_RING),
                                        (20000, 40, KERNEL_STAGED)])
def test_fixed_batch_graph_replay(oracle, n, L, kernel):
    key = synth.key256()
    d = torch.empty((n, L), dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    g = _capture(lambda: engine.highway_batch(key, d, 64, kernel=kernel, out=out))
    for seed in (3, 4):
        host = synth.counter_bytes(seed * 1000 + L, n * L).reshape(n, L)
        d.copy_(torch.from_numpy(host))
        g.replay()
        torch.cuda.synchronize()
        want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, host, 64, 4)
        assert np.array_equal(to_u64(out), want), (n, L, kernel, seed)


def test_ragged_and_sip_graph_replay(oracle):
    key, k2 = synth.key256(), synth.key128()
    lens = synth.lengths(5, 6000, 0, 700)
    off = np.zeros(6001, np.uint64)
    off[1:] = np.cumsum(lens)
    total = int(off[-1])
    d_buf = torch.empty(total, dtype=torch.uint8, device="cuda")
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    o1 = torch.empty(6000, dtype=torch.int64, device="cuda")
    o2 = torch.empty(6000, dtype=torch.int64, device="cuda")

    def step():
        engine.highway_ragged(key, d_buf, d_off, None, 64, out=o1)
        engine.sip_ragged(k2, d_buf, d_off, None, 2, 4, out=o2)

    g = _capture(step)
    for seed in (7, 8):
        host = synth.counter_bytes(seed, total)
        d_buf.copy_(torch.from_numpy(host))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(to_u64(o1), oracle.batch_ragged(oracle.ALG_HIGHWAY, key, host, off,
                                                              None, 64, 4))
        assert np.array_equal(to_u64(o2), oracle.batch_ragged(oracle.ALG_SIPHASH, k2, host, off,
                                                              None, 2, 4))


def test_ordered_ragged_graph_replay(oracle):
    """balance=True inside a capture: the three ordering launches and the
    ordered hashing launch replay together (the layout is fixed; the bytes
    change between replays)."""
    key = synth.key256()
    lens = synth.lengths(6, 9000, 0, 3000)
    off = np.zeros(9001, np.uint64)
    off[1:] = np.cumsum(lens)
    total = int(off[-1])
    d_buf = torch.empty(total, dtype=torch.uint8, device="cuda")
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    out = torch.empty(9000, dtype=torch.int64, device="cuda")
    g = _capture(lambda: engine.highway_ragged(key, d_buf, d_off, None, 64, out=out,
                                               kernel=KERNEL_RING, balance=True))
    for seed in (9, 10):
        host = synth.counter_bytes(seed, total)
        d_buf.copy_(torch.from_numpy(host))
        g.replay()
        torch.cuda.synchronize()
        want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, host, off, None, 64, 4)
        assert np.array_equal(to_u64(out), want), seed
