"""Seeded random layouts through every kernel, bit-exact against the oracle.

Each case draws a batch shape the structured tests do not pin: random
message counts and lengths, random offsets (packed, gapped, overlapping,
unsorted), a random byte shift of the device buffer, random widths and
round counts.  Fixed-length batches go through TMA / direct / split where the
shape allows; ragged ones through the staged and ring kernels (HighwayHash)
and the ring kernel (Sip).
"""
import numpy as np
import pytest
import torch

from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import (KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING, KERNEL_SPLIT,
                                          KERNEL_STAGED, KERNEL_TMA, to_u64)

pytestmark = pytest.mark.gpu


def _ragged_case(rng):
    n = int(rng.integers(1, 3000))
    kind = rng.choice(["short", "mixed", "long"])
    hi = {"short": 70, "mixed": 600, "long": 5000}[kind]
    lens = rng.integers(0, hi, n).astype(np.uint32)
    layout = rng.choice(["packed", "gapped", "random"])
    if layout == "packed":
        off = np.zeros(n, np.uint64)
        off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
        total = int(off[-1]) + int(lens[-1])
    elif layout == "gapped":
        gaps = rng.integers(0, 40, n).astype(np.uint64)
        off = np.cumsum(gaps + np.concatenate([[0], lens[:-1]]).astype(np.uint64)).astype(np.uint64)
        total = int(off[-1]) + int(lens[-1])
    else:
        total = int(lens.max()) + int(rng.integers(1, 20000))
        off = rng.integers(0, total - int(lens.max()) + 1, n).astype(np.uint64)
    buf = synth.counter_bytes(int(rng.integers(0, 1 << 30)), max(total, 1))
    return buf, off, lens


@pytest.mark.parametrize("seed", range(32))
def test_random_ragged(oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    key = rng.integers(0, 2**64, 4, dtype=np.uint64)
    k2 = key[:2].copy()
    for _ in range(4):
        buf, off, lens = _ragged_case(rng)
        shift = int(rng.integers(0, 16))
        raw = torch.from_numpy(np.concatenate([np.zeros(shift, np.uint8), buf])).cuda()
        d_buf = raw[shift:]
        d_off, d_len = (torch.from_numpy(off.view(np.int64)).cuda(),
                        torch.from_numpy(lens.view(np.int32)).cuda())
        width = int(rng.choice([64, 128, 256]))
        rounds = int(rng.integers(0, 6))
        want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, lens, width, rounds)
        for kernel in (KERNEL_STAGED, KERNEL_RING):
            got = to_u64(engine.highway_ragged(key, d_buf, d_off, d_len, width, rounds,
                                               kernel=kernel))
            assert np.array_equal(got, want), (seed, kernel, width, rounds, len(lens))
        c, d = (2, 4) if rng.integers(0, 2) else (1, 3)
        tree = bool(rng.integers(0, 2))
        alg = oracle.ALG_SIPTREE if tree else oracle.ALG_SIPHASH
        got = to_u64(engine.sip_ragged(k2, d_buf, d_off, d_len, c, d, tree))
        assert np.array_equal(got, oracle.batch_ragged(alg, k2, buf, off, lens, c, d)), seed


@pytest.mark.parametrize("seed", range(32))
def test_random_fixed(oracle, seed):
    rng = np.random.default_rng(2000 + seed)
    key = rng.integers(0, 2**64, 4, dtype=np.uint64)
    k2 = key[:2].copy()
    for _ in range(4):
        L = int(rng.choice([int(rng.integers(0, 200)), 16 * int(rng.integers(2, 80)),
                            128 * int(rng.integers(1, 40))]))
        n = int(rng.integers(1, 2500 if L <= 2048 else 300))
        m = synth.counter_bytes(int(rng.integers(0, 1 << 30)), n * L).reshape(n, L)
        d = torch.from_numpy(m).cuda()
        width = int(rng.choice([64, 128, 256]))
        rounds = int(rng.integers(0, 6))
        want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, m, width, rounds)
        sip_kernels = [KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING, KERNEL_STAGED]
        if L >= 32 and L % 16 == 0:
            sip_kernels.append(KERNEL_TMA)
        kernels = list(sip_kernels)
        if L >= 128 and L % 128 == 0:
            kernels.append(KERNEL_SPLIT)
        for kernel in kernels:
            got = to_u64(engine.highway_batch(key, d, width, rounds, kernel=kernel))
            assert np.array_equal(got, want), (seed, kernel, n, L, width, rounds)
        c, dd = (2, 4) if rng.integers(0, 2) else (1, 3)
        tree = bool(rng.integers(0, 2))
        alg = oracle.ALG_SIPTREE if tree else oracle.ALG_SIPHASH
        want = oracle.batch_fixed(alg, k2, m, c, dd)
        for kernel in sip_kernels:
            got = to_u64(engine.sip_batch(k2, d, c, dd, tree, kernel=kernel))
            assert np.array_equal(got, want), (seed, kernel, n, L, c, dd, tree)
