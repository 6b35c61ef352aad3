"""GPU parity: the CUDA engine (through the C ABI) against the reference.

Comparators, in order of authority:
  * the reference's frozen vectors and reference-generated fixtures
    (tests/golden/, made by tests/golden/gen_golden.py from lanehash);
  * the CPU oracle oracle/lh_oracle.c (itself pinned to those fixtures by
    tests/test_oracle.py) on the same seeded inputs.
Integer hashing: every comparison is bit-exact.
"""
import struct

import numpy as np
import pytest
import torch

import paper_1612_06257_b200 as lh
from conftest import golden_npy
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import (KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING, KERNEL_SPLIT,
                                          KERNEL_STAGED, KERNEL_TMA, to_u64)
from paper_1612_06257_b200.highway import Key256
from paper_1612_06257_b200.sip import SIPHASH_13, SIPHASH_24, Key128, SipParams

pytestmark = pytest.mark.gpu

DEV = "cuda"


def ramp(n):
    return bytes(i & 0xFF for i in range(n))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


# ---------------------------------------------------------------------------
# reference frozen vectors through the facade (one-shot, as T/test_highway.py)
# ---------------------------------------------------------------------------

def test_frozen_64(golden, ramp_key):
    for n, hexd in golden["frozen_64"].items():
        assert lh.highway_hash64(ramp_key, ramp(int(n))) == int(hexd, 16), n


def test_frozen_256(golden, ramp_key):
    for n, hexd in golden["frozen_256_hex"].items():
        assert lh.digest256_to_bytes(lh.highway_hash256(ramp_key, ramp(int(n)))).hex() == hexd


def test_published_siphash24(golden):
    key = Key128.from_bytes(bytes(range(16)))
    msg = bytes(range(64))
    for n, hexd in enumerate(golden["siphash24_reference_le_hex"]):
        assert struct.pack("<Q", lh.siphash(key, msg[:n])).hex() == hexd, n


def test_highway_cases_all_widths_and_rounds(golden):
    for case in golden["highway_cases"]:
        key = Key256.from_hex(case["key"])
        msg = bytes.fromhex(case["msg"])
        b = lh.get_backend()
        for r in (1, 2, 3, 4):
            want = [int(x, 16) for x in case[f"h256_r{r}"]]
            assert list(b.hash256(key, msg, r)) == want, (len(msg), r)
            assert list(b.hash128(key, msg, r)) == want[:2]
            assert b.hash64(key, msg, r) == want[0]
        assert b.hash64(key, msg) == int(case["h64"], 16)


def test_sip_cases(golden):
    for case in golden["sip_cases"]:
        key = Key128.from_hex(case["key"])
        msg = bytes.fromhex(case["msg"])
        assert lh.siphash(key, msg, SIPHASH_24) == int(case["sip24"], 16)
        assert lh.siphash(key, msg, SIPHASH_13) == int(case["sip13"], 16)
        assert lh.siphash(key, msg, SipParams(3, 5)) == int(case["sip35"], 16)
        assert lh.siptreehash(key, msg, SIPHASH_24) == int(case["tree24"], 16)
        assert lh.siptreehash(key, msg, SIPHASH_13) == int(case["tree13"], 16)
        assert lh.siptreehash(key, msg, SipParams(3, 5)) == int(case["tree35"], 16)


# ---------------------------------------------------------------------------
# cfg1: 4096 x 1 KiB, both kernels, host and device entry
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("kernel", [KERNEL_AUTO, KERNEL_DIRECT, KERNEL_TMA, KERNEL_RING])
def test_cfg1_kernels(kernel):
    key = synth.key256()
    msgs = synth.numpy_bytes(1, (4096, 1024))
    d = to_u64(engine.highway_batch(key, dev(msgs), 64, 4, kernel=kernel))
    assert np.array_equal(d, golden_npy("cfg1_hh64.npy"))


def test_cfg1_host_path_and_backend():
    key = synth.key256()
    msgs = synth.numpy_bytes(1, (4096, 1024))
    d = lh.get_backend().hash64_batch(key, msgs)  # numpy in -> numpy out
    assert d.dtype == np.uint64 and np.array_equal(d, golden_npy("cfg1_hh64.npy"))
    old = engine.HOST_CHUNK_BYTES
    engine.HOST_CHUNK_BYTES = 300 * 1024  # force many pipelined chunks
    try:
        d2 = engine.highway_batch(key, torch.from_numpy(msgs).pin_memory(), 64)
    finally:
        engine.HOST_CHUNK_BYTES = old
    assert np.array_equal(d2, golden_npy("cfg1_hh64.npy"))


@pytest.mark.parametrize("width", [64, 128, 256])
@pytest.mark.parametrize("kernel", [KERNEL_DIRECT, KERNEL_TMA])
def test_cfg1_widths_vs_oracle(oracle, width, kernel):
    key = synth.key256()
    msgs = synth.numpy_bytes(1, (4096, 1024))
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, msgs, width, 4)
    got = to_u64(engine.highway_batch(key, dev(msgs), width, 4, kernel=kernel))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("L", [0, 1, 8, 15, 16, 17, 31, 32, 33, 47, 48, 63, 64, 65, 100, 1000,
                               1023, 4095])
def test_fixed_rows_every_kernel(oracle, L):
    """Fixed-length rows through the direct, ring and (rows of <= 64 B)
    staged kernels and KERNEL_AUTO's choice for non-TMA shapes."""
    key = synth.key256()
    n = 3000 if L <= 1024 else 300
    msgs = synth.counter_bytes(90 + L, n * L).reshape(n, L)
    d = dev(msgs)
    kernels = [KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING] + ([KERNEL_STAGED] if L <= 64 else [])
    for width, rounds in ((64, 4), (256, 4), (128, 1), (64, 0)):
        want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, msgs, width, rounds)
        for kernel in kernels:
            got = to_u64(engine.highway_batch(key, d, width, rounds, kernel=kernel))
            assert np.array_equal(got, want), (L, kernel, width, rounds)
    for alg, tree in ((oracle.ALG_SIPTREE, True), (oracle.ALG_SIPHASH, False)):
        want = oracle.batch_fixed(alg, synth.key128(), msgs, 2, 4)
        for kernel in (KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING, KERNEL_STAGED):
            got = to_u64(engine.sip_batch(synth.key128(), d, 2, 4, tree, kernel=kernel))
            assert np.array_equal(got, want), (L, kernel, tree)
    with pytest.raises(ValueError):
        engine.sip_batch(synth.key128(), d, 2, 4, kernel=KERNEL_SPLIT)


@pytest.mark.parametrize("rounds", [0, 1, 2, 3, 5])
def test_reduced_and_extra_rounds(oracle, rounds):
    key = synth.key256()
    msgs = synth.counter_bytes(11, 2000 * 96).reshape(2000, 96)
    for kernel in (KERNEL_DIRECT, KERNEL_TMA):
        got = to_u64(engine.highway_batch(key, dev(msgs), 256, rounds, kernel=kernel))
        assert np.array_equal(got, oracle.batch_fixed(oracle.ALG_HIGHWAY, key, msgs, 256, rounds))


# ---------------------------------------------------------------------------
# every length / residue / alignment, both kernels
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("L", list(range(0, 70)) + [80, 96, 112, 127, 128, 144, 255, 256, 1008,
                                                    1023, 1024, 1040, 4096, 4112])
def test_fixed_lengths(oracle, L):
    key = synth.key256()
    n = 300
    msgs = synth.counter_bytes(20 + L, n * L).reshape(n, L)
    for width in (64, 256):
        want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, msgs, width, 4)
        kernels = [KERNEL_DIRECT, KERNEL_AUTO]
        if L >= 32 and L % 16 == 0:
            kernels.append(KERNEL_TMA)
        for kernel in kernels:
            got = to_u64(engine.highway_batch(key, dev(msgs), width, 4, kernel=kernel))
            assert np.array_equal(got, want), (L, width, kernel)
    for (name, alg, c, d, tree) in (("sip24", oracle.ALG_SIPHASH, 2, 4, False),
                                    ("sip13", oracle.ALG_SIPHASH, 1, 3, False),
                                    ("tree24", oracle.ALG_SIPTREE, 2, 4, True),
                                    ("tree13", oracle.ALG_SIPTREE, 1, 3, True),
                                    ("tree32", oracle.ALG_SIPTREE, 3, 2, True)):
        want = oracle.batch_fixed(alg, synth.key128(), msgs, c, d)
        kernels = [KERNEL_DIRECT] + ([KERNEL_TMA] if L >= 32 and L % 16 == 0 else [])
        for kernel in kernels:
            got = to_u64(engine.sip_batch(synth.key128(), dev(msgs), c, d, tree, kernel=kernel))
            assert np.array_equal(got, want), (name, L, kernel)


@pytest.mark.parametrize("shift", range(1, 16))
def test_unaligned_fixed_base(oracle, shift):
    key = synth.key256()
    n, L = 200, 100
    raw = synth.counter_bytes(31, n * L + 16)
    msgs = raw[shift:shift + n * L].reshape(n, L)
    d_raw = dev(raw)
    d_msgs = d_raw[shift:shift + n * L].view(n, L)
    got = to_u64(engine.highway_batch(key, d_msgs, 256, 4))
    assert np.array_equal(got, oracle.batch_fixed(oracle.ALG_HIGHWAY, key, msgs, 256, 4))
    got = to_u64(engine.sip_batch(synth.key128(), d_msgs, 2, 4, True))
    assert np.array_equal(got, oracle.batch_fixed(oracle.ALG_SIPTREE, synth.key128(), msgs, 2, 4))


def test_backend_equivalence_protocol(oracle):
    """T/test_acceptance.py:75-98: 10^4 random keys x lengths 0..1024."""
    rng = np.random.default_rng(2)
    mism = 0
    b = lh.get_backend()
    for _ in range(10_000):
        key = Key256.from_bytes(rng.integers(0, 256, 32, dtype=np.uint8).tobytes())
        n = int(rng.integers(0, 1025))
        msg = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        if b.hash64(key, msg) != oracle.highway(key.lanes, msg)[0]:
            mism += 1
    assert mism == 0


def test_zero_input_distinctness():
    """T/test_acceptance.py:119-126 shape: zero messages of lengths 0..1024."""
    key = synth.key256()
    lens = np.arange(1025, dtype=np.uint32)
    off = np.zeros(1025, np.uint64)
    off[1:] = np.cumsum(lens[:-1])
    buf = np.zeros(int(lens.sum()), np.uint8)
    d = engine.highway_ragged(key, buf, off, lens, 64)
    assert len(np.unique(d)) == 1025


# ---------------------------------------------------------------------------
# cfg2: remainder sweep, ragged u64 offsets, widths 64/128/256
# ---------------------------------------------------------------------------

def test_cfg2_remainder_sweep(oracle):
    key = synth.key256()
    buf, off, lens = synth.remainder_sweep_bytes(2, 1024, 64)
    d_buf, d_off, d_len = dev(buf), dev(off.view(np.int64)), dev(lens.view(np.int32))
    d256 = to_u64(engine.highway_ragged(key, d_buf, d_off, None, 256))
    assert np.array_equal(np.bitwise_xor.reduce(d256.reshape(1024, 64, 4), axis=1),
                          golden_npy("cfg2_fold256.npy"))
    d128 = to_u64(engine.highway_ragged(key, d_buf, d_off[:-1], d_len, 128))
    assert np.array_equal(d128, d256[:, :2])
    d64 = to_u64(engine.highway_ragged(key, d_buf, d_off, None, 64))
    assert np.array_equal(d64, d256[:, 0])
    assert np.array_equal(np.bitwise_xor.reduce(d64.reshape(1024, 64), axis=1),
                          golden_npy("cfg2_fold64.npy"))
    assert np.array_equal(d256, oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, None, 256, 4))


def test_ragged_sip_family(oracle):
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 300, 5000).astype(np.uint32)
    off = np.zeros(5001, np.uint64)
    off[1:] = np.cumsum(lens)
    buf = synth.counter_bytes(12, int(off[-1]))
    for alg, c, d, tree in ((oracle.ALG_SIPHASH, 2, 4, False), (oracle.ALG_SIPHASH, 1, 3, False),
                            (oracle.ALG_SIPTREE, 2, 4, True), (oracle.ALG_SIPTREE, 1, 3, True)):
        want = oracle.batch_ragged(alg, synth.key128(), buf, off, None, c, d)
        got = engine.sip_ragged(synth.key128(), buf, off, None, c, d, tree)
        assert np.array_equal(got, want)
        got2 = engine.sip_ragged(synth.key128(), buf, off[:-1], lens, c, d, tree)
        assert np.array_equal(got2, want)


def test_ragged_overlapping_and_reordered_offsets(oracle):
    """Offsets need not be sorted or disjoint (per-message independence)."""
    key = synth.key256()
    buf = synth.counter_bytes(13, 10000)
    rng = np.random.default_rng(9)
    off = rng.integers(0, 9000, 3000).astype(np.uint64)
    lens = rng.integers(0, 1000, 3000).astype(np.uint32)
    got = engine.highway_ragged(key, buf, off, lens, 256)
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, lens, 256, 4)
    assert np.array_equal(got, want)


def test_empty_batches():
    key = synth.key256()
    assert engine.highway_batch(key, torch.zeros((0, 64), dtype=torch.uint8, device=DEV)).numel() == 0
    assert engine.highway_batch(key, np.zeros((0, 64), np.uint8)).size == 0
    assert engine.prf64(key, 0, 0).numel() == 0
    d = to_u64(engine.highway_batch(key, torch.zeros((5, 0), dtype=torch.uint8, device=DEV)))
    assert len(set(d.tolist())) == 1


# ---------------------------------------------------------------------------
# PRF mode
# ---------------------------------------------------------------------------

def test_prf_golden_and_windows(oracle):
    key = synth.key256()
    d = to_u64(engine.prf64(key, 0, 4096))
    assert np.array_equal(d, golden_npy("prf_0_4096.npy"))
    d2 = to_u64(engine.prf64(key, 1000, 100))
    assert np.array_equal(d2, d[1000:1100])
    start = (1 << 40) + 12345
    assert np.array_equal(to_u64(engine.prf64(key, start, 5000, 3)),
                          oracle.prf64(key, start, 5000, 3))


# ---------------------------------------------------------------------------
# synthetic generator: device == numpy twin
# ---------------------------------------------------------------------------

def test_synth_device_matches_numpy():
    for nbytes, off in ((1000, 0), (1 << 20, 12345), (13, 7), (8, 0)):
        t = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
        synth.fill_device(t, 6, off)
        assert np.array_equal(t.cpu().numpy(), synth.counter_bytes(6, nbytes, off))
    L = torch.empty(100000, dtype=torch.int32, device=DEV)
    synth.lengths_device(L, 3, 8, 64)
    assert np.array_equal(L.cpu().numpy().view(np.uint32), synth.lengths(3, 100000, 8, 64))


# ---------------------------------------------------------------------------
# split-state long-message kernel (2 threads per message)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n,L", [(1, 128), (15, 256), (16, 640), (17, 1024), (300, 4096),
                                 (33, 65536), (40, 128 * 37)])
def test_split_kernel_vs_oracle(oracle, n, L):
    key = synth.key256()
    msgs = synth.counter_bytes(50 + n, n * L).reshape(n, L)
    d = dev(msgs)
    for width in (64, 128, 256):
        want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, msgs, width, 4)
        got = to_u64(engine.highway_batch(key, d, width, 4, kernel=KERNEL_SPLIT))
        assert np.array_equal(got, want), (n, L, width)
    for rounds in (0, 1, 5):
        want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, msgs, 256, rounds)
        got = to_u64(engine.highway_batch(key, d, 256, rounds, kernel=KERNEL_SPLIT))
        assert np.array_equal(got, want), (n, L, rounds)


def test_split_kernel_rejects_unsupported_shapes():
    key = synth.key256()
    with pytest.raises(ValueError):
        engine.highway_batch(key, torch.zeros((4, 96), dtype=torch.uint8, device=DEV),
                             kernel=KERNEL_SPLIT)
    with pytest.raises(ValueError):
        engine.sip_batch(synth.key128(), torch.zeros((4, 128), dtype=torch.uint8, device=DEV),
                         kernel=KERNEL_SPLIT)


# ---------------------------------------------------------------------------
# ragged short-message kernel: warp-staged fast path and its fallback
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["packed", "scattered", "mixed_long", "wide_span"])
def test_ragged_short_paths(oracle, case):
    rng = np.random.default_rng({"packed": 1, "scattered": 2, "mixed_long": 3, "wide_span": 4}[case])
    n = 20000
    if case == "packed":          # cfg3 shape: packed, every residue 0..64
        lens = rng.integers(0, 65, n).astype(np.uint32)
        off = np.zeros(n, np.uint64)
        off[1:] = np.cumsum(lens[:-1])
        buf = synth.counter_bytes(60, int(lens.sum()) + 1)
    elif case == "scattered":     # unsorted / overlapping offsets inside a 1.5 KB window per warp
        lens = rng.integers(0, 65, n).astype(np.uint32)
        warp_base = (np.arange(n) // 32) * 2000
        off = (warp_base + rng.integers(0, 1500, n)).astype(np.uint64)
        buf = synth.counter_bytes(61, int(off.max()) + 70)
    elif case == "mixed_long":    # some warps contain a message > 64 B (fallback)
        lens = rng.integers(0, 65, n).astype(np.uint32)
        lens[rng.choice(n, 200, replace=False)] = rng.integers(65, 600, 200)
        off = np.zeros(n, np.uint64)
        off[1:] = np.cumsum(lens[:-1])
        buf = synth.counter_bytes(62, int(lens.sum()) + 1)
    else:                         # short messages but spans wider than the staging cap
        lens = rng.integers(1, 65, n).astype(np.uint32)
        off = (np.arange(n, dtype=np.uint64) * 97) % np.uint64(n * 64)
        buf = synth.counter_bytes(63, n * 64 + 70)
    for width in (64, 256):
        got = engine.highway_ragged(synth.key256(), buf, off, lens, width)
        want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), buf, off, lens, width, 4)
        assert np.array_equal(got, want), (case, width)
    got = engine.highway_ragged(synth.key256(), buf, off, lens, 64, rounds=2)
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), buf, off, lens, 64, 2)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------------------
# every ragged kernel on every layout (KERNEL_AUTO picks by mean length)
# ---------------------------------------------------------------------------

def _ragged_layout(case):
    rng = np.random.default_rng({"sweep": 21, "long": 22, "scattered": 23, "tiny": 24}[case])
    if case == "sweep":        # cfg2 shape (small): every length 0..1023 twice, packed
        lens = np.repeat(np.arange(1024, dtype=np.uint32), 2)
    elif case == "long":       # ring main loop (>= 2 x 4 packets) plus tails
        lens = rng.integers(0, 3000, 3000).astype(np.uint32)
    elif case == "scattered":  # unsorted, overlapping spans
        lens = rng.integers(0, 1200, 4000).astype(np.uint32)
    else:                      # short keys, empty messages included
        lens = rng.integers(0, 70, 9000).astype(np.uint32)
    if case == "scattered":
        total = 200000
        off = rng.integers(0, total - 1200, len(lens)).astype(np.uint64)
    else:
        off = np.zeros(len(lens), np.uint64)
        off[1:] = np.cumsum(lens[:-1])
        total = int(lens.sum())
    # The last message ends exactly at the end of the allocation (no read past it).
    buf = synth.counter_bytes(80, max(total, 1))
    return buf, off, lens


@pytest.mark.parametrize("case", ["sweep", "long", "scattered", "tiny"])
@pytest.mark.parametrize("kernel", [KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING, KERNEL_STAGED])
def test_ragged_kernels_highway(oracle, case, kernel):
    buf, off, lens = _ragged_layout(case)
    d_buf, d_off, d_len = dev(buf), dev(off.view(np.int64)), dev(lens.view(np.int32))
    for width, rounds in ((64, 4), (128, 4), (256, 4), (64, 0), (64, 1), (256, 2), (64, 5)):
        got = to_u64(engine.highway_ragged(synth.key256(), d_buf, d_off, d_len, width, rounds,
                                           kernel=kernel))
        want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), buf, off, lens, width,
                                   rounds)
        assert np.array_equal(got, want), (case, width, rounds)


@pytest.mark.parametrize("shift", [1, 2, 3, 5, 7])
def test_ragged_ring_unaligned_device_buffer(oracle, shift):
    buf, off, lens = _ragged_layout("long")
    raw = np.concatenate([np.full(shift, 0xA5, np.uint8), buf])
    d_buf = dev(raw)[shift:]
    got = to_u64(engine.highway_ragged(synth.key256(), d_buf, dev(off.view(np.int64)),
                                       dev(lens.view(np.int32)), 256, kernel=KERNEL_DIRECT))
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), buf, off, lens, 256, 4)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("case", ["sweep", "long", "tiny", "scattered"])
@pytest.mark.parametrize("kernel", [KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING, KERNEL_STAGED])
def test_ragged_kernels_sip(oracle, case, kernel):
    buf, off, lens = _ragged_layout(case)
    for alg, c, d, tree in ((oracle.ALG_SIPHASH, 2, 4, False), (oracle.ALG_SIPHASH, 1, 3, False),
                            (oracle.ALG_SIPTREE, 2, 4, True), (oracle.ALG_SIPTREE, 1, 3, True)):
        got = engine.sip_ragged(synth.key128(), buf, off, lens, c, d, tree, kernel=kernel)
        want = oracle.batch_ragged(alg, synth.key128(), buf, off, lens, c, d)
        assert np.array_equal(got, want), (case, c, d, tree)


def test_ragged_kernel_choice_rejects_unknown():
    buf, off, lens = _ragged_layout("tiny")
    with pytest.raises(ValueError):
        engine.highway_ragged(synth.key256(), buf, off, lens, kernel=KERNEL_TMA)
    with pytest.raises(ValueError):
        engine.sip_ragged(synth.key128(), buf, off, lens, kernel=KERNEL_SPLIT)


@pytest.mark.parametrize("shift", [1, 3, 8, 13])
def test_ragged_unaligned_device_buffer(oracle, shift):
    """d_buf need not be aligned: the warp-staged kernel aligns on the absolute
    address."""
    rng = np.random.default_rng(shift)
    n = 5000
    lens = rng.integers(0, 65, n).astype(np.uint32)
    off = np.zeros(n, np.uint64)
    off[1:] = np.cumsum(lens[:-1])
    raw = synth.counter_bytes(70 + shift, int(lens.sum()) + 64)
    d_raw = dev(raw)
    d_buf = d_raw[shift:]
    buf = raw[shift:]
    got = to_u64(engine.highway_ragged(synth.key256(), d_buf, dev(off.view(np.int64)),
                                       dev(lens.view(np.int32)), 256))
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), buf, off, lens, 256, 4)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("form", ["offsets_n1", "offsets_lengths", "scattered"])
def test_ragged_host_pipelined_chunks(oracle, form):
    """Host ragged batches stream through the GPU in message-range chunks;
    force many small chunks and compare with the oracle."""
    rng = np.random.default_rng(11)
    n = 30000
    lens = rng.integers(0, 300, n).astype(np.uint32)
    if form == "scattered":
        off = rng.integers(0, 2_000_000, n).astype(np.uint64)
        buf = synth.counter_bytes(90, 2_000_400)
    else:
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        buf = synth.counter_bytes(91, int(off[-1]) + 7)
    old = engine.HOST_CHUNK_BYTES
    engine.HOST_CHUNK_BYTES = 100_000
    try:
        for width in (64, 256):
            if form == "offsets_n1":
                got = engine.highway_ragged(synth.key256(), buf, off, None, width)
                want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), buf, off, None,
                                           width, 4)
            else:
                o = off[:n]
                got = engine.highway_ragged(synth.key256(), buf, o, lens, width)
                want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), buf, o, lens,
                                           width, 4)
            assert np.array_equal(got, want), (form, width)
        o = off[:n]
        got = engine.sip_ragged(synth.key128(), buf, o, lens, 2, 4, tree=True)
        assert np.array_equal(got, oracle.batch_ragged(oracle.ALG_SIPTREE, synth.key128(), buf,
                                                       o, lens, 2, 4))
    finally:
        engine.HOST_CHUNK_BYTES = old


def test_multi_device_host_batches(oracle):
    """multi.py: shards on several devices in threads (here the one GPU,
    listed twice and three times: shards run concurrently on it)."""
    from paper_1612_06257_b200 import multi

    key = synth.key256()
    msgs = synth.counter_bytes(41, 3001 * 1024).reshape(3001, 1024)
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, msgs, 256, 4)
    for devs in ([0], [0, 0], [0, 0, 0]):
        assert np.array_equal(multi.highway_batch(key, msgs, 256, devices=devs), want), devs
    got = multi.sip_batch(synth.key128(), msgs, 1, 3, True, devices=[0, 0])
    assert np.array_equal(got, oracle.batch_fixed(oracle.ALG_SIPTREE, synth.key128(), msgs, 1, 3))
    lens = synth.lengths(5, 20000, 0, 200)
    off = np.zeros(20001, np.uint64)
    off[1:] = np.cumsum(lens)
    buf = synth.counter_bytes(42, int(off[-1]))
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, None, 64, 4)
    assert np.array_equal(multi.highway_ragged(key, buf, off, None, 64, devices=[0, 0]), want)
    assert np.array_equal(multi.highway_ragged(key, buf, off[:-1], lens, 64, devices=[0, 0, 0]),
                          want)


def test_read_only_host_inputs_zero_copy(oracle, tmp_path):
    """Read-only host memory (a file opened as np.memmap mode "r",
    np.frombuffer of bytes) is hashed without copies or warnings."""
    import warnings

    n, L = 4096, 96
    data = synth.counter_bytes(12, n * L)
    path = tmp_path / "msgs.bin"
    data.tofile(path)
    mm = np.memmap(path, dtype=np.uint8, mode="r", shape=(n, L))
    key = synth.key256()
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, data.reshape(n, L), 64, 4)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        assert np.array_equal(engine.highway_batch(key, mm), want)
        ro = np.frombuffer(data.tobytes(), np.uint8)
        off = np.arange(n + 1, dtype=np.uint64) * L
        assert np.array_equal(engine.highway_ragged(key, ro, off), want)
