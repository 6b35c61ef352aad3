"""lanehash.sip's device-level functions, mirrored in
paper_1612_06257_b200.sip and computed by the CUDA library: one test per
reference test, same assertions (T/test_sip.py:84-135, T/test_tree.py:40-67),
with the CPU oracle standing in for the reference's independent
transcription (oracle/lh_oracle.c, pinned by tests/test_oracle.py)."""
import struct

import numpy as np
import pytest

from paper_1612_06257_b200 import engine
from paper_1612_06257_b200.sip import (SIPHASH_13, SIPHASH_24, Key128, deinterleave, sip_round,
                                       siphash, siptreehash)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref_key():
    return Key128.from_bytes(bytes(range(16)))


def test_published_vectors(golden, ref_key):
    message = bytes(range(64))
    for n, expected in enumerate(golden["siphash24_reference_le_hex"]):
        assert struct.pack("<Q", siphash(ref_key, message[:n])).hex() == expected, n


def test_matches_independent_transcription(oracle, rng):
    for _ in range(256):
        key = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        msg = rng.integers(0, 256, int(rng.integers(0, 70)), dtype=np.uint8).tobytes()
        lanes = struct.unpack("<2Q", key)
        for p in (SIPHASH_24, SIPHASH_13):
            assert siphash(Key128.from_bytes(key), msg, p) == oracle.siphash(lanes, msg, p.c, p.d)


def test_sip_round_frozen_pair(golden):
    out = sip_round(sip_round((1, 2, 3, 4)))
    assert [f"{x:016x}" for x in out] == golden["sip_round_1234_twice"]
    assert out == (9263201270060220426, 2307743542053503000, 5255419393243893904,
                   10208987565802066018)


def test_sip_round_zero_fixed_point():
    assert sip_round((0, 0, 0, 0)) == (0, 0, 0, 0)


def test_sip_round_not_identity():
    state = (1, 2, 3, 4)
    assert sip_round(state) != state
    assert sip_round(sip_round(state)) != state


def test_sip_round_batch_vs_oracle(oracle, rng):
    import ctypes

    st = rng.integers(0, 1 << 64, (4096, 4), dtype=np.uint64)
    for rounds in (0, 1, 2, 5):
        got = engine.sip_round_states(st, rounds)
        for i in range(0, 4096, 97):
            v = st[i].copy()
            for _ in range(rounds):
                oracle.lib().lh_ref_sip_round(v.ctypes.data_as(ctypes.c_void_p))
            assert np.array_equal(got[i], v), (rounds, i)


def test_round_counts_matter(ref_key):
    msg = b"round count probe"
    assert siphash(ref_key, msg, SIPHASH_24) != siphash(ref_key, msg, SIPHASH_13)


def test_empty_differs_from_single_zero_byte(ref_key):
    assert siphash(ref_key, b"") != siphash(ref_key, b"\x00")


def test_key_matters():
    assert siphash(Key128(0, 0), b"key probe") != siphash(Key128(1, 0), b"key probe")


def test_tree_differs_from_flat(ref_key, rng):
    for _ in range(100):
        msg = rng.integers(0, 256, 64, dtype=np.uint8).tobytes()
        assert siptreehash(ref_key, msg) != siphash(ref_key, msg)


def test_tree_is_order_sensitive(ref_key):
    a, b = bytes(range(32)), bytes(range(32, 64))
    assert siptreehash(ref_key, a + b) != siptreehash(ref_key, b + a)


def test_tree_equals_manual_deinterleave_and_fold(ref_key, rng):
    for params in (SIPHASH_24, SIPHASH_13):
        for n in (0, 1, 31, 32, 33, 64, 100):
            msg = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
            lane_digests = [siphash(ref_key, lane, params) for lane in deinterleave(msg)]
            folded = siphash(ref_key, struct.pack("<4Q", *lane_digests), params)
            assert siptreehash(ref_key, msg, params) == folded


def test_tree_zero_padding_contract(ref_key):
    """T/test_tree.py:61-67: length-blind within a 32-byte block."""
    assert siptreehash(ref_key, bytes(1)) == siptreehash(ref_key, bytes(32))
    assert len({siptreehash(ref_key, bytes(n)) for n in (0, 32, 64, 96)}) == 4
