"""The reference module's host-level helpers, mirrored in
paper_1612_06257_b200.highway (CPU; no device).

One test per reference test, same assertions: T/test_highway.py:53-75,
93-118, 135-141, 196-222 and T/test_zipper.py:9-32.  The device-level
ones (update, update_remainder, finalize, hashes) are in
tests/test_gpu_highway_module.py.
"""
import numpy as np
import pytest

from paper_1612_06257_b200 import highway
from paper_1612_06257_b200.highway import (INIT0, INIT1, ZIPPER_OFFSETS, Key256, initialize,
                                           packet_lanes, permute_lanes, remainder_packet,
                                           zipper_merge)

M64 = (1 << 64) - 1


@pytest.fixture
def ramp_key():
    return Key256.from_bytes(bytes(range(32)))


def test_init_constants_cover_every_bit():
    combined = 0
    for lane in INIT0:
        combined |= lane
    assert combined == M64


def test_initialize_mixes_key_into_both_halves(ramp_key):
    v0, v1, mul0, mul1 = initialize(ramp_key)
    assert mul0 == INIT0 and mul1 == INIT1
    for i in range(4):
        assert v0[i] == ramp_key.lanes[i] ^ INIT0[i]
        rot = ((ramp_key.lanes[i] >> 32) | (ramp_key.lanes[i] << 32)) & M64
        assert v1[i] == rot ^ INIT1[i]


def test_zero_key_initial_state_is_the_constants():
    v0, v1, _, _ = initialize(Key256((0, 0, 0, 0)))
    assert v0 == INIT0 and v1 == INIT1


def test_remainder_packet_r4():
    packet = remainder_packet(b"\x01\x02\x03\x04")
    assert packet[:4] == b"\x01\x02\x03\x04" and packet[4:] == bytes(28)


def test_remainder_packet_r3():
    packet = remainder_packet(b"\x01\x02\x03")
    assert packet[:28] == bytes(28) and packet[28:] == b"\x01\x02\x03\x00"


def test_remainder_packet_r7():
    packet = remainder_packet(bytes(range(1, 8)))
    assert packet[:4] == b"\x01\x02\x03\x04"
    assert packet[4:28] == bytes(24)
    assert packet[28:] == b"\x05\x06\x07\x00"


def test_remainder_packet_rejects_bad_lengths():
    for bad in (b"", bytes(32)):
        with pytest.raises(ValueError):
            remainder_packet(bad)


def test_remainder_packet_matches_golden(golden):
    for r, hexp in golden["remainder_packets"].items():
        assert remainder_packet(bytes(range(1, int(r) + 1))).hex() == hexp


def test_permute_is_an_involution():
    rng = np.random.default_rng(0xC0FFEE)
    lanes = tuple(int(x) for x in rng.integers(0, 1 << 64, 4, dtype=np.uint64))
    assert permute_lanes(permute_lanes(lanes)) == lanes
    a, b, c, d = lanes
    rot = lambda x: ((x >> 32) | (x << 32)) & M64
    assert permute_lanes(lanes) == (rot(c), rot(d), rot(a), rot(b))


def test_packet_lanes_layout():
    packet = bytes(range(32))
    lanes = packet_lanes(packet)
    assert lanes[0] == int.from_bytes(packet[:8], "little")
    assert lanes[3] == int.from_bytes(packet[24:], "little")
    with pytest.raises(ValueError):
        packet_lanes(bytes(31))


def test_key256_round_trip():
    raw = bytes(range(100, 132))
    assert Key256.from_bytes(raw).to_bytes() == raw
    with pytest.raises(ValueError):
        Key256.from_bytes(bytes(31))


def test_state_arguments_validated_before_device():
    with pytest.raises(ValueError):
        highway.update_remainder(initialize(bytes(32)), b"")
    with pytest.raises(ValueError):
        highway.update_remainder(initialize(bytes(32)), bytes(32))
    with pytest.raises(ValueError):
        highway.finalize(initialize(bytes(32)), 96)
    with pytest.raises(ValueError):
        highway.update(initialize(bytes(32)), (0, 0, 0))


# T/test_zipper.py
def test_offset_table_is_a_permutation():
    assert sorted(ZIPPER_OFFSETS) == list(range(16))


def test_zipper_ramp_bytes():
    assert zipper_merge(bytes(range(16))) == bytes(ZIPPER_OFFSETS)


def test_zipper_identical_bytes_unchanged():
    assert zipper_merge(b"\xab" * 16) == b"\xab" * 16


def test_zipper_multiset_preserved_on_random_inputs():
    rng = np.random.default_rng(3)
    for _ in range(100):
        half = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        assert sorted(zipper_merge(half)) == sorted(half)


def test_zipper_wrong_length_rejected():
    for bad in (bytes(15), bytes(17)):
        with pytest.raises(ValueError):
            zipper_merge(bad)
