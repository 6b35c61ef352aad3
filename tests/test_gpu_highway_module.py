"""The reference module lanehash.highway's device-level functions, mirrored
in paper_1612_06257_b200.highway and computed by the CUDA library.

One test per reference test, same assertions (T/test_highway.py:77-156),
plus pins of update_remainder / finalize on raw states against the
reference's own outputs (tests/golden/update_states.npz).
"""
import numpy as np
import pytest

from conftest import golden_npy
from paper_1612_06257_b200 import engine, highway
from paper_1612_06257_b200.highway import (digest256_to_bytes, finalize, hash64, hash256,
                                           initialize, update, update_remainder)

pytestmark = pytest.mark.gpu


def ramp(n):
    return bytes(i & 0xFF for i in range(n))


def _state(row):
    return tuple(tuple(int(x) for x in row[i:i + 4]) for i in range(0, 16, 4))


def random_state(rng):
    return _state(rng.integers(0, 1 << 64, 16, dtype=np.uint64))


def test_frozen_digest64(golden, ramp_key):
    for n, hexd in golden["frozen_64"].items():
        assert hash64(ramp_key, ramp(int(n))) == int(hexd, 16), n


def test_frozen_digest256(golden, ramp_key):
    for n, hexd in golden["frozen_256_hex"].items():
        assert digest256_to_bytes(hash256(ramp_key, ramp(int(n)))).hex() == hexd


def test_digest64_is_lane0_of_digest256(ramp_key, rng):
    for _ in range(50):
        msg = rng.integers(0, 256, int(rng.integers(0, 200)), dtype="uint8").tobytes()
        assert hash64(ramp_key, msg) == hash256(ramp_key, msg)[0]


def test_length_mod_32_distinguishes_zero_tails(ramp_key):
    assert hash64(ramp_key, bytes(30)) != hash64(ramp_key, bytes(31))
    assert len({hash64(ramp_key, bytes(n)) for n in range(33)}) == 33


def test_update_remainder_rotation_depends_on_length(rng):
    state = random_state(rng)
    assert update_remainder(state, b"\x00") != update_remainder(state, b"\x00\x00")


def test_finalize_widths_agree_on_lane0(rng):
    state = random_state(rng)
    assert finalize(state, 64) == finalize(state, 256)[0]
    assert finalize(state, 128) == finalize(state, 256)[:2]  # derived width
    with pytest.raises(ValueError):
        finalize(state, 96)


def test_finalize_round_count_changes_digest(ramp_key):
    msg = ramp(17)
    assert len({hash64(ramp_key, msg, rounds=r) for r in (1, 2, 3, 4)}) == 4


def test_state_functions_match_reference_outputs():
    g = golden_npy("update_states.npz")
    for i, row in enumerate(g["raw"][:64]):
        state = _state(row[:16])
        tail = row[16:20].astype("<u8").tobytes()[:1 + i % 31]
        assert update_remainder(state, tail) == _state(g["rem"][i]), i
        assert finalize(state, 256, rounds=i % 6) == tuple(int(x) for x in g["fin"][i]), i


def test_batched_state_functions_match_reference_outputs():
    """The same 256 cases as one batch each (engine.remainder_states /
    finalize_states, one launch)."""
    g = golden_npy("update_states.npz")
    raw = g["raw"]
    tails = np.zeros((256, 32), np.uint8)
    tails[:] = raw[:, 16:20].astype("<u8").view(np.uint8).reshape(256, 32)
    r = np.array([1 + i % 31 for i in range(256)], np.uint32)
    mask = np.arange(32)[None, :] < r[:, None]
    tails_masked = np.where(mask, tails, 0).astype(np.uint8)
    assert np.array_equal(engine.remainder_states(raw[:, :16], tails, r), g["rem"])
    assert np.array_equal(engine.remainder_states(raw[:, :16], tails_masked, r), g["rem"])
    for rounds in range(6):
        sel = np.arange(256) % 6 == rounds
        got = engine.finalize_states(raw[sel, :16], 256, rounds)
        assert np.array_equal(got, g["fin"][sel]), rounds


def test_one_shot_equals_composed_primitives(ramp_key):
    """hash64 = initialize, update per packet, update_remainder, finalize
    (S/highway.py:237-249), each step on the device."""
    for n in (0, 5, 32, 45, 100):
        msg = ramp(n)
        s = initialize(ramp_key)
        full = n - n % 32
        for k in range(0, full, 32):
            s = update(s, highway.packet_lanes(msg[k:k + 32]))
        if n % 32:
            s = update_remainder(s, msg[full:])
        assert finalize(s, 64) == hash64(ramp_key, msg)
        assert finalize(s, 256) == hash256(ramp_key, msg)
