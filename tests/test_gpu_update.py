"""The raw Update and its inverse on the device.

Parity pins: the reference's own update / update_inverse outputs on the
acceptance gate's 100,000 random states (tests/golden/update_states.npz,
generated from S/highway.py:130-173), the bijectivity protocol of
T/test_update.py:56-67 and T/test_acceptance.py:42-63, and the v0-flip
property of T/test_update.py:70-84 -- all through the C ABI
(lh_highway_update_states / lh_highway_bijectivity).
"""
import hashlib
import time

import numpy as np
import pytest
import torch

from conftest import golden_npy
from paper_1612_06257_b200 import engine, highway, synth

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u8").tobytes()).hexdigest()


def _acceptance_raw():
    return np.random.default_rng(1).integers(0, 1 << 64, size=(100_000, 20), dtype=np.uint64)


def test_update_and_inverse_match_reference():
    g = golden_npy("update_states.npz")
    raw = _acceptance_raw()
    fwd = engine.update_states(raw[:, :16], raw[:, 16:])
    inv = engine.update_states(raw[:, :16], raw[:, 16:], inverse=True)
    assert np.array_equal(fwd[:256], g["fwd"])
    assert np.array_equal(inv[:256], g["inv"])
    assert [_sha(fwd), _sha(inv)] == [str(x) for x in g["sha"]]


def test_update_matches_oracle_random(oracle, rng):
    """T/test_update.py:49-53, at 2^20 states."""
    raw = rng.integers(0, 1 << 64, size=(1 << 20, 20), dtype=np.uint64)
    got = engine.update_states(raw[:, :16], raw[:, 16:])
    assert np.array_equal(got, oracle.update_states(raw[:, :16], raw[:, 16:]))
    zero = np.zeros((1 << 20, 4), np.uint64)
    assert np.array_equal(engine.update_states(raw[:, :16], zero),
                          oracle.update_states(raw[:, :16], zero))


def test_acceptance_gate_bijectivity():
    """T/test_acceptance.py:42-63: 100,000 round trips, 0 failures, < 5 s
    (here through the device, on resident tensors, in place)."""
    raw = _acceptance_raw()
    dev = torch.device("cuda", 0)
    st = torch.from_numpy(raw[:, :16].view(np.int64).copy()).to(dev)
    pk = torch.from_numpy(raw[:, 16:].view(np.int64).copy()).to(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    engine.update_states(st, pk)
    engine.update_states(st, pk, inverse=True)
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    assert np.array_equal(engine.to_u64(st), raw[:, :16])
    assert elapsed < 5.0
    engine.update_states(st, pk, inverse=True)  # T/test_update.py:63-67: other order
    engine.update_states(st, pk)
    assert np.array_equal(engine.to_u64(st), raw[:, :16])


def test_v0_flip_reaches_multipliers(rng):
    """T/test_update.py:70-84."""
    n = 10_000
    raw = rng.integers(0, 1 << 64, size=(n, 20), dtype=np.uint64)
    bits = rng.integers(0, 256, n)
    flipped = raw[:, :16].copy()
    flipped[np.arange(n), bits >> 6] ^= np.left_shift(np.uint64(1), (bits & 63).astype(np.uint64))
    a = engine.update_states(raw[:, :16], raw[:, 16:])
    b = engine.update_states(flipped, raw[:, 16:])
    assert np.any(a[:, 8:] != b[:, 8:], axis=1).mean() >= 0.99


def test_one_shot_mirror(oracle, ramp_key):
    """highway.update / update_inverse keep the reference's tuple signature."""
    s = highway.initialize(ramp_key)
    p = (1, 2, 3, (1 << 64) - 1)
    u = highway.update(s, p)
    flat = np.array([[x for lanes in s for x in lanes]], np.uint64)
    want = oracle.update_states(flat, np.array([p], np.uint64))[0]
    assert [x for lanes in u for x in lanes] == [int(x) for x in want]
    assert highway.update_inverse(u, p) == s


def test_device_self_test_matches_oracle(oracle):
    """lh_highway_bijectivity: synthetic cases generated on the device; the
    forward fold is checked against the oracle on the same words."""
    n = 1 << 18
    words = synth.counter_bytes(42, 20 * 8 * n).view("<u8").reshape(n, 20)
    fwd = oracle.update_states(words[:, :16], words[:, 16:])
    fold = int(np.bitwise_xor.reduce(fwd.reshape(-1)))
    assert engine.bijectivity(42, n) == (0, fold)
    assert engine.bijectivity(42, 0) == (0, 0)


def test_device_self_test_at_scale():
    """2^30 round trips on the device: the bijection the reference checks on
    100,000 states."""
    fails, _ = engine.bijectivity(7, 1 << 30)
    assert fails == 0
