"""Registry / _kernels drop-in on the GPU: every callable a reference caller
reaches through ``lanehash.registry`` (S/registry.py:106-160) or
``lanehash._kernels`` (S/_kernels.py:150-274) gives the oracle's digest, with
the reference's return types (int for 64-bit digests, tuple of lanes for
256-bit, LE byte images from ``digest``)."""
import numpy as np
import pytest

from paper_1612_06257_b200 import _kernels, quality, registry, synth
from paper_1612_06257_b200.highway import digest256_to_bytes

pytestmark = pytest.mark.gpu

KEY32 = bytes(range(32))
KEY16 = bytes(range(16))
LENGTHS = (0, 1, 7, 8, 31, 32, 33, 63, 64, 65, 200, 1024)


def _msg(n):
    return bytes((7 * i + 3) & 0xFF for i in range(n))


@pytest.mark.parametrize("name,alg,c,d", [("siphash24", 1, 2, 4), ("siphash13", 1, 1, 3),
                                          ("siptree24", 2, 2, 4), ("siptree13", 2, 1, 3)])
def test_sip_family_callables(oracle, name, alg, c, d):
    a = registry.get_algorithm(name)
    ref = oracle.siptree if alg == 2 else oracle.siphash
    k = np.frombuffer(KEY16, np.uint64)
    for n in LENGTHS:
        want = ref(k, _msg(n), c, d)
        got = a.hash64(KEY16, _msg(n))
        assert isinstance(got, int) and got == want
        assert a.digest(KEY16, _msg(n)) == want.to_bytes(8, "little")
        h = a.make_hasher(KEY16)
        h.append(_msg(n)[:5]).append(_msg(n)[5:])
        fin = h.finish()
        assert isinstance(fin, int) and fin == want


def test_highway_callables(oracle):
    k = np.frombuffer(KEY32, np.uint64)
    a64, a128, a256 = (registry.get_algorithm(f"highway{w}") for w in (64, 128, 256))
    for n in LENGTHS:
        want = oracle.highway(k, _msg(n))
        assert a64.hash64(KEY32, _msg(n)) == want[0]
        assert a64.digest(KEY32, _msg(n)) == want[0].to_bytes(8, "little")
        assert a256.digest(KEY32, _msg(n)) == digest256_to_bytes(want)
        assert a128.digest(KEY32, _msg(n)) == digest256_to_bytes(want)[:16]
        h = a64.make_hasher(KEY32)
        h.append(_msg(n))
        assert h.finish() == want[0]
        h = a256.make_hasher(KEY32)
        h.append(_msg(n)[:33]).append(_msg(n)[33:])
        fin = h.finish()
        assert isinstance(fin, tuple) and fin == want


def test_digest_batch_matches_digest():
    for name in registry.VECTOR_ALGORITHMS:
        a = registry.get_algorithm(name)
        key = KEY32 if a.key_size == 32 else KEY16
        msgs = [_msg(n) for n in LENGTHS]
        rows = a.digest_batch(key, msgs)
        assert [r.tobytes() for r in rows] == [a.digest(key, m) for m in msgs]


def test_finalization_variant(oracle):
    k = np.frombuffer(KEY32, np.uint64)
    for rounds in (1, 2, 3, 4):
        fn = registry.finalization_variant(rounds)
        assert fn(KEY32, _msg(40)) == oracle.highway(k, _msg(40), rounds)[0]


def test_kernels_hash_batch(oracle):
    key = synth.key256()
    for L in (0, 8, 33, 1024):
        msgs = synth.numpy_bytes(L + 1, (257, L))
        for algo, p1, p2, alg in ((0, 4, 0, oracle.ALG_HIGHWAY), (0, 2, 0, oracle.ALG_HIGHWAY),
                                  (1, 2, 4, oracle.ALG_SIPHASH), (1, 1, 3, oracle.ALG_SIPHASH),
                                  (2, 2, 4, oracle.ALG_SIPTREE)):
            got = _kernels.hash_batch(algo, key, msgs, p1, p2)
            want = oracle.batch_fixed(alg, key, msgs, 64 if algo == 0 else p1,
                                      p1 if algo == 0 else p2)
            assert got.dtype == np.uint64 and np.array_equal(got, want), (L, algo, p1, p2)


def test_kernels_single_message_functions(oracle):
    key = synth.key256()
    m = np.frombuffer(_msg(77), np.uint8)
    want = oracle.highway(key, m.tobytes(), 3)
    assert _kernels.highway64(key, m, 3) == want[0]
    assert _kernels.highway256(key, m, 3) == want
    assert _kernels.siphash(key, m, 2, 4) == oracle.siphash(key, m.tobytes(), 2, 4)
    assert _kernels.siptreehash(key, m, 1, 3) == oracle.siptree(key, m.tobytes(), 1, 3)


def test_kernels_avalanche_counts(oracle):
    key = synth.key256()
    msgs = synth.numpy_bytes(9, (300, 6))
    before = msgs.copy()
    for algo, p1, p2, alg in ((0, 4, 0, oracle.ALG_HIGHWAY), (1, 2, 4, oracle.ALG_SIPHASH),
                              (2, 1, 3, oracle.ALG_SIPTREE)):
        got = _kernels.avalanche_counts(algo, key, msgs, p1, p2)
        want = oracle.avalanche_counts(alg, key, msgs, p1, p2)
        assert np.array_equal(got, want)
    assert np.array_equal(msgs, before)


def test_kernel_and_host_paths_agree():
    """T/test_quality.py:107-113: the device tally and the harness's host loop
    over ``fn`` give identical counts."""
    fast = quality.HashUnderTest.from_name("highway64")
    slow = quality.HashUnderTest(fast.name, fast.key_size, fast.fn, kernel=None)
    a = quality.avalanche_bias(fast, size=4, iterations=40, seed=3)
    b = quality.avalanche_bias(slow, size=4, iterations=40, seed=3)
    assert np.array_equal(a.counts, b.counts)
