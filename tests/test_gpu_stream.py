"""Streaming (incremental) hashing on the device (§8f row 1).

Parity pins: chunk-split invariance against the one-shot digest, as the
reference tests it (T/test_highway.py:156-193, T/test_acceptance.py:101-116,
T/test_sip.py:155-176, T/test_tree.py:70-91), with the one-shot digest from
the CPU oracle; misuse raises RuntimeError like the reference hashers.
"""
import numpy as np
import pytest
import torch

import paper_1612_06257_b200 as lh
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import ALG_HIGHWAY, ALG_SIPHASH, ALG_SIPTREE, to_u64
from paper_1612_06257_b200.sip import SIPHASH_13, SIPHASH_24, Key128

pytestmark = pytest.mark.gpu


def ramp(n):
    return bytes(i & 0xFF for i in range(n))


def _random_chunked_batch(rng, n, max_len, max_chunks):
    """n messages with random lengths and random cut points, as a list of
    per-append ragged (buf, offsets, lengths) triples plus the messages."""
    lens = rng.integers(0, max_len + 1, n)
    msgs = [synth.counter_bytes(1000 + i, int(L)) for i, L in enumerate(lens)]
    ncuts = int(rng.integers(1, max_chunks + 1))
    cuts = [np.sort(rng.integers(0, int(L) + 1, ncuts - 1)) for L in lens]
    appends = []
    for k in range(ncuts):
        parts = []
        for i in range(n):
            b = [0] + list(cuts[i]) + [int(lens[i])]
            parts.append(msgs[i][b[k]:b[k + 1]])
        plens = np.array([len(p) for p in parts], np.uint32)
        off = np.zeros(n, np.uint64)
        off[1:] = np.cumsum(plens[:-1])
        buf = np.concatenate(parts) if plens.sum() else np.zeros(1, np.uint8)
        appends.append((buf, off, plens))
    return msgs, appends


@pytest.mark.parametrize("alg", [ALG_HIGHWAY, ALG_SIPHASH, ALG_SIPTREE])
def test_batch_chunk_split_invariance(oracle, alg):
    rng = np.random.default_rng(100 + alg)
    n = 777
    msgs, appends = _random_chunked_batch(rng, n, 300, 6)
    lens = np.array([len(m) for m in msgs], np.uint32)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    whole = np.concatenate(msgs)
    if alg == ALG_HIGHWAY:
        for width in (64, 128, 256):
            sb = engine.StreamBatch(alg, synth.key256(), n, width=256)
            for buf, o, L in appends:
                sb.append(buf, o, L)
            got = to_u64(sb.finish(width))
            want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), whole, off, None,
                                       width, 4)
            assert np.array_equal(got, want), width
    else:
        oalg = oracle.ALG_SIPHASH if alg == ALG_SIPHASH else oracle.ALG_SIPTREE
        for c, d in ((2, 4), (1, 3), (3, 5)):
            sb = engine.StreamBatch(alg, synth.key128(), n, c=c, d=d)
            for buf, o, L in appends:
                sb.append(buf, o, L)
            got = to_u64(sb.finish())
            want = oracle.batch_ragged(oalg, synth.key128(), whole, off, None, c, d)
            assert np.array_equal(got, want), (c, d)


@pytest.mark.parametrize("chunk", [0, 1, 7, 31, 32, 33, 100, 4096])
def test_fixed_layout_appends(oracle, chunk):
    n, reps = 300, 3
    data = synth.counter_bytes(77 + chunk, n * chunk * reps).reshape(reps, n, chunk)
    whole = np.concatenate([data[r] for r in range(reps)], axis=1)
    sb = engine.StreamBatch(ALG_HIGHWAY, synth.key256(), n, width=256)
    for r in range(reps):
        sb.append(data[r])
    got = to_u64(sb.finish())
    assert np.array_equal(got, oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(),
                                                  whole, 256, 4))


def test_streaming_hasher_matches_one_shot(oracle, ramp_key):
    """T/test_highway.py:156-172."""
    msg = ramp(200)
    expected = oracle.highway(ramp_key.lanes, msg)[0]
    rng = np.random.default_rng(0xC0FFEE)
    for _ in range(30):
        cuts = sorted(rng.integers(0, len(msg) + 1, size=4).tolist())
        h = lh.StreamingHasher(ramp_key)
        prev = 0
        for cut in cuts + [len(msg)]:
            h.append(msg[prev:cut])
            prev = cut
        assert h.finish() == expected


def test_streaming_hasher_contract(oracle, ramp_key):
    """T/test_highway.py:175-193."""
    h = lh.StreamingHasher(ramp_key)
    h.append(b"").append(b"").append(ramp(5)).append(b"")
    assert h.finish() == oracle.highway(ramp_key.lanes, ramp(5))[0]
    h = lh.StreamingHasher(ramp_key)
    h.append(b"abc")
    h.finish()
    with pytest.raises(RuntimeError):
        h.finish()
    h = lh.StreamingHasher(ramp_key)
    h.finish()
    with pytest.raises(RuntimeError):
        h.append(b"x")
    h = lh.StreamingHasher(ramp_key)
    h.append(ramp(33))
    assert h.finish(256) == tuple(oracle.highway(ramp_key.lanes, ramp(33)))


def test_sip_streaming(oracle):
    """T/test_sip.py:155-176 and T/test_tree.py:70-91."""
    key = Key128.from_bytes(bytes(range(16)))
    msg = bytes(range(64)) * 2
    rng = np.random.default_rng(5)
    for params in (SIPHASH_24, SIPHASH_13):
        want = oracle.siphash(key.lanes, msg, params.c, params.d)
        want_t = oracle.siptree(key.lanes, msg, params.c, params.d)
        for _ in range(10):
            cuts = sorted(rng.integers(0, len(msg) + 1, size=3).tolist())
            h, t = lh.SipHasher(key, params), lh.SipTreeHasher(key, params)
            prev = 0
            for cut in cuts + [len(msg)]:
                h.append(msg[prev:cut])
                t.append(msg[prev:cut])
                prev = cut
            assert h.finish() == want
            assert t.finish() == want_t
    h = lh.SipHasher(key)
    h.append(b"abc")
    h.finish()
    with pytest.raises(RuntimeError):
        h.finish()
    with pytest.raises(RuntimeError):
        h.append(b"x")


def test_acceptance_chunk_split_1000(oracle):
    """T/test_acceptance.py:101-116, as one batch of 1000 messages."""
    rng = np.random.default_rng(3)
    msgs, appends = _random_chunked_batch(rng, 1000, 300, 6)
    key = synth.key256()
    sb = engine.StreamBatch(ALG_HIGHWAY, key, 1000)
    for buf, o, L in appends:
        sb.append(buf, o, L)
    got = to_u64(sb.finish())
    want = np.array([oracle.highway(key, m.tobytes())[0] for m in msgs], np.uint64)
    assert np.array_equal(got, want)


def test_stream_batch_misuse():
    sb = engine.StreamBatch(ALG_HIGHWAY, synth.key256(), 4)
    with pytest.raises(ValueError):
        sb.append(np.zeros((3, 8), np.uint8))
    with pytest.raises(ValueError):
        engine.StreamBatch(ALG_SIPHASH, synth.key128(), 4).finish(width=128)
    sb.finish()
    with pytest.raises(RuntimeError):
        sb.append(np.zeros((4, 8), np.uint8))


@pytest.mark.parametrize("rounds", [0, 1, 2, 3, 5])
def test_stream_finalization_rounds(oracle, rounds):
    """Every kernel is checked at several round counts (a ptxas miscompile
    once showed only for rounds >= 1)."""
    n, L = 257, 100
    data = synth.counter_bytes(500 + rounds, n * L).reshape(n, L)
    sb = engine.StreamBatch(ALG_HIGHWAY, synth.key256(), n, width=256, rounds=rounds)
    sb.append(data[:, :37])
    sb.append(data[:, 37:])
    got = to_u64(sb.finish())
    assert np.array_equal(got, oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(), data,
                                                  256, rounds))


@pytest.mark.parametrize("alg", [ALG_HIGHWAY, ALG_SIPHASH, ALG_SIPTREE])
def test_tma_block_appends_with_and_without_pending_tails(oracle, alg):
    """Fixed-layout whole-block chunks on >= 1,024 messages take the
    TMA-staged append; rows left with a pending tail by an earlier ragged
    append take the generic path inside it.  Digests equal the one-shot."""
    rng = np.random.default_rng(alg + 40)
    n = 3000
    chunks = [128, 96, 1024, 32]
    key = synth.key256() if alg == ALG_HIGHWAY else synth.key128()
    # Rows 0..n/2 get a ragged head of 0..40 bytes first (pending tails).
    head = rng.integers(0, 41, n).astype(np.uint32)
    head[n // 2:] = 0
    total = head.astype(np.int64) + sum(chunks)
    msgs = [synth.counter_bytes(500 + i, int(t)) for i, t in enumerate(total)]
    sb = engine.StreamBatch(alg, key, n)
    off = np.zeros(n, np.uint64)
    off[1:] = np.cumsum(head[:-1])
    hb = np.concatenate([m[:h] for m, h in zip(msgs, head)]) if head.sum() else np.zeros(1, np.uint8)
    sb.append(hb, off, head)
    pos = head.astype(np.int64).copy()
    for c in chunks:
        block = np.stack([m[p:p + c] for m, p in zip(msgs, pos)])
        sb.append(torch.from_numpy(block).cuda())
        pos += c
    got = to_u64(sb.finish())
    buf = np.concatenate(msgs)
    moff = np.zeros(n + 1, np.uint64)
    moff[1:] = np.cumsum(total)
    oalg = {ALG_HIGHWAY: oracle.ALG_HIGHWAY, ALG_SIPHASH: oracle.ALG_SIPHASH,
            ALG_SIPTREE: oracle.ALG_SIPTREE}[alg]
    p1, p2 = (64, 4) if alg == ALG_HIGHWAY else (2, 4)
    want = oracle.batch_ragged(oalg, key, buf, moff, None, p1, p2)
    assert np.array_equal(got, want)
