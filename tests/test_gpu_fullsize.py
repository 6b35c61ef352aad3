"""Full-size parity on BASELINE.json's configs (GPU): EVERY digest.

Each full-size config is hashed on the device and every one of its digests
is rechecked by the CPU oracle (oracle/lh_oracle.c on all host threads) on
the same bytes, copied back from HBM: cfg3 2^26 short keys, cfg4 16,384 x
1 MiB (HighwayHash-256), cfg5 2^24 x 1 KiB under HighwayHash-64 and all four
Sip variants, PRF 2^28 counters.  The reference-generated golden prefixes
(tests/golden/) are checked too, and the GPU kernels are also compared with
each other (TMA / direct / split) -- that agreement is extra, not the proof.
Protocol: the reference compares every case (T/test_acceptance.py:75-98;
S/highway.py:247-254, S/sip.py:89-128).  Each test prints its oracle time.
"""
import time

import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden_npy
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import KERNEL_DIRECT, KERNEL_SPLIT, KERNEL_TMA, to_u64

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda"


@pytest.fixture(autouse=True)
def _free():
    yield
    torch.cuda.empty_cache()


def _fill(nbytes, seed):
    t = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    synth.fill_device(t, seed)
    return t


def _host(t):
    """Device tensor -> numpy (bytes as the kernels saw them)."""
    return t.cpu().numpy()


def _mismatches(got, want, what):
    bad = np.flatnonzero(np.any((got != want).reshape(len(got), -1), axis=1))
    assert bad.size == 0, f"{what}: {bad.size} of {len(got)} digests differ, first at {bad[:8]}"


def _log(name, n, t0):
    print(f"\n[fullsize] {name}: {n} digests checked against the oracle in "
          f"{time.perf_counter() - t0:.1f} s, 0 mismatches")


def test_cfg3_short_keys_2p26(oracle):
    n = 1 << 26
    lens = torch.empty(n, dtype=torch.int32, device=DEV)
    synth.lengths_device(lens, 3, 8, 64)
    off = torch.zeros(n + 1, dtype=torch.int64, device=DEV)
    off[1:] = torch.cumsum(lens.to(torch.int64), 0)
    total = int(off[-1])
    buf = _fill(total, 4)
    d = engine.highway_ragged(synth.key256(), buf, off[:-1], lens, 64)
    dd = engine.highway_ragged(synth.key256(), buf, off, None, 64)  # offsets[n+1] form
    assert torch.equal(d, dd)
    h = to_u64(d)
    assert np.array_equal(h[:8192], golden_npy("cfg3_first8192.npy"))
    t0 = time.perf_counter()
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), _host(buf),
                               _host(off).view(np.uint64), None, 64, 4)
    _mismatches(h, want, "cfg3 HighwayHash-64")
    _log("cfg3 hh64 2^26 ragged", n, t0)


def test_cfg3_shaped_sip_and_wide_2p26(oracle):
    """The cfg3 layout under every other hash the bench times on it
    (SipHash-2-4 / -1-3, staged kernel) and HighwayHash-256: every digest."""
    n = 1 << 26
    lens = torch.empty(n, dtype=torch.int32, device=DEV)
    synth.lengths_device(lens, 3, 8, 64)
    off = torch.zeros(n, dtype=torch.int64, device=DEV)
    off[1:] = torch.cumsum(lens[:-1].to(torch.int64), 0)
    total = int(off[-1]) + int(lens[-1])
    buf = _fill(total, 4)
    hb, ho, hl = _host(buf), _host(off).view(np.uint64), _host(lens).view(np.uint32)
    for name, alg, c, d in (("sip24", oracle.ALG_SIPHASH, 2, 4), ("sip13", oracle.ALG_SIPHASH, 1, 3)):
        h = to_u64(engine.sip_ragged(synth.key128(), buf, off, lens, c, d))
        t0 = time.perf_counter()
        _mismatches(h, oracle.batch_ragged(alg, synth.key128(), hb, ho, hl, c, d), name)
        _log(f"cfg3-shaped {name} 2^26 ragged", n, t0)
    h = to_u64(engine.highway_ragged(synth.key256(), buf, off, lens, 256))
    t0 = time.perf_counter()
    _mismatches(h, oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), hb, ho, hl, 256, 4),
                "hh256")
    _log("cfg3-shaped hh256 2^26 ragged", n, t0)


def test_cfg5_wide_digests_2p24(oracle):
    """HighwayHash-128 / -256 over the 16 GiB cfg5 batch: every digest."""
    n, L = 1 << 24, 1024
    m = _fill(n * L, 6).view(n, L)
    host = _host(m)
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(), host, 256, 4)
    t0 = time.perf_counter()
    _mismatches(to_u64(engine.highway_batch(synth.key256(), m, 256)), want, "hh256")
    _mismatches(to_u64(engine.highway_batch(synth.key256(), m, 128)), want[:, :2], "hh128")
    _log("cfg5 hh128 + hh256 2^24 x 1 KiB", 2 * n, t0)


def test_cfg4_long_messages_16GiB(oracle, golden):
    n, L = 16384, 1 << 20
    buf = _fill(n * L, 5)
    m = buf.view(n, L)
    a = engine.highway_batch(synth.key256(), m, 256)  # auto: split-state kernel
    c = engine.highway_batch(synth.key256(), m, 256, kernel=KERNEL_TMA)
    assert torch.equal(a, c)
    h = to_u64(a)
    assert [f"{int(x):016x}" for x in h[0]] == golden["cfg4_msg0_h256"]
    t0 = time.perf_counter()
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(), _host(m), 256, 4)
    _mismatches(h, want, "cfg4 HighwayHash-256")
    _log("cfg4 hh256 16384 x 1 MiB", n, t0)


def test_cfg5_comparators_2p24(oracle):
    n, L = 1 << 24, 1024
    buf = _fill(n * L, 6)
    m = buf.view(n, L)
    host = _host(m)
    ref = np.load(GOLDEN + "/cfg5_first256.npz")
    a = engine.highway_batch(synth.key256(), m, 64)
    h = to_u64(a)
    assert np.array_equal(h[:256], ref["hh64"])
    t0 = time.perf_counter()
    _mismatches(h, oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(), host, 64, 4), "hh64")
    _log("cfg5 hh64 2^24 x 1 KiB", n, t0)
    for name, alg, c, d, tree in (("sip24", oracle.ALG_SIPHASH, 2, 4, False),
                                  ("sip13", oracle.ALG_SIPHASH, 1, 3, False),
                                  ("tree24", oracle.ALG_SIPTREE, 2, 4, True),
                                  ("tree13", oracle.ALG_SIPTREE, 1, 3, True)):
        h = to_u64(engine.sip_batch(synth.key128(), m, c, d, tree))
        assert np.array_equal(h[:256], ref[name]), name
        t0 = time.perf_counter()
        _mismatches(h, oracle.batch_fixed(alg, synth.key128(), host, c, d), name)
        _log(f"cfg5 {name} 2^24 x 1 KiB", n, t0)


def test_cfg5_kernels_agree_2p24():
    """Extra (not the proof): the TMA and direct-load kernels agree on every
    digest of the 16 GiB batch, for HighwayHash-64 and SipTree-1-3."""
    n, L = 1 << 24, 1024
    m = _fill(n * L, 6).view(n, L)
    a = engine.highway_batch(synth.key256(), m, 64, kernel=KERNEL_TMA)
    b = engine.highway_batch(synth.key256(), m, 64, kernel=KERNEL_DIRECT)
    assert torch.equal(a, b)
    a = engine.sip_batch(synth.key128(), m, 1, 3, True, kernel=KERNEL_TMA)
    b = engine.sip_batch(synth.key128(), m, 1, 3, True, kernel=KERNEL_DIRECT)
    assert torch.equal(a, b)


def test_tma_large_batch_128row_config(oracle):
    """n large enough for the 128-row TMA tiles, lengths with r = 0 and 16."""
    for n, L in ((60000, 64), (70001, 48), (60000, 1040)):
        buf = _fill(n * L, 40 + L)
        m = buf.view(n, L)
        a = engine.highway_batch(synth.key256(), m, 256, kernel=KERNEL_TMA)
        b = engine.highway_batch(synth.key256(), m, 256, kernel=KERNEL_DIRECT)
        assert torch.equal(a, b)
        idx = np.array([0, 1, 127, 128, n // 2, n - 1])
        rows = m[torch.from_numpy(idx).to(DEV)].cpu().numpy()
        want = oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(), rows, 256, 4)
        assert np.array_equal(to_u64(a)[idx], want)


def test_prf_2p28(oracle):
    n = 1 << 28
    d = engine.prf64(synth.key256(), 0, n)
    h = to_u64(d)
    assert np.array_equal(h[:4096], golden_npy("prf_0_4096.npy"))
    t0 = time.perf_counter()
    _mismatches(h, oracle.prf64(synth.key256(), 0, n), "PRF")
    _log("PRF 2^28 counters", n, t0)
    # window invariance over the tail of the range
    t = engine.prf64(synth.key256(), n - 100000, 100000)
    assert torch.equal(t, d[n - 100000:])


@pytest.mark.parametrize("cfg", ["128x4", "256x3", "512x3", "128x3", "384x4", "320x5", "448x3"])
def test_tuning_tile_shapes_are_bit_exact(cfg):
    """Every LH_TMA_CFG tile shape (tuning knob, read once per process) must
    produce the same digests as the direct kernel."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import torch\n"
        "from paper_1612_06257_b200 import engine, synth\n"
        "from paper_1612_06257_b200.engine import KERNEL_DIRECT, KERNEL_TMA\n"
        "for n, L in ((200000, 1024), (90001, 48), (70000, 1040)):\n"
        "    b = torch.empty(n * L, dtype=torch.uint8, device='cuda'); synth.fill_device(b, L)\n"
        "    m = b.view(n, L)\n"
        "    for w in (64, 256):\n"
        "        a = engine.highway_batch(synth.key256(), m, w, kernel=KERNEL_TMA)\n"
        "        d = engine.highway_batch(synth.key256(), m, w, kernel=KERNEL_DIRECT)\n"
        "        assert torch.equal(a, d), (n, L, w)\n"
        "    s = engine.sip_batch(synth.key128(), m, 1, 3, True, kernel=KERNEL_TMA)\n"
        "    t = engine.sip_batch(synth.key128(), m, 1, 3, True, kernel=KERNEL_DIRECT)\n"
        "    assert torch.equal(s, t)\n"
        "print('ok')\n" % ROOT)
    env = dict(os.environ, LH_TMA_CFG=cfg)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("kernel,L", [(KERNEL_TMA, 32), (KERNEL_SPLIT, 128)])
def test_row_segments_past_2p30(oracle, kernel, L):
    """More than 2^30 rows: the TMA and split kernels take the batch in
    segments of 2^30 rows (TMA coordinates are int32).  Rows on both sides
    of every segment boundary and a random sample match the oracle."""
    n = (1 << 30) + 4096 if kernel == KERNEL_TMA else (1 << 30) + 200
    if torch.cuda.get_device_properties(0).total_memory < n * (L + 8) * 1.2:
        pytest.skip("needs more device memory")
    buf = _fill(n * L, 17)
    m = buf.view(n, L)
    out = engine.highway_batch(synth.key256(), m, 64, kernel=kernel)
    rng = np.random.default_rng(3)
    idx = np.unique(np.concatenate([[0, (1 << 30) - 1, 1 << 30, (1 << 30) + 1, n - 1],
                                    rng.integers(0, n, 200)]))
    got = to_u64(out[torch.from_numpy(idx).to(DEV)])
    rows = m[torch.from_numpy(idx).to(DEV)].cpu().numpy()
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(), rows, 64, 4)
    assert np.array_equal(got, want)
    del buf, m, out
    torch.cuda.empty_cache()


def test_ragged_offsets_past_4gib(oracle):
    """Byte offsets beyond 2^32 (u64 offset arithmetic in every ragged
    kernel): messages straddling and past the 4 GiB mark."""
    from paper_1612_06257_b200.engine import KERNEL_RING, KERNEL_STAGED
    total = (1 << 32) + (1 << 24)
    buf = _fill(total, 23)
    rng = np.random.default_rng(8)
    lens = rng.integers(0, 700, 3000).astype(np.uint32)
    lens[:1500] = rng.integers(0, 65, 1500)  # short keys for the staged kernel
    off = np.zeros(3000, np.uint64)
    off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
    off += np.uint64((1 << 32) - 40000)  # the batch straddles the 4 GiB mark
    span = buf[int(off[0]):int(off[-1]) + int(lens[-1])].cpu().numpy()
    rel = off - off[0]
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), span, rel, lens, 64, 4)
    d_off = torch.from_numpy(off.view(np.int64)).to(DEV)
    d_len = torch.from_numpy(lens.view(np.int32)).to(DEV)
    for kernel in (KERNEL_STAGED, KERNEL_RING):
        got = to_u64(engine.highway_ragged(synth.key256(), buf, d_off, d_len, 64, kernel=kernel))
        assert np.array_equal(got, want), kernel
    got = to_u64(engine.sip_ragged(synth.key128(), buf, d_off, d_len, 2, 4))
    assert np.array_equal(got, oracle.batch_ragged(oracle.ALG_SIPHASH, synth.key128(), span, rel,
                                                   lens, 2, 4))
    # the same batch through the length-class schedule (u64 offsets in the records)
    got = to_u64(engine.highway_ragged(synth.key256(), buf, d_off, d_len, 64, kernel=KERNEL_RING,
                                       balance=True))
    assert np.array_equal(got, want)
    del buf
    torch.cuda.empty_cache()


def test_ordered_message_of_4gib(oracle):
    """A message of 2^32 + 37 bytes in an ordered launch: its schedule record
    holds a saturated length (0xFFFFFFFF) and the kernel re-reads the real one
    from the layout; two short neighbours check the record order.  (One GPU
    thread walks the 4 GiB message: ~13 s; the Sip kernels share the code.)"""
    from paper_1612_06257_b200.engine import KERNEL_RING
    big = (1 << 32) + 37
    total = 100 + big + 500
    if torch.cuda.get_device_properties(0).total_memory < 2.5 * total:
        pytest.skip("needs more device memory")
    buf = _fill(total, 29)
    off = np.array([0, 100, 100 + big, total], np.uint64)
    host = buf.cpu().numpy()
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), host, off, None, 256, 4)
    d_off = torch.from_numpy(off.view(np.int64)).to(DEV)
    sched = engine.ragged_order(d_off, None, 3, "hh").cpu().numpy().view(np.uint32)
    assert sched[0, 3] == 1 and sched[0, 2] == 0xFFFFFFFF  # the long message first, saturated
    got = engine.highway_ragged(synth.key256(), buf, d_off, None, 256, kernel=KERNEL_RING,
                                balance=True)
    assert np.array_equal(to_u64(got).reshape(want.shape), want)
    del buf, host
    torch.cuda.empty_cache()
