"""Host-side logic that runs without a GPU: the C-ABI library loads and exports
every symbol include/lanehash_b200.h declares, argument validation and
error mapping mirror the reference (ValueError), the reference-shaped types,
and the synthetic-input generator's numpy twin."""
import ctypes
import struct

import numpy as np
import pytest

import paper_1612_06257_b200 as lh
from paper_1612_06257_b200 import _lib, engine, synth
from paper_1612_06257_b200.highway import Key256
from paper_1612_06257_b200.sip import Key128, SipParams


def test_library_exports_every_declared_symbol():
    l = _lib.lib()
    declared = _lib.declared_symbols()
    assert len(declared) >= 11
    for name in declared:
        assert hasattr(l, name), name


def test_version_and_strerror():
    assert "sm_100a" in _lib.version()
    l = _lib.lib()
    for code in (0, -1, -2, -3, -4, -5, -99):
        assert l.lh_strerror(code)


def test_abi_rejects_bad_arguments_before_touching_the_device():
    l = _lib.lib()
    key4 = (ctypes.c_uint64 * 4)(1, 2, 3, 4)
    key2 = (ctypes.c_uint64 * 2)(1, 2)
    buf = ctypes.create_string_buffer(64)
    out = (ctypes.c_uint64 * 8)()
    addr = ctypes.addressof
    # width not in {64,128,256}
    assert l.lh_highway_fixed(addr(buf), 1, 32, key4, 96, 4, addr(out), None) == _lib.LH_EINVAL
    # negative rounds
    assert l.lh_highway_fixed(addr(buf), 1, 32, key4, 64, -1, addr(out), None) == _lib.LH_EINVAL
    # NULL key / NULL out
    assert l.lh_highway_fixed(addr(buf), 1, 32, None, 64, 4, addr(out), None) == _lib.LH_EINVAL
    assert l.lh_highway_fixed(addr(buf), 1, 32, key4, 64, 4, None, None) == _lib.LH_EINVAL
    # misaligned digest pointer
    assert l.lh_highway_fixed(addr(buf), 1, 32, key4, 64, 4, addr(out) + 1, None) == _lib.LH_EALIGN
    # SipParams must be positive (S/sip.py:60-62)
    assert l.lh_siphash_fixed(addr(buf), 1, 8, key2, 0, 4, 0, addr(out), None) == _lib.LH_EINVAL
    assert l.lh_siphash_fixed(addr(buf), 1, 8, key2, 2, 0, 0, addr(out), None) == _lib.LH_EINVAL
    # ragged: misaligned offsets
    assert l.lh_highway_ragged(addr(buf), addr(buf) + 4, None, 1, key4, 64, 4, addr(out),
                               None) == _lib.LH_EALIGN
    # unknown kernel id
    assert l.lh_highway_fixed_kernel(addr(buf), 1, 32, key4, 64, 4, addr(out), None, 7) == \
        _lib.LH_EINVAL
    # overflow of n * len
    assert l.lh_highway_fixed(addr(buf), 1 << 40, 1 << 40, key4, 64, 4, addr(out), None) == \
        _lib.LH_ETOOBIG
    assert l.lh_synth_fill(addr(buf) + 1, 8, 0, 0, 0, None) == _lib.LH_EALIGN
    # raw Update: inverse flag must be 0/1, states 8-byte aligned
    assert l.lh_highway_update_states(addr(out), addr(out), 1, 2, None) == _lib.LH_EINVAL
    assert l.lh_highway_update_states(None, addr(out), 1, 0, None) == _lib.LH_EINVAL
    assert l.lh_highway_update_states(addr(out) + 4, addr(out), 1, 0, None) == _lib.LH_EALIGN
    assert l.lh_highway_bijectivity(0, 1, None, None) == _lib.LH_EINVAL


def test_check_maps_errors_like_the_reference():
    with pytest.raises(ValueError):
        _lib.check(_lib.LH_EINVAL)
    with pytest.raises(ValueError):
        _lib.check(_lib.LH_EALIGN)
    with pytest.raises(_lib.EngineError):
        _lib.check(_lib.LH_ECUDA)
    _lib.check(_lib.LH_OK)


def test_python_api_validates_before_device():
    with pytest.raises(ValueError):
        engine.highway_batch(Key256((1, 2, 3, 4)), np.zeros((2, 32), np.uint8), width=96)
    with pytest.raises(ValueError):
        engine.sip_batch(Key128(1, 2), np.zeros((2, 32), np.uint8), c=0)
    with pytest.raises(ValueError):
        lh.select_backend("simd512")


def test_constants_match_reference(golden):
    assert [f"{x:016x}" for x in lh.INIT0] == golden["init0"]
    assert [f"{x:016x}" for x in lh.INIT1] == golden["init1"]
    assert list(lh.ZIPPER_OFFSETS) == golden["zipper_offsets"]
    assert sorted(lh.ZIPPER_OFFSETS) == list(range(16))
    assert bytes(lh.ZIPPER_OFFSETS).hex() == "030c02050e010f000b040a0d09060807"


def test_initialize_matches_reference_layout(golden):
    """S/highway.py:122-127 (host key expansion) against the golden init lanes."""
    from paper_1612_06257_b200 import highway

    key = bytes(range(32))
    v0, v1, m0, m1 = highway.initialize(key)
    lanes = struct.unpack("<4Q", key)
    rot = lambda x: ((x >> 32) | (x << 32)) & ((1 << 64) - 1)
    init0 = [int(x, 16) for x in golden["init0"]]
    init1 = [int(x, 16) for x in golden["init1"]]
    assert list(v0) == [k ^ c for k, c in zip(lanes, init0)]
    assert list(v1) == [rot(k) ^ c for k, c in zip(lanes, init1)]
    assert list(m0) == init0 and list(m1) == init1
    with pytest.raises(ValueError):
        highway.update(((0,) * 4,) * 3, (0,) * 4)


def test_zipper_prmt_selectors_match_byte_table():
    """The GPU zipper (csrc/lh_device.cuh) is 5 PRMT per lane pair; replay the
    same selectors with a Python byte_perm and compare to the byte table."""

    def byte_perm(x, y, s):
        src = struct.pack("<II", x, y)
        return int.from_bytes(bytes(src[(s >> (4 * i)) & 7] for i in range(4)), "little")

    rng = np.random.default_rng(7)
    for _ in range(200):
        data = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        w0, w1, w2, w3 = struct.unpack("<4I", data)
        u = byte_perm(w1, w3, 0x5041)
        r0 = byte_perm(w0, u, 0x4253)
        r1 = byte_perm(w3, w0, 0x4352)
        r2 = byte_perm(w2, u, 0x7263)
        r3 = byte_perm(w2, w1, 0x7061)
        assert struct.pack("<4I", r0, r1, r2, r3) == bytes(data[o] for o in lh.ZIPPER_OFFSETS)


def test_key_types_mirror_reference():
    raw = bytes(range(32))
    assert Key256.from_bytes(raw).to_bytes() == raw
    assert Key256.from_hex(raw.hex()) == Key256.from_bytes(raw)
    with pytest.raises(ValueError):
        Key256.from_bytes(bytes(31))
    with pytest.raises(ValueError):
        Key256((1, 2, 3))
    raw16 = bytes(range(16))
    assert Key128.from_bytes(raw16).to_bytes() == raw16
    with pytest.raises(ValueError):
        Key128.from_bytes(bytes(8))
    with pytest.raises(ValueError):
        SipParams(0, 4)
    with pytest.raises(ValueError):
        SipParams(2, 0)


def test_digest_byte_images():
    assert lh.digest64_to_bytes(0x0102030405060708) == bytes((8, 7, 6, 5, 4, 3, 2, 1))
    assert struct.unpack("<4Q", lh.digest256_to_bytes((1, 2, 3, 4))) == (1, 2, 3, 4)
    assert struct.unpack("<2Q", lh.digest128_to_bytes((5, 6))) == (5, 6)


def test_synth_numpy_twin_properties():
    w = synth.words(1, 0, 1000)
    assert len(np.unique(w)) == 1000
    # word_offset windows agree
    assert np.array_equal(synth.words(1, 500, 100), w[500:600])
    b = synth.counter_bytes(1, 8 * 1000)
    assert np.array_equal(b.view(np.uint64), w)
    assert np.array_equal(synth.counter_bytes(1, 13), b[:13])
    lens = synth.lengths(3, 100000, 8, 64)
    assert lens.min() == 8 and lens.max() == 64
    assert abs(lens.mean() - 36) < 0.2
    k = synth.key256()
    assert [f"{int(x):016x}" for x in k] == ["a30febcfd9c2825f", "4510bdf882d9d721",
                                            "0a7d3da94ecde8b8", "043b27b61342f01d"]


def test_remainder_sweep_layout():
    lens, off, kind = synth.remainder_sweep_layout(1024, 64)
    assert len(lens) == 65536 and int(off[-1]) == 33521664
    assert (kind == 0).sum() == 32768 and (kind == 1).sum() == 16384


def test_stream_abi_validation_without_device():
    l = _lib.lib()
    assert [l.lh_stream_state_bytes(a) > 0 for a in range(3)] == [True] * 3
    assert l.lh_stream_state_bytes(7) == 0
    key4 = (ctypes.c_uint64 * 4)(1, 2, 3, 4)
    buf = ctypes.create_string_buffer(512)
    base = (ctypes.addressof(buf) + 15) & ~15
    assert l.lh_stream_init(0, base, 1, key4, 96, 4, None) == _lib.LH_EINVAL
    assert l.lh_stream_init(1, base, 1, key4, 0, 4, None) == _lib.LH_EINVAL
    assert l.lh_stream_init(0, base + 8, 1, key4, 64, 4, None) == _lib.LH_EALIGN
    assert l.lh_stream_init(9, base, 1, key4, 64, 4, None) == _lib.LH_EINVAL
    assert l.lh_stream_finish(1, base, 1, base, 2, None) == _lib.LH_EINVAL


def test_cli_rejects_bad_arguments_before_hashing():
    from paper_1612_06257_b200 import cli, vectors

    for argv in (["hash", "--algo", "md5"], ["hash", "--key", "zz"],
                 ["hash", "--key", "00"], ["avalanche", "--sizes", "2"],
                 ["avalanche", "--samples", "4"], ["bench", "--preset", "nope"],
                 ["bench", "--sizes", "x"]):
        with pytest.raises(SystemExit) as e:
            cli.main(argv)
        assert e.value.code == 2, argv
    with pytest.raises(ValueError):
        vectors.VectorRecord.from_line("a,b,c")
    assert vectors.ramp(3) == b"\x00\x01\x02"
    for argv in (["avalanche", "--sizes", "40", "--iters", "10"],
                 ["avalanche", "--sizes", "abc"], ["bench", "--reps", "0", "--sizes", "8"],
                 ["bench", "--runs", "0", "--sizes", "8"]):
        with pytest.raises(SystemExit):
            cli.main(argv)


def test_cli_size_range_parsing():
    """T/test_vectors_cli.py:199-202."""
    from paper_1612_06257_b200 import cli

    parser = cli.build_parser()
    assert cli._parse_sizes(parser, "4..6") == [4, 5, 6]
    assert cli._parse_sizes(parser, "1,8..10,32") == [1, 8, 9, 10, 32]


def test_balance_cost_model():
    """engine.balance_gain: nothing to gain from a balanced batch, more from
    an unbalanced one, and a small batch never pays for its ordering."""
    from paper_1612_06257_b200 import engine

    n = 1 << 20
    saved, cost = engine.balance_gain("hh", 4, n, wsum=37 * n, wmax32=37 * n)
    assert saved == 0.0 and cost > 0
    # U[0, 2048]-like: efficiency 0.55
    s1, c1 = engine.balance_gain("hh", 4, n, wsum=37 * n, wmax32=int(37 * n / 0.55))
    assert s1 > engine.BALANCE_MARGIN * c1
    s2, _ = engine.balance_gain("sip", 2, n, wsum=131 * n, wmax32=int(131 * n / 0.55))
    assert s2 > s1  # SipHash-2-4 spends more per byte
    # 1,000 messages: the fixed cost dominates
    s3, c3 = engine.balance_gain("hh", 4, 1000, wsum=37 * 1000, wmax32=int(37 * 1000 / 0.5))
    assert s3 < c3
    assert engine.balance_gain("hh", 4, 0, 0, 0) == (0.0, engine.BALANCE_COST_S[0])
