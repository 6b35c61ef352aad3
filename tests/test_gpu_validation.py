"""Argument validation at the Python boundary (GPU): caller-supplied ``out=``
tensors and ragged layouts are checked before any kernel writes or reads
(a bad one would be an out-of-bounds device access), and the metadata pass
lh_ragged_plan gives the spans numpy gives."""
import numpy as np
import pytest
import torch

from paper_1612_06257_b200 import _lib, engine, synth
from paper_1612_06257_b200.engine import KERNEL_RING, KERNEL_STAGED, to_u64

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _msgs(n=64, L=40):
    return torch.from_numpy(synth.numpy_bytes(1, (n, L))).to(DEV)


@pytest.mark.parametrize("bad", [
    lambda n: torch.empty(n, dtype=torch.int32, device=DEV),          # dtype
    lambda n: torch.empty(n - 1, dtype=torch.int64, device=DEV),      # too short
    lambda n: torch.empty((n, 2), dtype=torch.int64, device=DEV),     # width mismatch
    lambda n: torch.empty(2 * n, dtype=torch.int64, device=DEV)[::2],  # non-contiguous
    lambda n: torch.empty(n, dtype=torch.int64),                      # host tensor
])
def test_fixed_out_rejected(bad):
    m = _msgs()
    with pytest.raises(ValueError):
        engine.highway_batch(synth.key256(), m, 64, out=bad(len(m)))
    with pytest.raises(ValueError):
        engine.sip_batch(synth.key128(), m, 2, 4, out=bad(len(m)))


def test_fixed_out_accepted_and_written(oracle):
    m = _msgs()
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, synth.key256(), m.cpu().numpy(), 256, 4)
    out = torch.zeros((len(m), 4), dtype=torch.int64, device=DEV)
    r = engine.highway_batch(synth.key256(), m, 256, out=out)
    assert r is out and np.array_equal(to_u64(out), want)
    out_u = torch.zeros((len(m), 4), dtype=torch.uint64, device=DEV)
    engine.highway_batch(synth.key256(), m, 256, out=out_u)
    assert np.array_equal(out_u.view(torch.int64).cpu().numpy().view(np.uint64), want)


def test_prf_and_ragged_out_rejected():
    with pytest.raises(ValueError):
        engine.prf64(synth.key256(), 0, 100, out=torch.empty(99, dtype=torch.int64, device=DEV))
    buf = torch.zeros(100, dtype=torch.uint8, device=DEV)
    off = torch.tensor([0, 10, 20], dtype=torch.int64, device=DEV)
    with pytest.raises(ValueError):
        engine.highway_ragged(synth.key256(), buf, off, None, 128,
                              out=torch.empty(2, dtype=torch.int64, device=DEV))


@pytest.mark.parametrize("host", [False, True])
def test_ragged_layout_rejected(host):
    buf = np.zeros(1000, np.uint8)
    cases = [
        (np.array([0, 10, 5, 20], np.uint64), None),                                 # decreasing
        (np.array([0, 10, 20, 1001], np.uint64), None),                              # past end
        (np.array([0, 990], np.uint64), np.array([5, 11], np.uint32)),               # past end
        (np.array([0, 2 ** 64 - 8], np.uint64), np.array([5, 100], np.uint32)),      # wraps
    ]
    for off, lens in cases:
        args = (buf, off, lens) if host else (
            torch.from_numpy(buf).to(DEV), torch.from_numpy(off.view(np.int64)).to(DEV),
            None if lens is None else torch.from_numpy(lens.view(np.int32)).to(DEV))
        for fn, key in ((engine.highway_ragged, synth.key256()), (engine.sip_ragged, synth.key128())):
            with pytest.raises(ValueError, match="invalid ragged layout"):
                fn(key, *args)


def test_ragged_check_false_skips_plan(oracle):
    """check=False (caller-validated CUDA inputs) hashes the same digests."""
    lens = synth.lengths(7, 5000, 0, 300)
    off = np.zeros(5001, np.uint64)
    off[1:] = np.cumsum(lens)
    buf = synth.counter_bytes(8, int(off[-1]))
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, synth.key256(), buf, off, None, 64, 4)
    d = (torch.from_numpy(buf).to(DEV), torch.from_numpy(off.view(np.int64)).to(DEV))
    for check in (True, False):
        got = engine.highway_ragged(synth.key256(), *d, None, 64, check=check)
        assert np.array_equal(to_u64(got), want)


def test_plan_spans_match_numpy():
    rng = np.random.default_rng(5)
    n = 100_003
    starts = rng.integers(0, 1 << 40, n).astype(np.uint64)
    lens = rng.integers(0, 1 << 20, n).astype(np.uint32)
    d_off = torch.from_numpy(starts.view(np.int64)).to(DEV)
    d_len = torch.from_numpy(lens.view(np.int32)).to(DEV)
    for chunk in (n, 7919, 40000):
        lo, hi = engine._plan(d_off, d_len, n, chunk, 2 ** 64 - 1, torch.device(DEV))
        ends = starts + lens.astype(np.uint64)
        for k in range(len(lo)):
            a, b = k * chunk, min(n, (k + 1) * chunk)
            assert lo[k] == starts[a:b].min() and hi[k] == ends[a:b].max()


def test_lengths_past_2gib_are_unsigned(oracle):
    """A u32 length >= 2^31 (it was sign-extended on the host
    path's span computation) hashes the whole message."""
    L = (1 << 31) + 37
    buf = torch.empty(L + 64, dtype=torch.uint8, device=DEV)
    synth.fill_device(buf, 12)
    off = torch.tensor([16, 3], dtype=torch.int64, device=DEV)
    lens = torch.tensor([np.int32(np.uint32(L).view(np.int32)), 40], dtype=torch.int32,
                        device=DEV)
    host = buf.cpu().numpy()
    want = [oracle.highway(synth.key256(), host[16:16 + L].tobytes())[0],
            oracle.highway(synth.key256(), host[3:43].tobytes())[0]]
    for kernel in (KERNEL_RING, KERNEL_STAGED):
        got = to_u64(engine.highway_ragged(synth.key256(), buf, off, lens, 64, kernel=kernel))
        assert [int(x) for x in got] == want
    del buf
    torch.cuda.empty_cache()


def test_plan_rejects_bad_arguments():
    l = _lib.lib()
    res = torch.zeros(3, dtype=torch.int64, device=DEV)
    off = torch.zeros(4, dtype=torch.int64, device=DEV)
    assert l.lh_ragged_plan(off.data_ptr(), None, 3, 0, 100, res.data_ptr(), res.data_ptr(),
                            res.data_ptr(), None) == _lib.LH_EINVAL
    assert l.lh_ragged_plan(off.data_ptr() + 4, None, 3, 3, 100, res.data_ptr(), res.data_ptr(),
                            res.data_ptr(), None) == _lib.LH_EALIGN


def test_stream_ragged_append_layout_rejected():
    sb = engine.StreamBatch(engine.ALG_HIGHWAY, synth.key256(), 3)
    buf = torch.zeros(100, dtype=torch.uint8, device=DEV)
    bad = torch.tensor([0, 50, 40, 101], dtype=torch.int64, device=DEV)
    with pytest.raises(ValueError, match="invalid ragged layout"):
        sb.append(buf, bad)
    ok = torch.tensor([0, 50, 60, 100], dtype=torch.int64, device=DEV)
    sb.append(buf, ok)
    assert sb.finish().shape == (3,)
