"""Length-class schedule of ragged batches (lh_ragged_plan_stats,
lh_ragged_order, lh_*_ragged_ordered): the order is a permutation grouped by
class, the statistic matches a numpy restatement, and ordered launches give
the oracle's digests in message order."""
import numpy as np
import pytest
import torch

from oracle import oracle
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import KERNEL_RING

pytestmark = pytest.mark.gpu


def _layout(n, lo, hi, seed=3, with_len=True):
    lens = synth.lengths(seed, n, lo, hi)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(lens, dtype=np.uint64)
    buf = synth.counter_bytes(seed + 1, int(off[-1]) + 1)
    return buf, (off[:-1] if with_len else off), (lens if with_len else None), lens


def _class(units):
    u = np.minimum(units.astype(np.int64), 0x7FFFFFFF)
    e = np.floor(np.log2(np.maximum(u, 1))).astype(np.int64)
    big = 128 + (e - 7) * 8 + ((u >> np.maximum(e - 3, 0)) & 7)
    return np.where(u < 128, u, big)


@pytest.mark.parametrize("kind,shift", [("hh", 5), ("sip", 3)])
def test_order_is_a_permutation_grouped_by_class(kind, shift):
    buf, off, lens, L = _layout(50_001, 0, 9000)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_len = torch.from_numpy(lens.view(np.int32)).cuda()
    sched = engine.ragged_order(d_off, d_len, len(L), kind).cpu().numpy().view(np.uint32)
    order = sched[:, 3]
    assert np.array_equal(np.sort(order), np.arange(len(L), dtype=np.uint32))
    # each record carries its message's offset and length
    assert np.array_equal(sched[:, 0].astype(np.uint64) | (sched[:, 1].astype(np.uint64) << 32),
                          off[order])
    assert np.array_equal(sched[:, 2], L[order])
    cls = _class(L[order] >> shift)
    assert np.all(np.diff(cls) <= 0)  # longest class first, classes contiguous
    # offsets[n+1] form gives the same grouping
    off2 = np.zeros(len(L) + 1, np.uint64)
    off2[1:] = np.cumsum(L, dtype=np.uint64)
    order2 = engine.ragged_order(torch.from_numpy(off2.view(np.int64)).cuda(), None, len(L), kind)
    assert np.array_equal(_class(L[order2.cpu().numpy().view(np.uint32)[:, 3]] >> shift), cls)


def test_plan_stats_match_numpy():
    buf, off, lens, L = _layout(40_000, 0, 3000)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_len = torch.from_numpy(lens.view(np.int32)).cuda()
    for kind, (shift, fixed) in engine._WORK_UNITS.items():
        _, _, (wsum, wmax32) = engine._plan(d_off, d_len, len(L), len(L), len(buf), d_off.device,
                                            kind)
        w = (L.astype(np.int64) >> shift) + fixed
        pad = (-len(w)) % 32
        groups = np.concatenate([w, np.zeros(pad, np.int64)]).reshape(-1, 32)
        assert wsum == w.sum() and wmax32 == 32 * groups.max(axis=1).sum()
    # sorted lengths: efficient, so the automatic schedule keeps the natural order
    Ls = np.sort(L)
    offs = np.zeros(len(Ls), np.uint64)
    offs[1:] = np.cumsum(Ls[:-1], dtype=np.uint64)
    _, _, (wsum, wmax32) = engine._plan(torch.from_numpy(offs.view(np.int64)).cuda(),
                                        torch.from_numpy(Ls.view(np.int32)).cuda(), len(Ls),
                                        len(Ls), len(buf), d_off.device, "hh")
    assert wsum / wmax32 > 0.95
    saved, cost = engine.balance_gain("hh", 4, len(Ls), wsum, wmax32)
    assert saved < cost


@pytest.mark.parametrize("with_len", [True, False])
@pytest.mark.parametrize("width", [64, 256])
def test_ordered_highway_matches_oracle(with_len, width):
    key = synth.key256()
    buf, off, lens, L = _layout(20_011, 0, 2048, seed=9, with_len=with_len)
    want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, lens, width, 4)
    for balance in (True, None, False):
        got = engine.highway_ragged(key, buf, off, lens, width, kernel=KERNEL_RING,
                                    balance=balance)
        assert np.array_equal(np.asarray(got).reshape(want.shape), want), balance


@pytest.mark.parametrize("c,d,tree", [(2, 4, False), (1, 3, False), (2, 4, True), (3, 5, False)])
def test_ordered_sip_matches_oracle(c, d, tree):
    key = synth.key128()
    buf, off, lens, L = _layout(12_345, 0, 700, seed=11)
    alg = oracle.ALG_SIPTREE if tree else oracle.ALG_SIPHASH
    want = oracle.batch_ragged(alg, key, buf, off, lens, c, d)
    d_b = torch.from_numpy(buf).cuda()
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_len = torch.from_numpy(lens.view(np.int32)).cuda()
    for balance in (True, None):
        got = engine.sip_ragged(key, d_b, d_off, d_len, c, d, tree, kernel=KERNEL_RING,
                                balance=balance)
        assert np.array_equal(engine.to_u64(got), want), balance


def test_auto_schedule_orders_only_unbalanced_batches(monkeypatch):
    calls = []
    real = engine.ragged_order
    monkeypatch.setattr(engine, "ragged_order", lambda *a, **k: calls.append(1) or real(*a, **k))
    key = synth.key256()
    buf, off, lens, L = _layout(200_000, 0, 4096, seed=5)
    d = [torch.from_numpy(buf).cuda(), torch.from_numpy(off.view(np.int64)).cuda(),
         torch.from_numpy(lens.view(np.int32)).cuda()]
    engine.highway_ragged(key, *d, 64)                  # random lengths: ordered
    assert len(calls) == 1
    engine.highway_ragged(key, *d, 64, check=False)     # nothing measured: natural order
    engine.highway_ragged(key, *d, 64, balance=False)
    assert len(calls) == 1
    # equal lengths: efficient as is
    lens2 = np.full(200_000, 512, np.uint32)
    off2 = (np.arange(200_000, dtype=np.uint64) * 512)
    buf2 = synth.counter_bytes(6, 200_000 * 512)
    engine.highway_ragged(key, torch.from_numpy(buf2).cuda(),
                          torch.from_numpy(off2.view(np.int64)).cuda(),
                          torch.from_numpy(lens2.view(np.int32)).cuda(), 64)
    assert len(calls) == 1
    # a small batch: ordering would cost more than it saves
    engine.highway_ragged(key, d[0], d[1][:1000], d[2][:1000], 64)
    assert len(calls) == 1


def test_reused_schedule():
    """A schedule built once serves every batch of the same layout."""
    key = synth.key256()
    buf, off, lens, L = _layout(10_000, 0, 1500, seed=13)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_len = torch.from_numpy(lens.view(np.int32)).cuda()
    sched = engine.ragged_order(d_off, d_len, len(L), "hh")
    for seed in (21, 22):
        b = synth.counter_bytes(seed, len(buf))
        want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, b, off, lens, 64, 4)
        got = engine.highway_ragged(key, torch.from_numpy(b).cuda(), d_off, d_len, 64,
                                    kernel=KERNEL_RING, schedule=sched)
        assert np.array_equal(engine.to_u64(got), want)
    with pytest.raises(ValueError):
        engine.highway_ragged(key, torch.from_numpy(buf).cuda(), d_off, d_len, 64,
                              kernel=KERNEL_RING, schedule=sched[:-1])
    with pytest.raises(ValueError):
        engine.highway_ragged(key, torch.from_numpy(buf).cuda(), d_off, d_len, 64,
                              kernel=engine.KERNEL_STAGED, schedule=sched)
