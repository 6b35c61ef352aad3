"""Parity of an A/B library build's short-key kernel against the oracle on
cfg3-shaped and awkward layouts (run with LH_LIBRARY=ab/lib_x.so)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import KERNEL_STAGED

key = synth.key256()
rng = np.random.default_rng(7)
bad = 0
for trial, (n, lo, hi, mode) in enumerate([(200001, 8, 64, "packed"), (70000, 0, 64, "packed"), (50000, 0, 80, "packed"),
                                          (40000, 8, 64, "gaps"), (30000, 8, 64, "shuffled"), (20000, 1, 64, "overlap"),
                                          (129, 8, 64, "packed"), (127, 8, 64, "packed"), (5, 64, 64, "packed")]):
    lens = rng.integers(lo, hi + 1, n).astype(np.uint32)
    if mode == "packed":
        off = np.zeros(n, np.uint64); off[1:] = np.cumsum(lens[:-1])
    elif mode == "gaps":
        off = np.cumsum(lens.astype(np.uint64) + rng.integers(0, 40, n).astype(np.uint64)) - lens
    elif mode == "shuffled":
        off = np.zeros(n, np.uint64); off[1:] = np.cumsum(lens[:-1]); p = rng.permutation(n); off, lens = off[p], lens[p]
    else:
        off = rng.integers(0, 5000, n).astype(np.uint64)
    total = int((off + lens).max()) + 3
    buf = synth.counter_bytes(11 + trial, total)
    for use_len in (True, False):
        if not use_len and mode != "packed":
            continue
        if use_len:
            o, l = off, lens
        else:
            o = np.zeros(n + 1, np.uint64); o[1:] = np.cumsum(lens); l = None
        for w in (64, 256):
            want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, o, l, w, 4)
            got = engine.highway_ragged(key, buf, o, l, w, kernel=KERNEL_STAGED)
            ok = np.array_equal(np.asarray(got).reshape(want.shape), want)
            bad += not ok
            print(trial, n, mode, "len" if use_len else "off", w, "ok" if ok else "MISMATCH", flush=True)
# fixed rows <= 64 B
for L in (8, 12, 33, 64):
    m = synth.counter_bytes(5, 3000 * L).reshape(3000, L)
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, m, 64, 4)
    got = engine.to_u64(engine.highway_batch(key, torch.from_numpy(m).cuda(), 64, 4, kernel=KERNEL_STAGED))
    ok = np.array_equal(got, want); bad += not ok
    print("fixed", L, "ok" if ok else "MISMATCH")
print("BAD", bad)
sys.exit(1 if bad else 0)
