#!/usr/bin/env python
"""Randomised parity soak: random batches (sizes, length distributions,
layouts, widths, rounds, kernels, schedules) through the engine against the
CPU oracle.  usage: python scripts/fuzz_parity.py [seconds] [seed]
Prints one line per mismatch and a summary; exit status 1 on any mismatch."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from oracle import oracle
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import (KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING, KERNEL_SPLIT,
                                          KERNEL_STAGED, KERNEL_TMA)

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
key, k128 = synth.key256(), synth.key128()
T = len(os.sched_getaffinity(0))
t_end = time.time() + budget
cases = digests = bad = 0
FAULT = os.environ.get("FUZZ_FAULT") == "1"  # self-test: corrupt one digest in ~2% of the cases


def _same(got, want):
    got = got.reshape(want.shape).copy()
    if FAULT and got.size and rng.random() < 0.02:
        got.reshape(-1)[int(rng.integers(0, got.size))] ^= np.uint64(1)
    return np.array_equal(got, want)


def ragged_case():
    global cases, digests, bad
    n = int(rng.choice([1, 31, 33, 127, 129, 1000, 4097, 20000, 70000]))
    dist = rng.choice(["short", "mixed", "medium", "long", "pow2", "zeros"])
    if dist == "short":
        lens = rng.integers(0, 65, n)
    elif dist == "mixed":
        lens = rng.integers(0, 200, n)
    elif dist == "medium":
        lens = rng.integers(0, 1500, n)
    elif dist == "long":
        lens = rng.integers(0, 20000, min(n, 3000)); n = len(lens)
    elif dist == "pow2":
        lens = rng.choice([0, 16, 32, 64, 128, 256, 1024], n)
    else:
        lens = np.where(rng.random(n) < 0.5, 0, rng.integers(0, 100, n))
    lens = lens.astype(np.uint32)
    mode = rng.choice(["packed", "gaps", "shuffled", "overlap"])
    if mode == "packed":
        off = np.zeros(n, np.uint64); off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
    elif mode == "gaps":
        off = (np.cumsum(lens.astype(np.uint64) + rng.integers(0, 50, n).astype(np.uint64)) - lens).astype(np.uint64)
    elif mode == "shuffled":
        off = np.zeros(n, np.uint64); off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
        p = rng.permutation(n); off, lens = off[p], lens[p]
    else:
        off = rng.integers(0, 3000, n).astype(np.uint64)
    base_shift = int(rng.integers(0, 16))  # unaligned buffer base
    total = int((off + lens).max()) + 1
    raw = torch.empty(total + 16, dtype=torch.uint8, device="cuda")
    synth.fill_device(raw[: (total + 16) // 8 * 8], int(rng.integers(1, 1 << 30)))
    buf = raw[base_shift: base_shift + total]
    host = buf.cpu().numpy()
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_len = torch.from_numpy(lens.view(np.int32)).cuda()
    use_off_form = mode == "packed" and rng.random() < 0.4
    if use_off_form:
        o2 = np.zeros(n + 1, np.uint64); o2[1:] = np.cumsum(lens, dtype=np.uint64)
        d_off, d_len, ho, hl = torch.from_numpy(o2.view(np.int64)).cuda(), None, o2, None
    else:
        ho, hl = off, lens
    algo = rng.choice(["hh", "sip", "tree"])
    kern = int(rng.choice([KERNEL_AUTO, KERNEL_RING, KERNEL_STAGED, KERNEL_DIRECT]))
    bal = [None, True, False][int(rng.integers(0, 3))]
    if algo == "hh":
        w = int(rng.choice([64, 128, 256])); r = int(rng.choice([0, 1, 3, 4, 5]))
        got = engine.to_u64(engine.highway_ragged(key, buf, d_off, d_len, w, r, kernel=kern, balance=bal))
        want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, host, ho, hl, w if w != 128 else 256, r, nthreads=T)
        if w == 128:
            want = want[:, :2]
        desc = f"hh{w} r{r}"
    else:
        c, d = [(2, 4), (1, 3), (3, 5)][int(rng.integers(0, 3))]
        tree = algo == "tree"
        got = engine.to_u64(engine.sip_ragged(k128, buf, d_off, d_len, c, d, tree, kernel=kern, balance=bal))
        want = oracle.batch_ragged(oracle.ALG_SIPTREE if tree else oracle.ALG_SIPHASH, k128, host, ho, hl, c, d, nthreads=T)
        desc = f"{'tree' if tree else 'sip'}{c}{d}"
    ok = _same(got, want)
    cases += 1; digests += n; bad += not ok
    if not ok:
        print("MISMATCH ragged", desc, n, dist, mode, "offform" if use_off_form else "lens", "kernel", kern, "balance", bal,
              "base", base_shift, flush=True)


def fixed_case():
    global cases, digests, bad
    n = int(rng.choice([1, 100, 1023, 1025, 5000, 40000]))
    L = int(rng.choice([0, 1, 8, 12, 31, 32, 33, 48, 63, 64, 65, 100, 128, 144, 256, 1000, 1024, 4096, 4112]))
    raw = torch.empty(n * L + 32, dtype=torch.uint8, device="cuda")
    synth.fill_device(raw[: (n * L + 32) // 8 * 8], int(rng.integers(1, 1 << 30)))
    shift = int(rng.choice([0, 0, 16, 3]))
    m = raw[shift: shift + n * L].view(n, L)
    host = m.cpu().numpy()
    algo = rng.choice(["hh", "sip", "tree"])
    kerns = [KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING]
    if L % 16 == 0 and L >= 32 and shift % 16 == 0:
        kerns.append(KERNEL_TMA)
    if algo == "hh" and L >= 128 and L % 128 == 0 and shift % 16 == 0:
        kerns.append(KERNEL_SPLIT)
    if L <= 64 or algo != "hh":
        kerns.append(KERNEL_STAGED)
    kern = int(rng.choice(kerns))
    try:
        if algo == "hh":
            w = int(rng.choice([64, 128, 256])); r = int(rng.choice([0, 2, 4]))
            got = engine.to_u64(engine.highway_batch(key, m, w, r, kernel=kern))
            want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, host, w if w != 128 else 256, r, nthreads=T)
            if w == 128:
                want = want[:, :2]
            desc = f"hh{w} r{r}"
        else:
            c, d = [(2, 4), (1, 3), (3, 5)][int(rng.integers(0, 3))]
            tree = algo == "tree"
            got = engine.to_u64(engine.sip_batch(k128, m, c, d, tree, kernel=kern))
            want = oracle.batch_fixed(oracle.ALG_SIPTREE if tree else oracle.ALG_SIPHASH, k128, host, c, d, nthreads=T)
            desc = f"{'tree' if tree else 'sip'}{c}{d}"
    except ValueError:
        return  # a kernel that does not take this shape
    ok = _same(got, want)
    cases += 1; digests += n; bad += not ok
    if not ok:
        print("MISMATCH fixed", desc, n, L, "kernel", kern, "shift", shift, flush=True)


while time.time() < t_end:
    (ragged_case if rng.random() < 0.65 else fixed_case)()
print(f"fuzz_parity: {cases} cases, {digests} digests, {bad} mismatching cases in {budget:.0f} s")
sys.exit(1 if bad else 0)
