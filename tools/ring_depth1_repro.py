#!/usr/bin/env python
"""Reproducer for the round-1 "depth-1 ring reader" wrong digests (DESIGN.md
§10): seeded random ragged layouts hashed by the staged kernel (whose
fallback inlines the ring reader) and the ring kernel, bit-compared with the
oracle.  Run it against an A/B build:

  LH_NVCC_EXTRA="-DLH_ALLOW_DEPTH1 -DLH_FALLBACK_DEPTH=1 -DLH_RING_DEPTH=1" \\
      python paper_1612_06257_b200/_build.py --so ab/libb200hash_d1.so --obj ab/obj_d1
  LH_LIBRARY=ab/libb200hash_d1.so python tools/ring_depth1_repro.py

Prints one JSON line per (case, kernel, rounds): mismatches, and for the
failing messages their lengths, address alignments and whether their
128-message group took the staged fast path or the fallback.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle  # noqa: E402
from paper_1612_06257_b200 import _lib, engine  # noqa: E402
from paper_1612_06257_b200.engine import KERNEL_RING, KERNEL_STAGED, to_u64  # noqa: E402
from test_gpu_random_layouts import _ragged_case  # noqa: E402


def fast_path_groups(off, lens, n):
    """Host replica of k_ragged_short's per-group fast-path test (MPL 4)."""
    fast = np.zeros(n, bool)
    for base in range(0, n, 128):
        idx = np.arange(base, min(n, base + 128))
        s0 = int(off[base])
        st, ln = off[idx].astype(np.int64), lens[idx].astype(np.int64)
        ok = np.all((ln <= 64) & (st >= s0) & (st + ln - s0 <= 8192))
        fast[idx] = ok
    return fast


def main():
    lib = os.environ.get("LH_LIBRARY", "default")
    bad_total = 0
    for seed in range(8):
        rng = np.random.default_rng(1000 + seed)
        key = rng.integers(0, 2**64, 4, dtype=np.uint64)
        for case in range(4):
            buf, off, lens = _ragged_case(rng)
            shift = int(rng.integers(0, 16))
            raw = torch.from_numpy(np.concatenate([np.zeros(shift, np.uint8), buf])).cuda()
            d_buf = raw[shift:]
            d_off = torch.from_numpy(off.view(np.int64)).cuda()
            d_len = torch.from_numpy(lens.view(np.int32)).cuda()
            fast = fast_path_groups(off, lens, len(lens))
            base_addr = d_buf.data_ptr()
            for rounds in (0, 1, 3, 4):
                want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, lens, 64, rounds)
                for kname, kernel in (("staged", KERNEL_STAGED), ("ring", KERNEL_RING)):
                    got = to_u64(engine.highway_ragged(key, d_buf, d_off, d_len, 64, rounds,
                                                       kernel=kernel, check=False))
                    bad = np.flatnonzero(got != want)
                    bad_total += len(bad)
                    if len(bad) or (case == 0 and rounds == 4):
                        print(json.dumps({
                            "lib": lib, "seed": seed, "case": case, "kernel": kname,
                            "rounds": rounds, "n": len(lens), "bad": int(len(bad)),
                            "bad_lens": np.unique(lens[bad]).tolist()[:20],
                            "bad_align16": np.unique((base_addr + off[bad].astype(np.int64)) % 16
                                                     ).tolist(),
                            "bad_in_fast_group": int(fast[bad].sum()),
                            "fallback_msgs": int((~fast).sum()),
                            "bad_nfull_zero": int((lens[bad] < 32).sum())}), flush=True)
    print(json.dumps({"lib": lib, "version": _lib.version(), "total_bad": bad_total}))


if __name__ == "__main__":
    main()
