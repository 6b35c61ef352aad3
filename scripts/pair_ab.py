#!/usr/bin/env python
"""A/B of the pair-split ring kernel (k_ragged_pair) vs the one-thread ring
(k_ragged_ring) on ragged HighwayHash shapes; run once per setting of
LH_PAIR_MAX_PER_SM (read once per process).  Prints one JSON line per shape."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1612_06257_b200 import engine, synth  # noqa: E402
from paper_1612_06257_b200.engine import KERNEL_RING  # noqa: E402


def timeit(fn, steps=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record()
    for i in range(steps):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    return float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]))


def main():
    key = synth.key256()
    tag = os.environ.get("LH_PAIR_MAX_PER_SM", "default")
    shapes = []
    b, off, lens = synth.remainder_sweep_bytes(2, 1024, 64)
    shapes.append(("cfg2 sweep", b, off, None))
    for n, hi in ((16384, 2048), (65536, 2048), (131072, 2048), (1 << 20, 2048), (65536, 300)):
        lens = synth.lengths(9, n, 0, hi)
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        shapes.append((f"U[0,{hi}] n={n}", synth.counter_bytes(10, int(off[-1])), off, None))
    for name, buf, off, _ in shapes:
        d_b = torch.from_numpy(buf).cuda()
        d_o = torch.from_numpy(off.view(np.int64)).cuda()
        n = len(off) - 1
        for w in (64, 256):
            o = torch.empty((n, w // 64) if w > 64 else (n,), dtype=torch.int64, device="cuda")
            ms = timeit(lambda: engine.highway_ragged(key, d_b, d_o, None, w, out=o,
                                                      kernel=KERNEL_RING, check=False))
            print(json.dumps({"pair_max_per_sm": tag, "shape": name, "width": w, "n": n,
                              "ms": round(ms, 4), "GB_per_s": round(len(buf) / ms / 1e6, 1),
                              "fold": f"{int(np.bitwise_xor.reduce(engine.to_u64(o).reshape(-1))):016x}"}),
                  flush=True)


if __name__ == "__main__":
    main()
