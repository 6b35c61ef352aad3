#!/usr/bin/env python
"""A/B of the fixed-length HighwayHash kernels on long-message shapes
(cfg4 and smaller / sharded variants): CUDA-event median per launch,
device-resident inputs, digests cross-checked between kernels.
usage: python scripts/fixed_ab.py [n:L ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1612_06257_b200 import engine, synth  # noqa: E402
from paper_1612_06257_b200.engine import KERNEL_SPLIT, KERNEL_TMA  # noqa: E402


def med(fn, steps=10, warmup=3):
    for _ in range(warmup):
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
    shapes = sys.argv[1:] or ["16384:1048576", "2048:1048576", "4096:1048576", "131072:4096",
                              "65536:1024"]
    key = synth.key256()
    for sh in shapes:
        n, L = (int(x) for x in sh.split(":"))
        buf = torch.empty(n * L, dtype=torch.uint8, device="cuda")
        synth.fill_device(buf, 5)
        m = buf.view(n, L)
        res = {"n": n, "L": L}
        outs = {}
        for name, k in (("tma", KERNEL_TMA), ("split", KERNEL_SPLIT)):
            o = torch.empty((n, 4), dtype=torch.int64, device="cuda")
            ms = med(lambda: engine.highway_batch(key, m, 256, kernel=k, out=o))
            res[name + "_ms"] = round(ms, 4)
            res[name + "_GBs"] = round(n * L / ms / 1e6, 1)
            outs[name] = o
        res["agree"] = bool(torch.equal(outs["tma"], outs["split"]))
        print(json.dumps(res), flush=True)
        del buf, m, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
