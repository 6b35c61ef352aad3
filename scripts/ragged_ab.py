#!/usr/bin/env python
"""A/B of the ragged kernels (KERNEL_STAGED vs KERNEL_RING register ring)
on ragged shapes: the cfg2 sweep, the cfg3 short keys, and medium/long
random lengths.  CUDA-event median per launch, device-resident inputs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1612_06257_b200 import engine, synth  # noqa: E402
from paper_1612_06257_b200.engine import KERNEL_RING, KERNEL_STAGED  # noqa: E402


def med(fn, steps=30, warmup=5):
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


def shape(name):
    if name == "cfg2":
        b, off, lens = synth.remainder_sweep_bytes(2, 1024, 64)
        return b, off[:-1], lens
    n, lo, hi = {"cfg3": (1 << 26, 8, 64), "U0_2048_2^20": (1 << 20, 0, 2048),
                 "U512_1536_2^22": (1 << 22, 512, 1536), "U0_256_2^22": (1 << 22, 0, 256),
                 "U64_192_2^24": (1 << 24, 64, 192)}[name]
    lens = synth.lengths(3, n, lo, hi)
    off = np.zeros(n, np.uint64)
    off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
    return None, off, lens


def main():
    key = synth.key256()
    names = sys.argv[1:] or ["cfg2", "U0_256_2^22", "U64_192_2^24", "U0_2048_2^20",
                             "U512_1536_2^22", "cfg3"]
    for name in names:
        b, off, lens = shape(name)
        total = int(off[-1]) + int(lens[-1])
        if b is None:
            d_b = torch.empty(total, dtype=torch.uint8, device="cuda")
            synth.fill_device(d_b, 4)
        else:
            d_b = torch.from_numpy(b).cuda()
        d_off = torch.from_numpy(off.view(np.int64)).cuda()
        d_len = torch.from_numpy(lens.view(np.int32)).cuda()
        n = len(lens)
        o = torch.empty(n, dtype=torch.int64, device="cuda")
        res = {"shape": name, "n": n, "bytes": total}
        ref = None
        for kname, k in (("staged", KERNEL_STAGED), ("ring", KERNEL_RING)):
            ms = med(lambda: engine.highway_ragged(key, d_b, d_off, d_len, 64, out=o, kernel=k))
            res[kname + "_ms"] = round(ms, 4)
            res[kname + "_GBs"] = round(total / ms / 1e6, 1)
            if ref is None:
                ref = o.clone()
            else:
                res["agree"] = bool(torch.equal(ref, o))
        for kname, k in (("sip24_auto", engine.KERNEL_AUTO), ("sip24_ring", KERNEL_RING)):
            ms = med(lambda: engine.sip_ragged(synth.key128(), d_b, d_off, d_len, 2, 4, out=o,
                                               kernel=k), steps=10, warmup=2)
            res[kname + "_ms"] = round(ms, 4)
        print(json.dumps(res), flush=True)
        del d_b, d_off, d_len, o
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
