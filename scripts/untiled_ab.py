#!/usr/bin/env python
"""Fixed-length batches the TMA kernel does not take (row length not a
multiple of 16): direct vs ring vs staged vs KERNEL_AUTO's choice.
CUDA-event median per launch, device-resident rows."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import torch  # noqa: E402

from paper_1612_06257_b200 import engine, synth  # noqa: E402
from paper_1612_06257_b200.engine import (KERNEL_AUTO, KERNEL_DIRECT, KERNEL_RING,  # noqa: E402
                                          KERNEL_STAGED)
from ragged_ab import med  # noqa: E402


def main():
    key = synth.key256()
    for n, L in ((1 << 24, 8), (1 << 24, 12), (1 << 23, 20), (1 << 23, 24), (1 << 22, 33),
                 (1 << 22, 60), (1 << 21, 100), (1 << 20, 200), (1 << 20, 1000),
                 (1 << 18, 4095)):
        buf = torch.empty(n * L, dtype=torch.uint8, device="cuda")
        synth.fill_device(buf, 3)
        m = buf.view(n, L)
        res = {"n": n, "L": L}
        ref = None
        for name, k in (("auto", KERNEL_AUTO), ("direct", KERNEL_DIRECT), ("ring", KERNEL_RING),
                        ("staged", KERNEL_STAGED)):
            if k == KERNEL_STAGED and L > 64:
                continue
            o = torch.empty(n, dtype=torch.int64, device="cuda")
            res[name + "_ms"] = round(med(lambda: engine.highway_batch(key, m, 64, kernel=k,
                                                                       out=o)), 4)
            ref = o if ref is None else ref
            res.setdefault("agree", True)
            res["agree"] &= bool(torch.equal(ref, o))
        print(json.dumps(res), flush=True)
        del buf, m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
