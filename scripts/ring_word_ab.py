#!/usr/bin/env python
"""Ring-kernel word size A/B on ragged batches: random lengths and
constant power-of-two lengths (per-lane strided loads at a 2^k stride).
Prints HighwayHash-64 and SipHash-2-4 / -1-3 ms per launch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1612_06257_b200 import engine, synth  # noqa: E402
from paper_1612_06257_b200.engine import KERNEL_RING  # noqa: E402
from ragged_ab import med, shape  # noqa: E402


def main():
    key, k2 = synth.key256(), synth.key128()
    cases = [("cfg2", None), ("U0_256_2^22", None), ("U0_2048_2^20", None),
             ("U512_1536_2^22", None), ("cfg3", None), ("const256", 256), ("const1024", 1024),
             ("const4096", 4096), ("const1000", 1000)]
    for name, L in cases:
        if L is None:
            b, off, lens = shape(name)
            total = int(off[-1]) + int(lens[-1])
        else:
            n = (1 << 30) // L
            lens = np.full(n, L, np.uint32)
            off = np.arange(n, dtype=np.uint64) * np.uint64(L)
            b, total = None, n * L
        if b is None:
            d_b = torch.empty(total, dtype=torch.uint8, device="cuda")
            synth.fill_device(d_b, 4)
        else:
            d_b = torch.from_numpy(b).cuda()
        d_off = torch.from_numpy(off.view(np.int64)).cuda()
        d_len = torch.from_numpy(lens.view(np.int32)).cuda()
        n = len(lens)
        o = torch.empty(n, dtype=torch.int64, device="cuda")
        r = {"shape": name}
        r["hh64"] = round(med(lambda: engine.highway_ragged(key, d_b, d_off, d_len, 64, out=o,
                                                            kernel=KERNEL_RING), 10, 3), 4)
        r["sip24"] = round(med(lambda: engine.sip_ragged(k2, d_b, d_off, d_len, 2, 4, out=o),
                               10, 3), 4)
        r["sip13"] = round(med(lambda: engine.sip_ragged(k2, d_b, d_off, d_len, 1, 3, out=o),
                               10, 3), 4)
        print(json.dumps(r), flush=True)
        del d_b, d_off, d_len, o
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
