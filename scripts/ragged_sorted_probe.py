#!/usr/bin/env python
"""How much a length-grouped schedule would buy on random-length ragged
batches: the same (offsets, lengths) arrays in natural order and permuted by
descending length class, through the existing ring kernel (digests come out
permuted; only the time is compared)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import KERNEL_RING, KERNEL_AUTO
from ragged_ab import med

key = synth.key256()
for name, (n, lo, hi) in {"U0_2048_2^20": (1 << 20, 0, 2048), "U512_1536_2^22": (1 << 22, 512, 1536),
                          "U0_256_2^22": (1 << 22, 0, 256), "U64_192_2^24": (1 << 24, 64, 192),
                          "U0_8192_2^18": (1 << 18, 0, 8192)}.items():
    lens = synth.lengths(3, n, lo, hi)
    off = np.zeros(n, np.uint64); off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
    total = int(off[-1]) + int(lens[-1])
    d_b = torch.empty(total, dtype=torch.uint8, device="cuda"); synth.fill_device(d_b, 4)
    perm = np.argsort(-(lens.astype(np.int64) >> 5), kind="stable")
    res = {"shape": name, "n": n, "GiB": round(total / 2**30, 2)}
    o = torch.empty(n, dtype=torch.int64, device="cuda")
    for tag, oo, ll in (("natural", off, lens), ("sorted", off[perm], lens[perm])):
        d_off = torch.from_numpy(oo.view(np.int64)).cuda(); d_len = torch.from_numpy(ll.view(np.int32)).cuda()
        for kn, k in (("hh_ring", KERNEL_RING),):
            ms = med(lambda: engine.highway_ragged(key, d_b, d_off, d_len, 64, out=o, kernel=k, check=False), steps=10, warmup=3)
            res[f"{kn}_{tag}_ms"] = round(ms, 4); res[f"{kn}_{tag}_GBs"] = round(total / ms / 1e6, 1)
        ms = med(lambda: engine.sip_ragged(synth.key128(), d_b, d_off, d_len, 2, 4, out=o, kernel=KERNEL_RING, check=False), steps=10, warmup=3)
        res[f"sip24_ring_{tag}_ms"] = round(ms, 4)
    print(json.dumps(res), flush=True)
    del d_b; torch.cuda.empty_cache()
