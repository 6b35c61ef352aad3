#!/usr/bin/env python
"""Random-length ragged batches through the public ragged API: natural
order (balance=False) vs the length-class schedule (balance=True, which
includes the three ordering launches) and the automatic choice (check=True:
validation pass + decision).  CUDA-event medians, device-resident inputs."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1612_06257_b200 import engine, synth
from ragged_ab import med

SHAPES = {"U0_2048_2^20": (1 << 20, 0, 2048), "U512_1536_2^22": (1 << 22, 512, 1536),
          "U0_256_2^22": (1 << 22, 0, 256), "U64_192_2^24": (1 << 24, 64, 192),
          "U0_8192_2^18": (1 << 18, 0, 8192), "U0_1024_2^16": (1 << 16, 0, 1024),
          "fixed1000_2^20": (1 << 20, 1000, 1000)}
key, k128 = synth.key256(), synth.key128()
for name in sys.argv[1:] or SHAPES:
    n, lo, hi = SHAPES[name]
    lens = synth.lengths(3, n, lo, hi)
    off = np.zeros(n, np.uint64); off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
    total = int(off[-1]) + int(lens[-1])
    d_b = torch.empty(total, dtype=torch.uint8, device="cuda"); synth.fill_device(d_b, 4)
    d_off = torch.from_numpy(off.view(np.int64)).cuda(); d_len = torch.from_numpy(lens.view(np.int32)).cuda()
    o = torch.empty(n, dtype=torch.int64, device="cuda")
    res = {"shape": name, "n": n, "GiB": round(total / 2**30, 2)}
    for k in ("hh", "sip"):
        _, _, (ws, wm) = engine._plan(d_off, d_len, n, n, total, d_b.device, k)
        res["eff_" + k] = ws / wm
        sv, c = engine.balance_gain(k, 2 if k == "sip" else 4, n, ws, wm)
        res["model_" + k] = [round(sv * 1e3, 4), round(c * 1e3, 4)]
    ref = {}
    for tag, kw in (("natural", dict(check=False, balance=False)), ("ordered", dict(check=False, balance=True)),
                    ("auto_checked", dict(check=True)), ("natural_checked", dict(check=True, balance=False))):
        ms = med(lambda: engine.highway_ragged(key, d_b, d_off, d_len, 64, out=o, **kw), steps=10, warmup=3)
        res[f"hh_{tag}_ms"] = round(ms, 4)
        ref.setdefault("hh", o.clone()); assert torch.equal(ref["hh"], o)
        ms = med(lambda: engine.sip_ragged(k128, d_b, d_off, d_len, 2, 4, out=o, **kw), steps=10, warmup=3)
        res[f"sip24_{tag}_ms"] = round(ms, 4)
        ref.setdefault("sip", o.clone()); assert torch.equal(ref["sip"], o)
    res["eff_hh"] = round(res["eff_hh"], 3); res["eff_sip"] = round(res["eff_sip"], 3)
    print(json.dumps(res), flush=True)
    del d_b; torch.cuda.empty_cache()
