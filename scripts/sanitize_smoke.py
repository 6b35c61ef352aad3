#!/usr/bin/env python
"""Every kernel once, small inputs, checked against the oracle -- the program
run under compute-sanitizer (memcheck / racecheck / synccheck, one tool per
call).  Exit 0 only if every digest matches."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1612_06257_b200 import engine, quality, synth  # noqa: E402
from paper_1612_06257_b200.engine import KERNEL_DIRECT, KERNEL_SPLIT, KERNEL_TMA, to_u64  # noqa

key, k2 = synth.key256(), synth.key128()
ok = True


def check(name, got, want):
    global ok
    good = np.array_equal(got, want)
    ok &= good
    print(f"{name}: {'ok' if good else 'MISMATCH'}", flush=True)


for n, L in ((700, 1024), (300, 48), (40, 4096)):
    m = synth.counter_bytes(L, n * L).reshape(n, L)
    d = torch.from_numpy(m).cuda()
    want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, m, 256, 4)
    for kern in (KERNEL_TMA, KERNEL_DIRECT) + ((KERNEL_SPLIT,) if L % 128 == 0 else ()):
        check(f"hh256 n={n} L={L} k={kern}", to_u64(engine.highway_batch(key, d, 256, kernel=kern)), want)
    check(f"sip24 n={n} L={L}", to_u64(engine.sip_batch(k2, d, 2, 4, False, kernel=KERNEL_TMA)),
          oracle.batch_fixed(oracle.ALG_SIPHASH, k2, m, 2, 4))
    check(f"tree13 n={n} L={L}", to_u64(engine.sip_batch(k2, d, 1, 3, True, kernel=KERNEL_TMA)),
          oracle.batch_fixed(oracle.ALG_SIPTREE, k2, m, 1, 3))
lens = synth.lengths(3, 3000, 0, 70)
off = np.zeros(3001, np.uint64)
off[1:] = np.cumsum(lens)
buf = synth.counter_bytes(4, int(off[-1]) + 1)
check("ragged hh64", engine.highway_ragged(key, buf, off, None, 64),
      oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, None, 64, 4))
check("ragged sip13", engine.sip_ragged(k2, buf, off, None, 1, 3),
      oracle.batch_ragged(oracle.ALG_SIPHASH, k2, buf, off, None, 1, 3))
lens2 = synth.lengths(5, 800, 0, 1500)
off2 = np.zeros(801, np.uint64)
off2[1:] = np.cumsum(lens2)
buf2 = synth.counter_bytes(6, int(off2[-1]))  # last message ends at the allocation's end
check("ragged ring hh256", engine.highway_ragged(key, buf2, off2, None, 256, kernel=KERNEL_DIRECT),
      oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf2, off2, None, 256, 4))
check("ragged ring tree24", engine.sip_ragged(k2, buf2, off2, None, 2, 4, True, kernel=KERNEL_DIRECT),
      oracle.batch_ragged(oracle.ALG_SIPTREE, k2, buf2, off2, None, 2, 4))
check("prf", to_u64(engine.prf64(key, 5, 3000)), oracle.prf64(key, 5, 3000))
sb = engine.StreamBatch(engine.ALG_HIGHWAY, key, 3000)
half = off[:-1] + (lens // 2).astype(np.uint64)
sb.append(buf, off[:-1], (lens // 2).astype(np.uint32))
sb.append(buf, half, (lens - lens // 2).astype(np.uint32))
check("stream", to_u64(sb.finish()), oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, None, 64, 4))
msgs = synth.counter_bytes(9, 200 * 12).reshape(200, 12)
check("avalanche", quality.avalanche_counts(0, key, msgs, 4, 0),
      oracle.avalanche_counts(0, key, msgs, 4, 0))
t = torch.empty(1001, dtype=torch.uint8, device="cuda")
synth.fill_device(t, 3)
check("synth", t.cpu().numpy(), synth.counter_bytes(3, 1001))
torch.cuda.synchronize()
sys.exit(0 if ok else 1)
