import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import KERNEL_DIRECT, KERNEL_SPLIT, KERNEL_TMA
key = synth.key256()
for n, L in ((4096, 1024), (65536, 1024), (131072, 1024), (262144, 1024), (600000, 1024), (1 << 20, 256)):
    m = torch.from_numpy(synth.counter_bytes(1, n * L).reshape(n, L)).cuda()
    o = torch.empty(n, dtype=torch.int64, device="cuda")
    res = {}
    for k in (KERNEL_TMA, KERNEL_SPLIT, KERNEL_DIRECT):
        for _ in range(5): engine.highway_batch(key, m, 64, kernel=k, out=o)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(50): engine.highway_batch(key, m, 64, kernel=k, out=o)
        ev[1].record(); torch.cuda.synchronize()
        res[k] = round(ev[0].elapsed_time(ev[1]) / 50 * 1e3, 1)
    print(n, L, "us per launch (tma, split, direct):", res[KERNEL_TMA], res[KERNEL_SPLIT], res[KERNEL_DIRECT])
