"""cfg2 (lengths ascending, 64 per length) through the ring kernel in natural\norder, with a schedule built once and reused, and with the ordering inside\nevery call: device time per call by graph replay."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "scripts"))
import numpy as np, torch
from functools import partial
from paper_1612_06257_b200 import engine, synth
from paper_1612_06257_b200.engine import KERNEL_RING
from bench_configs import _graph_time
key = synth.key256()
b, off, lens = synth.remainder_sweep_bytes(2, 1024, 64)
d_b = torch.from_numpy(b).cuda(); d_off = torch.from_numpy(off.view(np.int64)).cuda()
n = len(lens); o = torch.empty(n, dtype=torch.int64, device="cuda")
dev = d_b.device
nat = _graph_time(partial(engine.highway_ragged, key, d_b, d_off, None, 64, out=o, check=False))
ref = o.clone()
sched = engine.ragged_order(d_off, None, n, "hh")
k = engine.as_key256(key)
fn = partial(engine.highway_ragged, key, d_b, d_off, None, 64, out=o, check=False, kernel=KERNEL_RING, schedule=sched)
srt = _graph_time(fn)
print("cfg2 natural %.4f ms, precomputed schedule %.4f ms, equal %s" % (nat, srt, torch.equal(ref, o)))
full = _graph_time(partial(engine.highway_ragged, key, d_b, d_off, None, 64, out=o, check=False, balance=True))
print("cfg2 with ordering inside: %.4f ms" % full)
