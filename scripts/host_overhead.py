#!/usr/bin/env python
"""Host-side cost per call of the small-batch entry points (cfg1, cfg2):
CPU wall time per call with no synchronisation (launch-bound batches are
bound by this, not by the kernel), and the kernel time alone from a CUDA
graph replay of the same call."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1612_06257_b200 import _lib, engine, synth  # noqa: E402


def host_us(fn, n=300):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    dt = time.perf_counter() - t
    torch.cuda.synchronize()
    return dt / n * 1e6


def graph_us(fn, reps=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def main():
    key = synth.key256()
    msgs = torch.from_numpy(synth.numpy_bytes(1, (4096, 1024))).cuda()
    o = torch.empty(4096, dtype=torch.int64, device="cuda")
    b, off, lens = synth.remainder_sweep_bytes(2, 1024, 64)
    d_b = torch.from_numpy(b).cuda()
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    o2 = torch.empty(len(lens), dtype=torch.int64, device="cuda")
    lib = _lib.lib()
    k4 = (__import__("ctypes").c_uint64 * 4)(*[int(x) for x in key])
    st = torch.cuda.current_stream().cuda_stream
    rows = {
        "cfg1 engine.highway_batch": lambda: engine.highway_batch(key, msgs, 64, out=o),
        "cfg1 raw ctypes lh_highway_fixed": lambda: lib.lh_highway_fixed(
            msgs.data_ptr(), 4096, 1024, k4, 64, 4, o.data_ptr(), st),
        "cfg1 raw ctypes, n = 0 (argument checks only)": lambda: lib.lh_highway_fixed(
            msgs.data_ptr(), 0, 1024, k4, 64, 4, o.data_ptr(), st),
        "cfg1 raw ctypes, direct kernel (no tensor map)": lambda: lib.lh_highway_fixed_kernel(
            msgs.data_ptr(), 4096, 1024, k4, 64, 4, o.data_ptr(), st, engine.KERNEL_DIRECT),
        "lh_version (bare ctypes call)": lambda: lib.lh_version(),
        "cfg2 engine.highway_ragged": lambda: engine.highway_ragged(key, d_b, d_off, None, 64,
                                                                    out=o2),
        "cfg2 raw ctypes lh_highway_ragged_kernel(ring)": lambda: lib.lh_highway_ragged_kernel(
            d_b.data_ptr(), d_off.data_ptr(), None, len(lens), k4, 64, 4, o2.data_ptr(), st,
            engine.KERNEL_DIRECT),
    }
    for name, fn in rows.items():
        print(json.dumps({"call": name, "host_us_per_call": round(host_us(fn), 2),
                          "graph_replay_us_per_call": round(graph_us(fn), 2)}), flush=True)


if __name__ == "__main__":
    main()
