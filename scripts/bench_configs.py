#!/usr/bin/env python
"""Device-resident throughput of every BASELINE.json config (one GPU).

Prints one JSON object per workload (and writes them to --out): GB/s of
payload hashed, messages/s, per-launch ms (CUDA events on the launching
stream, median of --steps after --warmup), and the HBM roofline fraction
against MEASURED_PEAKS.json.  Inputs are generated in HBM by the seeded
counter generator (paper_1612_06257_b200/synth.py).  Not the driver's bench
(bench.py is); this is the per-config table in profiles/.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import ClockSampler  # noqa: E402
from paper_1612_06257_b200 import engine, synth  # noqa: E402

LAST_CLOCKS = {}  # NVML SM clock / throttle reasons of the last timed region


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


SETTLE_S = 2.0  # idle before each workload so none inherits the previous one's power-cap state


def time_launch(fn, steps, warmup):
    torch.cuda.synchronize()
    time.sleep(SETTLE_S)
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    with ClockSampler(torch.cuda.current_device(), period=0.01) as clk:
        ev[0].record(st)
        for i in range(steps):
            fn()
            ev[i + 1].record(st)
        torch.cuda.synchronize()
    LAST_CLOCKS.clear()
    LAST_CLOCKS.update(clk.summary())
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return float(np.median(ms)), float(np.min(ms))


def row(name, ms, payload, nmsgs, alg_bytes, note, extra=None):
    pk = peak_gbs()
    r = {"workload": name, "ms_median": round(ms, 4),
         "GB_per_s": round(payload / ms / 1e6, 1),
         "msgs_per_s": round(nmsgs / ms * 1e3, 1),
         "hbm_alg_bytes": alg_bytes,
         "hbm_frac_of_measured_copy": round(alg_bytes / ms / 1e6 / pk, 4),
         "note": note, "clocks": dict(LAST_CLOCKS)}
    if extra:
        r.update(extra)
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default="")
    ap.add_argument("--settle", type=float, default=SETTLE_S)
    a = ap.parse_args()
    globals()["SETTLE_S"] = a.settle
    dev = torch.device("cuda", 0)
    key, k128 = synth.key256(), synth.key128()
    out = []
    want = set(a.only.split(",")) if a.only else None

    def on(n):
        return want is None or n in want

    def emit(r):
        print(json.dumps(r), flush=True)
        out.append(r)

    # cfg5-shaped 2^24 x 1 KiB batch (seed 6): HH64 + the Sip comparators
    if on("cfg5") or on("hh64"):
        n, L = 1 << 24, 1024
        buf = torch.empty(n * L, dtype=torch.uint8, device=dev)
        synth.fill_device(buf, 6)
        m = buf.view(n, L)
        o = torch.empty(n, dtype=torch.int64, device=dev)
        ms, _ = time_launch(lambda: engine.highway_batch(key, m, 64, out=o), a.steps, a.warmup)
        emit(row("hh64 2^24x1KiB", ms, n * L, n, n * L + 8 * n, "HBM/ALU"))
        for name, c, d, tree in (("siphash24", 2, 4, False), ("siphash13", 1, 3, False),
                                 ("siptree24", 2, 4, True), ("siptree13", 1, 3, True)):
            ms, _ = time_launch(lambda: engine.sip_batch(k128, m, c, d, tree, out=o), a.steps,
                                a.warmup)
            emit(row(f"{name} 2^24x1KiB (cfg5)", ms, n * L, n, n * L + 8 * n, "INT-bound"))
        for w in (128, 256):
            o2 = torch.empty((n, w // 64), dtype=torch.int64, device=dev)
            ms, _ = time_launch(lambda: engine.highway_batch(key, m, w, out=o2), a.steps, a.warmup)
            emit(row(f"hh{w} 2^24x1KiB", ms, n * L, n, n * L + w // 8 * n, "HBM/ALU"))
            del o2
        del buf, m, o
        torch.cuda.empty_cache()

    if on("prf"):
        n = 1 << 28
        o = torch.empty(n, dtype=torch.int64, device=dev)
        ms, _ = time_launch(lambda: engine.prf64(key, 0, n, out=o), a.steps, a.warmup)
        emit(row("prf64 2^28 counters (cfg5)", ms, 0, n, 8 * n, "INT-bound (5 Updates/counter)"))
        del o
        torch.cuda.empty_cache()

    if on("cfg3"):
        n = 1 << 26
        lens = torch.empty(n, dtype=torch.int32, device=dev)
        synth.lengths_device(lens, 3, 8, 64)
        off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        off[1:] = torch.cumsum(lens.to(torch.int64), 0)
        total = int(off[-1])
        buf = torch.empty(total, dtype=torch.uint8, device=dev)
        synth.fill_device(buf, 4)
        o = torch.empty(n, dtype=torch.int64, device=dev)
        offs = off[:-1]
        ms, _ = time_launch(lambda: engine.highway_ragged(key, buf, offs, lens, 64, out=o),
                            a.steps, a.warmup)
        emit(row("cfg3 short keys 2^26 x U[8,64] (offsets+lengths)", ms, total, n,
                 total + 12 * n + 8 * n, "INT-bound (finalization)"))
        for name, c, d, tree in (("siphash24", 2, 4, False), ("siphash13", 1, 3, False)):
            ms, _ = time_launch(lambda: engine.sip_ragged(k128, buf, offs, lens, c, d, tree, out=o),
                                a.steps, a.warmup)
            emit(row(f"cfg3-shaped short keys, {name} (ragged)", ms, total, n,
                     total + 12 * n + 8 * n, "INT-bound"))
        del buf, lens, off, o
        torch.cuda.empty_cache()

    if on("cfg2"):
        b, off, lens = synth.remainder_sweep_bytes(2, 1024, 64)
        d_b = torch.from_numpy(b).to(dev)
        d_off = torch.from_numpy(off.view(np.int64)).to(dev)
        n = len(lens)
        for w in (64, 128, 256):
            o = torch.empty((n, w // 64) if w > 64 else (n,), dtype=torch.int64, device=dev)
            ms, _ = time_launch(lambda: engine.highway_ragged(key, d_b, d_off, None, w, out=o),
                                a.steps, a.warmup)
            emit(row(f"cfg2 remainder sweep L=0..1023 x64 hh{w}", ms, len(b), n,
                     len(b) + 8 * n + w // 8 * n, "L2-resident, launch-bound"))

    if on("cfg4"):
        n, L = 16384, 1 << 20
        buf = torch.empty(n * L, dtype=torch.uint8, device=dev)
        synth.fill_device(buf, 5)
        m = buf.view(n, L)
        o = torch.empty((n, 4), dtype=torch.int64, device=dev)
        ms, _ = time_launch(lambda: engine.highway_batch(key, m, 256, out=o), max(3, a.steps // 4),
                            1)
        emit(row("cfg4 16384 x 1 MiB hh256", ms, n * L, n, n * L + 32 * n,
                 "parallelism-starved: 16384 sequential chains"))
        del buf, m, o
        torch.cuda.empty_cache()

    if on("cfg1"):
        msgs = torch.from_numpy(synth.numpy_bytes(1, (4096, 1024))).to(dev)
        o = torch.empty(4096, dtype=torch.int64, device=dev)
        ms, _ = time_launch(lambda: engine.highway_batch(key, msgs, 64, out=o), a.steps, a.warmup)
        emit(row("cfg1 4096 x 1 KiB hh64", ms, 4096 * 1024, 4096, 4096 * 1032,
                 "L2-resident, launch-bound"))
        # The same call captured 32 times in a CUDA graph: the host launch
        # cost (~9 us per Python call) leaves; the kernel's own time remains.
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(32):
                engine.highway_batch(key, msgs, 64, out=o)
        ms, _ = time_launch(g.replay, max(3, a.steps // 4), 2)
        emit(row("cfg1 4096 x 1 KiB hh64, CUDA-graph replay (per call)", ms / 32, 4096 * 1024,
                 4096, 4096 * 1032, "kernel-bound: 36-Update chain per thread pair"))

    if on("e2e"):
        # End to end from pinned host memory through the public API (H2D, kernel, D2H).
        n, L = 1 << 21, 1024
        host = torch.empty((n, L), dtype=torch.uint8, pin_memory=True)
        tmp = torch.empty(n * L, dtype=torch.uint8, device=dev)
        synth.fill_device(tmp, 1)
        host.view(-1).copy_(tmp)
        del tmp
        engine.highway_batch(key, host, 64)
        t0 = time.perf_counter()
        for _ in range(3):
            engine.highway_batch(key, host, 64)
        dt = (time.perf_counter() - t0) / 3
        emit({"workload": "e2e hh64 2^21 x 1 KiB from pinned host", "ms": round(dt * 1e3, 2),
              "GB_per_s": round(n * L / dt / 1e9, 2)})
        m = 1 << 24  # cfg3-shaped ragged, host-resident (pinned)
        lens = torch.empty(m, dtype=torch.int32, device=dev)
        synth.lengths_device(lens, 3, 8, 64)
        off = torch.zeros(m, dtype=torch.int64, device=dev)
        off[1:] = torch.cumsum(lens.to(torch.int64), 0)[:-1]
        total = int(off[-1] + lens[-1])
        b = torch.empty(total, dtype=torch.uint8, device=dev)
        synth.fill_device(b, 4)
        hb, ho, hl = (t.cpu().pin_memory() for t in (b, off, lens))
        del b, off, lens
        engine.highway_ragged(key, hb, ho, hl, 64)
        t0 = time.perf_counter()
        for _ in range(3):
            engine.highway_ragged(key, hb, ho, hl, 64)
        dt = (time.perf_counter() - t0) / 3
        emit({"workload": "e2e cfg3-shaped ragged 2^24 keys from pinned host", "ms": round(dt * 1e3, 2),
              "GB_per_s_payload": round(total / dt / 1e9, 2),
              "GB_per_s_incl_metadata": round((total + 12 * m) / dt / 1e9, 2),
              "msgs_per_s": round(m / dt, 1)})

    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
