#!/usr/bin/env python
"""Device-resident throughput of every BASELINE.json config (one GPU), each
with its roofline and the CPU baseline of the same config.

``run_all`` is called by bench.py at N=1 (the ``configs`` array of its JSON
line); run directly it prints one JSON object per workload.  Per workload:
per-launch ms (CUDA events on the launching stream, median of ``steps``
after ``warmup``), GB/s of payload, messages/s, the roofline that bounds it
(HBM: algorithmic bytes / launch time against MEASURED_PEAKS.json; INT: the
canonical-op roof of paper_1612_06257_b200/introof.py, canonical and
pipe-balanced), the kernels launched (torch.profiler), and ``cpu_baseline``:
the oracle port (oracle/lh_oracle.c, every host thread) on a bounded sample
of the same config's inputs, repeated for >= cpu_seconds.

Inputs: the seeded counter generator in HBM (synth.py; its host twin
oracle.synth_fill for the CPU samples), seeds per SURVEY §8d.  Ragged
launches use check=False: the layouts are generated here, and the timed
quantity is the hashing kernel (the C ABI's contract).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from functools import partial

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1612_06257_b200 import engine, introof, synth  # noqa: E402


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


SETTLE_S = 1.0  # idle before each row, so none inherits an earlier one's power-cap clocks
LAST_CLOCKS: dict = {}


def _time(fn, steps, warmup, settle=0.0):
    torch.cuda.synchronize()
    if settle:
        time.sleep(settle)
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    from bench import ClockSampler

    with ClockSampler(torch.cuda.current_device(), period=0.005) as clk:
        ev[0].record(st)
        for i in range(steps):
            fn()
            ev[i + 1].record(st)
        torch.cuda.synchronize()
    LAST_CLOCKS.clear()
    LAST_CLOCKS.update(clk.summary())
    return float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]))


def _cpu(fn, nbytes, nmsgs, sample, seconds):
    from bench import _threads, cpu_rate

    fn()  # warm
    gbs, passes, secs = cpu_rate(fn, nbytes, seconds)
    return {"value": round(gbs, 3), "unit": "GB/s", "msgs_per_s": round(passes * nmsgs / secs, 1),
            "cores": _threads(), "kind": "port",
            "sample": f"{sample}; {passes} passes, {secs:.2f} s, oracle/lh_oracle.c"}


def _graph_time(fn, per_graph=16, reps=10):
    """Device time per call: per_graph calls captured in one CUDA graph and
    replayed (no host launch overhead between kernels)."""
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up on a side stream, as torch.cuda.graph requires
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(per_graph):
            fn()
    return _time(g.replay, reps, 2) / per_graph


def _row(name, fn, steps, warmup, payload, nmsgs, alg_bytes, mix, cpu, bound, calls, verbose,
         extra=None):
    ms = _time(fn, steps, warmup, SETTLE_S)
    clocks = dict(LAST_CLOCKS)
    call_ms = None
    if bound == "latency":
        # Small batches: a Python call costs more than its kernel; the
        # fractions use the device time of graph-replayed calls.
        call_ms, ms = ms, _graph_time(fn)
    if calls is not None:  # kernel names: filled in after one profiler session (bench.py)
        calls.append((name, fn))
    pk = peak_gbs()
    hbm = alg_bytes / ms / 1e6
    r = {"workload": name, "ms": round(ms, 4),
         **({"ms_per_python_call": round(call_ms, 4),
             "ms_note": "ms = device time per call (16 calls captured in a CUDA graph, "
                        "replayed); ms_per_python_call includes the host call"}
            if call_ms is not None else {}),
         "GB_per_s": round(payload / ms / 1e6, 1) if payload else None,
         "msgs_per_s": round(nmsgs / ms * 1e3, 1),
         "roofline": {"bound": bound, "hbm_achieved_gbs": round(hbm, 1), "hbm_peak_gbs": pk,
                      "hbm_frac": round(hbm / pk, 4), "alg_bytes": alg_bytes}}
    if mix is not None:
        ir = introof.launch_roof(mix, nmsgs)
        if ir:
            ir["frac_canonical"] = round(ir["t_int_canonical_ms"] / ms, 4)
            ir["frac_balanced"] = round(ir["t_int_balanced_ms"] / ms, 4)
            ir["frac_slot"] = round(ir["t_int_slot_ms"] / ms, 4)
            r["roofline"]["int_pipe"] = ir
    # INT-bound rows: against the ALU-slot bound (the tightest measured one).
    r["roofline"]["frac"] = (r["roofline"]["hbm_frac"] if bound == "hbm" else
                             r["roofline"].get("int_pipe", {}).get("frac_slot"))
    if bound != "hbm":
        r["roofline"]["frac_basis"] = "int_pipe.t_int_slot_ms"
    r["cpu_baseline"] = cpu
    r["clocks"] = {k: clocks.get(k) for k in ("sm_mhz", "reasons", "samples")}
    r.update(extra or {})
    if verbose:
        print(json.dumps(r), flush=True)
    return r


def _mean_mix(fn_mix, lengths):
    """Per-message mean of a length-dependent mix over a length histogram."""
    vals, counts = np.unique(lengths, return_counts=True)
    m = introof.Mix()
    for v, c in zip(vals.tolist(), counts.tolist()):
        m.add(fn_mix(int(v)), c / len(lengths))
    return m


def run_all(dev, steps=20, warmup=3, cpu_seconds=1.0, only=None, calls=None, verbose=False):
    """One row per config.  ``calls`` (a list) collects (workload, fn) so the
    caller can profile every config's launches in one CUPTI session; inputs
    stay alive through the closures until the caller drops the list."""
    from oracle import oracle as orc

    def _row_(*a, extra=None):
        return _row(*a, calls, verbose, extra)

    key, k128 = synth.key256(), synth.key128()
    T = len(os.sched_getaffinity(0))
    rows = []

    def on(n):
        return only is None or n in only

    if on("cfg1"):
        h = synth.numpy_bytes(1, (4096, 1024))
        msgs = torch.from_numpy(h).to(dev)
        o = torch.empty(4096, dtype=torch.int64, device=dev)
        cpu = _cpu(lambda: orc.batch_fixed(orc.ALG_HIGHWAY, key, h, 64, 4, nthreads=T),
                   h.nbytes, 4096, "cfg1 whole (4096 x 1 KiB)", cpu_seconds)
        rows.append(_row_("cfg1 4096 x 1 KiB hh64", partial(engine.highway_batch, key, msgs, 64, out=o),
                         steps * 5, warmup, h.nbytes, 4096, h.nbytes + 8 * 4096,
                         introof.highway_mix(1024), cpu, "latency"))

    if on("cfg2"):
        b, off, lens = synth.remainder_sweep_bytes(2, 1024, 64)
        d_b = torch.from_numpy(b).to(dev)
        d_off = torch.from_numpy(off.view(np.int64)).to(dev)
        n = len(lens)
        for w in (64, 128, 256):
            o = torch.empty((n, w // 64) if w > 64 else (n,), dtype=torch.int64, device=dev)
            cpu = _cpu(lambda: orc.batch_ragged(orc.ALG_HIGHWAY, key, b, off, None, w, 4,
                                                nthreads=T),
                       len(b), n, "cfg2 whole (65,536 ragged msgs)", cpu_seconds)
            rows.append(_row_(f"cfg2 remainder sweep L=0..1023 x64 hh{w}",
                             partial(engine.highway_ragged, key, d_b, d_off, None, w, out=o,
                                     check=False),
                             steps * 5, warmup, len(b), n, len(b) + 8 * n + w // 8 * n,
                             _mean_mix(lambda L: introof.highway_mix(L, w), lens), cpu, "latency"))

    if on("cfg3"):
        n = 1 << 26
        lens = torch.empty(n, dtype=torch.int32, device=dev)
        synth.lengths_device(lens, 3, 8, 64)
        off = torch.zeros(n, dtype=torch.int64, device=dev)
        off[1:] = torch.cumsum(lens[:-1].to(torch.int64), 0)
        total = int(off[-1]) + int(lens[-1])
        buf = torch.empty(total, dtype=torch.uint8, device=dev)
        synth.fill_device(buf, 4)
        o = torch.empty(n, dtype=torch.int64, device=dev)
        hl = lens[: 1 << 22].cpu().numpy().view(np.uint32)
        ho = off[: 1 << 22].cpu().numpy().view(np.uint64)
        hb = orc.synth_fill(int(ho[-1]) + int(hl[-1]), 4, nthreads=T)
        mix = _mean_mix(lambda L: introof.highway_mix(L, 64), hl)
        cpu = _cpu(lambda: orc.batch_ragged(orc.ALG_HIGHWAY, key, hb, ho, hl, 64, 4, nthreads=T),
                   len(hb), len(hl), "first 2^22 cfg3 keys", cpu_seconds)
        rows.append(_row_("cfg3 short keys 2^26 x U[8,64] hh64 (offsets+lengths)",
                         partial(engine.highway_ragged, key, buf, off, lens, 64, out=o, check=False),
                         steps, warmup, total, n, total + 12 * n + 8 * n, mix, cpu, "int"))
        for name, alg, c, d in (("siphash24", orc.ALG_SIPHASH, 2, 4),
                                ("siphash13", orc.ALG_SIPHASH, 1, 3)):
            cpu = _cpu(lambda: orc.batch_ragged(alg, k128, hb, ho, hl, c, d, nthreads=T),
                       len(hb), len(hl), "first 2^22 cfg3 keys", cpu_seconds)
            rows.append(_row_(f"cfg3-shaped 2^26 short keys {name}",
                             partial(engine.sip_ragged, k128, buf, off, lens, c, d, out=o,
                                     check=False),
                             steps, warmup, total, n, total + 20 * n,
                             _mean_mix(lambda L: introof.sip_mix(L, c, d), hl), cpu, "int"))
        if calls is None:  # else the closures keep the inputs for the profiler pass
            del buf, lens, off, o
            torch.cuda.empty_cache()

    if on("ragged"):
        # Not a BASELINE config: random-length ragged messages through the
        # public call (validation + schedule decision + hashing), natural
        # order vs the automatic length-class schedule.
        n = 1 << 20
        lens = torch.empty(n, dtype=torch.int32, device=dev)
        synth.lengths_device(lens, 3, 0, 2048)
        off = torch.zeros(n, dtype=torch.int64, device=dev)
        off[1:] = torch.cumsum(lens[:-1].to(torch.int64), 0)
        total = int(off[-1]) + int(lens[-1])
        buf = torch.empty(total, dtype=torch.uint8, device=dev)
        synth.fill_device(buf, 4)
        o = torch.empty(n, dtype=torch.int64, device=dev)
        hl = lens[: 1 << 18].cpu().numpy().view(np.uint32)
        ho = off[: 1 << 18].cpu().numpy().view(np.uint64)
        hb = orc.synth_fill(int(ho[-1]) + int(hl[-1]), 4, nthreads=T)
        for name, kind, alg, c, d in (("hh64", "hh", orc.ALG_HIGHWAY, 64, 4),
                                      ("siphash24", "sip", orc.ALG_SIPHASH, 2, 4)):
            call = engine.highway_ragged if kind == "hh" else engine.sip_ragged
            k = key if kind == "hh" else k128
            cpu = _cpu(lambda: orc.batch_ragged(alg, k, hb, ho, hl, c, d, nthreads=T),
                       len(hb), len(hl), "first 2^18 messages", cpu_seconds)
            mix = _mean_mix((lambda L: introof.highway_mix(L, 64)) if kind == "hh" else
                            (lambda L: introof.sip_mix(L, c, d)), hl)
            nat = _time(partial(call, k, buf, off, lens, c, d, out=o, balance=False), steps,
                        warmup)
            r = _row_(f"ragged 2^20 x U[0,2048] {name} (checked call, automatic schedule)",
                      partial(call, k, buf, off, lens, c, d, out=o), steps, warmup, total, n,
                      total + 20 * n, mix, cpu, "int", extra={"ms_natural_order": round(nat, 4)})
            rows.append(r)
        if calls is None:
            del buf, lens, off, o
            torch.cuda.empty_cache()

    if on("cfg4"):
        L = 1 << 20
        h = orc.synth_fill(256 * L, 5, nthreads=T).reshape(256, L)
        cpu = _cpu(lambda: orc.batch_fixed(orc.ALG_HIGHWAY, key, h, 256, 4, nthreads=T), h.nbytes,
                   256, "first 256 cfg4 messages (256 MiB)", cpu_seconds)
        buf = torch.empty(16384 * L, dtype=torch.uint8, device=dev)
        synth.fill_device(buf, 5)
        # The whole batch, then the per-GPU shard of a 2/4/8-GPU strong split.
        for n in (16384, 8192, 4096, 2048):
            m = buf[: n * L].view(n, L)
            o = torch.empty((n, 4), dtype=torch.int64, device=dev)
            r = _row_(f"cfg4 {n} x 1 MiB hh256" + ("" if n == 16384 else
                                                   f" (1/{16384 // n} shard of cfg4)"),
                     partial(engine.highway_batch, key, m, 256, out=o), max(3, steps // 2), 1,
                     n * L, n, n * L + 32 * n, introof.highway_mix(L, 256), cpu, "hbm")
            if n < 16384:
                g = 16384 // n
                r["strong_scaling_projection"] = {
                    "gpus": g, "aggregate_GB_per_s": round(16384 * L / r["ms"] / 1e6, 1),
                    "note": f"each of {g} GPUs hashes {n} messages; aggregate = 16 GiB / "
                            f"shard time (no collective in the loop)"}
            rows.append(r)
        if calls is None:
            del buf, m, o
            torch.cuda.empty_cache()

    if on("cfg5"):
        n, L = 1 << 24, 1024
        buf = torch.empty(n * L, dtype=torch.uint8, device=dev)
        synth.fill_device(buf, 6)
        m = buf.view(n, L)
        o = torch.empty(n, dtype=torch.int64, device=dev)
        hs = orc.synth_fill((1 << 18) * L, 6, nthreads=T).reshape(1 << 18, L)
        cpu = _cpu(lambda: orc.batch_fixed(orc.ALG_HIGHWAY, key, hs, 64, 4, nthreads=T), hs.nbytes,
                   len(hs), "first 2^18 cfg5 messages", cpu_seconds)
        rows.append(_row_("cfg5 hh64 2^24 x 1 KiB", partial(engine.highway_batch, key, m, 64, out=o),
                         steps, warmup, n * L, n, n * L + 8 * n, introof.highway_mix(L), cpu,
                         "hbm"))
        for name, alg, c, d, tree in (("siphash24", orc.ALG_SIPHASH, 2, 4, False),
                                      ("siphash13", orc.ALG_SIPHASH, 1, 3, False),
                                      ("siptree24", orc.ALG_SIPTREE, 2, 4, True),
                                      ("siptree13", orc.ALG_SIPTREE, 1, 3, True)):
            cpu = _cpu(lambda: orc.batch_fixed(alg, k128, hs, c, d, nthreads=T), hs.nbytes, len(hs),
                       "first 2^18 cfg5 messages", cpu_seconds)
            mix = introof.siptree_mix(L, c, d) if tree else introof.sip_mix(L, c, d)
            t_hbm = (n * L + 8 * n) / (peak_gbs() * 1e9) * 1e3
            t_int = (introof.launch_roof(mix, n) or {}).get("t_int_balanced_ms", 0)
            rows.append(_row_(f"cfg5 {name} 2^24 x 1 KiB",
                             partial(engine.sip_batch, k128, m, c, d, tree, out=o), steps, warmup,
                             n * L, n, n * L + 8 * n, mix, cpu,
                             "hbm" if t_hbm >= t_int else "int"))
        if calls is None:
            del buf, m, o
            torch.cuda.empty_cache()

    if on("prf"):
        n = 1 << 28
        o = torch.empty(n, dtype=torch.int64, device=dev)
        cpu = _cpu(lambda: orc.prf64(key, 0, 1 << 24, nthreads=T), 0, 1 << 24,
                   "counters 0..2^24-1", cpu_seconds)
        rows.append(_row_("prf64 2^28 counters (cfg5)", partial(engine.prf64, key, 0, n, out=o),
                         steps, warmup, 0, n, 8 * n, introof.prf_mix(), cpu, "int"))
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    ap.add_argument("--cpu-seconds", type=float, default=1.0)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rows = run_all(torch.device("cuda", 0), a.steps, a.warmup, a.cpu_seconds,
                   set(a.only.split(",")) if a.only else None, verbose=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
