#!/usr/bin/env python
"""Benchmark of the B200 keyed-hash engine (one JSON line on rank 0).

Headline workload (BASELINE.json metric "HighwayHash GB/s hashed (1 KiB
msgs)"): HighwayHash-64 over 2^24 messages x 1,024 bytes (16 GiB) per GPU --
SURVEY.md §8d's roofline batch, cfg1's message shape scaled up.  Inputs are
generated in HBM by the seeded counter generator (seed 1) before timing and
are 130x the L2 size, so no flush is needed.  One step = one launch of the
hot path over the whole per-GPU batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--scaling weak|strong] [--no-configs]

--gpus N > 1 without torchrun spawns N ranks itself (one process per GPU,
NCCL); under torchrun WORLD_SIZE must equal N.  --scaling weak (default):
2^24 messages per GPU; strong: a fixed global 2^24 x 1 KiB batch (and cfg4's
16,384 x 1 MiB) split by message index (shard.fixed_shard).

The line carries: the headline value and roofline (HBM against
MEASURED_PEAKS.json; the read ceiling measured in this run; the integer roof
from profiles/int_peak.json), burst and sustained (power-capped) regimes,
e2e through the public API from pinned host memory (aggregate over ranks),
the kernels actually launched (torch.profiler/CUPTI), and at N=1 one entry
per BASELINE.json config (cfg1-cfg5, PRF, cfg4's 1/2/4/8-GPU shards) with
its own roofline and CPU baseline.

--impl reference times the reference algorithm's CPU implementation on the
host cores (the oracle port oracle/lh_oracle.c on every thread; the
reference package is Python/numba and does not travel to the GPU box) on
the SAME workload: the full 2^24 x 1 KiB batch per step, generated on the
host by the oracle's twin of the counter generator.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HighwayHash GB/s hashed (1 KiB msgs) at 1/8 GPU; % of HBM/INT-pipe roofline"
UNIT = "GB/s"
MSG_BYTES = 1024
N_MSGS = 1 << 24
DIGEST_BYTES = 8
DATA_SEED = 1


# ---------------------------------------------------------------------------
# Measurement helpers
# ---------------------------------------------------------------------------

def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _ncu_summary():
    """The committed ncu --set full summary of the headline kernel
    (profiles/ncu_summary.json), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler for the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.05, enabled: bool = True):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.power_mw, self.power_limit_mw = [], None
        self.period, self._stop = period, threading.Event()
        self.ok = False
        if not enabled:
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = self._handle(pynvml, index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            try:
                self.power_limit_mw = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h)
            except Exception:
                pass
            self.ok = True
        except Exception:
            pass

    @staticmethod
    def _handle(pynvml, index):
        """NVML handle of CUDA device `index`, matched by PCI address (NVML and
        CUDA may enumerate GPUs in different orders)."""
        try:
            import torch

            p = torch.cuda.get_device_properties(index)
            bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(index)

    def _power_mw(self):
        """Instantaneous board power (NVML_FI_DEV_POWER_INSTANT); the plain
        power reading is a ~1 s average that lags a 100 ms timed region."""
        nv = self.nv
        try:
            fv = nv.nvmlDeviceGetFieldValues(self.h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
            if fv.nvmlReturn == 0:
                v = fv.value
                return int({0: v.dVal, 1: v.uiVal, 2: v.ulVal, 3: v.ullVal, 4: v.sllVal,
                            5: v.siVal}.get(fv.valueType, v.uiVal))
        except Exception:
            pass
        return nv.nvmlDeviceGetPowerUsage(self.h)

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            self.power_mw.append(self._power_mw())
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            self._sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        reasons = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        out = {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
               "reasons": reasons, "samples": len(self.samples)}
        if self.power_mw:  # board power while timing, against the enforced limit
            out["power_w"] = round(float(np.median(self.power_mw)) / 1e3, 1)
            out["power_w_max"] = round(max(self.power_mw) / 1e3, 1)
        if self.power_limit_mw:
            out["power_limit_w"] = round(self.power_limit_mw / 1e3, 1)
        return out


def _host_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0))}


def _threads():
    return len(os.sched_getaffinity(0))


def config_dict(ws: int, scaling: str, per_gpu: int) -> dict:
    """The workload description both arms print (same keys and values)."""
    return {"workload": "hh64_2^24x1KiB (HighwayHash-64, 2^24 messages x 1,024 B per GPU, SURVEY "
                        "§8d roofline batch)" if scaling == "weak" else
                        "hh64_2^24x1KiB_strong (HighwayHash-64, one global batch of 2^24 messages "
                        "x 1,024 B split by message index)",
            "messages_per_gpu": per_gpu, "global_messages": per_gpu * ws if scaling == "weak"
            else N_MSGS, "msg_bytes": MSG_BYTES, "digest_bits": 64, "rounds": 4,
            "parallelism": f"dp{ws} (message-index shards, no collective)",
            "l2": "inputs 16 GiB per GPU >> 126 MB L2; no flush needed"}


# ---------------------------------------------------------------------------
# Distributed control plane (NCCL on GPUs; gloo for the CPU test)
# ---------------------------------------------------------------------------

class Plane:
    """Rank bookkeeping, barriers and max/sum over ranks.  World size 1 is a
    no-op plane."""

    def __init__(self, backend: str, device=None):
        import torch
        import torch.distributed as dist

        self.ws = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", str(self.rank)))
        self.dist = dist if self.ws > 1 else None
        self.device = device
        if self.dist and not dist.is_initialized():
            kw = {"device_id": device} if backend == "nccl" else {}
            dist.init_process_group(backend, **kw)
        self._t = lambda v: torch.tensor([float(v)], dtype=torch.float64,
                                         device=device if backend == "nccl" else "cpu")

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def _reduce(self, v, op):
        if not self.dist:
            return float(v)
        t = self._t(v)
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v):
        return self._reduce(v, self.dist.ReduceOp.MAX if self.dist else None)

    def sum(self, v):
        return self._reduce(v, self.dist.ReduceOp.SUM if self.dist else None)

    def gather_u64(self, v: int):
        """[v of rank 0, v of rank 1, ...] (u64 values)."""
        if not self.dist:
            return [v]
        import torch

        dev = self.device if self.device is not None else "cpu"
        t = torch.tensor([np.array([v], np.uint64).view(np.int64)[0]], dtype=torch.int64,
                         device=dev)
        parts = [torch.zeros_like(t) for _ in range(self.ws)]
        self.dist.all_gather(parts, t)
        return [int(p.item()) & ((1 << 64) - 1) for p in parts]

    def close(self):
        if self.dist and self.dist.is_initialized():
            self.dist.destroy_process_group()


def headline_shard(ws: int, rank: int, scaling: str, n_per_gpu: int):
    """[start, stop) of this rank's messages of the global batch."""
    from paper_1612_06257_b200 import shard

    if scaling == "weak":
        return rank * n_per_gpu, (rank + 1) * n_per_gpu
    return shard.fixed_shard(n_per_gpu, ws, rank)


def summarise(plane: Plane, step_ms, total_ms: float, payload_bytes: int, steps: int,
              scaling: str, global_payload: int):
    """Whole-job value: bytes all ranks hashed / max-over-ranks time."""
    t_max = plane.max(total_ms)
    total_bytes = plane.sum(payload_bytes) if scaling == "weak" else global_payload
    return {"value": total_bytes * steps / (t_max / 1e3) / 1e9, "t_max_ms": t_max,
            "bytes_per_step": total_bytes}


# ---------------------------------------------------------------------------
# Reference arm: the CPU implementation on the same workload
# ---------------------------------------------------------------------------

def cpu_rate(fn, nbytes: int, min_seconds: float, min_passes: int = 1):
    """Run fn until both min_passes and min_seconds are reached; GB/s."""
    times = []
    t_start = time.perf_counter()
    while len(times) < min_passes or time.perf_counter() - t_start < min_seconds:
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return len(times) * nbytes / sum(times) / 1e9, len(times), sum(times)


def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc
    from paper_1612_06257_b200 import synth

    threads = _threads()
    n, L = args.msgs, MSG_BYTES
    msgs = orc.synth_fill(n * L, DATA_SEED, nthreads=threads).reshape(n, L)
    key = synth.key256()
    for _ in range(max(args.warmup, 1)):
        orc.batch_fixed(orc.ALG_HIGHWAY, key, msgs, 64, 4, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.batch_fixed(orc.ALG_HIGHWAY, key, msgs, 64, 4, nthreads=threads)
        times.append(time.perf_counter() - t0)
    secs = sum(times)
    gbs = args.steps * n * L / secs / 1e9
    sample = (f"{args.steps} passes x {n} msgs x {L} B (the whole per-GPU batch, seed 1), "
              f"oracle/lh_oracle.c on {threads} threads, {secs:.2f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / max(1, args.steps) * 1e3, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (counter generator seed 1, generated on the host)",
        "config": config_dict(1, args.scaling, n),
        "cpu_baseline": {"value": round(gbs, 3), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "host": _host_info()},
        "e2e": {"value": round(gbs, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "msgs_per_s": round(args.steps * n / secs, 1),
        "checksum": f"{int(np.bitwise_xor.reduce(orc.batch_fixed(orc.ALG_HIGHWAY, key, msgs, 64, 4, nthreads=threads))):016x}",
    }
    if ws > 1:
        line["note"] = ("rank 0 alone runs the CPU implementation on one rank's batch; GB/s is "
                        "per host, the GPU arm's value is the whole job")
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------

def kernels_of_many(calls):
    """{name: [kernel names]} for each (name, fn) in calls: the GPU kernels
    one call of fn launches, from ONE torch.profiler (CUPTI) session outside
    any timed region (a second session in the same process records nothing).
    Each call runs alone between device syncs inside its own record_function
    range; kernels are assigned to the range they start in."""
    import torch
    from torch.profiler import ProfilerActivity, profile, record_function

    try:
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            for name, fn in calls:
                with record_function("lhcall::" + name):
                    fn()
                    torch.cuda.synchronize()
        evs = prof.events()
        ranges = sorted((e.time_range.start, e.time_range.end, e.name[len("lhcall::"):])
                        for e in evs if e.name.startswith("lhcall::"))
        out = {name: [] for name, _ in calls}
        for e in evs:
            if not str(getattr(e, "device_type", "")).endswith("CUDA"):
                continue
            if "Memcpy" in e.name or "Memset" in e.name or e.name.startswith("lhcall::"):
                continue
            t = e.time_range.start
            owner = [r for r in ranges if r[0] <= t]
            if owner:
                out[owner[-1][2]].append(e.name)
        return out
    except Exception as exc:  # CUPTI unavailable: say so, do not guess
        return {name: [f"unavailable: {type(exc).__name__}: {exc}"] for name, _ in calls}


def _event_ms(fn, steps, warmup, stream):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]


def read_probe_gbs(buf, stream):
    """HBM read ceiling measured now, on this buffer: lh_read_probe (16-byte
    streaming loads), best of 5 launches."""
    import torch

    from paper_1612_06257_b200 import _lib

    sink = torch.zeros(64, dtype=torch.int64, device=buf.device)
    nbytes = buf.numel() & ~15

    def go():
        _lib.check(_lib.lib().lh_read_probe(buf.data_ptr(), nbytes, sink.data_ptr(),
                                            stream.cuda_stream), "lh_read_probe")

    ms = _event_ms(go, 5, 2, stream)
    return nbytes / (min(ms) / 1e3) / 1e9


def run_ours(args):
    import torch

    from paper_1612_06257_b200 import engine, introof, synth

    local = int(os.environ.get("LOCAL_RANK", os.environ.get("RANK", "0")))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    plane = Plane("nccl", dev)
    ws, rank = plane.ws, plane.rank
    key = synth.key256()
    L = MSG_BYTES
    start, stop = headline_shard(ws, rank, args.scaling, args.msgs)
    n = stop - start
    buf = torch.empty(n * L, dtype=torch.uint8, device=dev)
    synth.fill_device(buf, DATA_SEED, word_offset=start * L // 8)
    msgs = buf.view(n, L)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()

    def step():
        engine.highway_batch(key, msgs, 64, 4, out=out)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    plane.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local, enabled=not args.no_clock_sampler) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            step()
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    plane.barrier()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    s = summarise(plane, step_ms, total_ms, n * L, args.steps, args.scaling, N_MSGS * L)
    value, t_max = s["value"], s["t_max_ms"]
    fold = int(np.bitwise_xor.reduce(engine.to_u64(out)))
    folds = plane.gather_u64(fold)

    # --- what ran, and the roofs (outside the timed region) ---
    sustained = None
    if not args.no_sustained:
        sus = _event_ms(step, args.sustained_steps, 0, stream)
        k = min(20, len(sus) // 2)
        with ClockSampler(local, enabled=not args.no_clock_sampler) as sclk:
            tail = _event_ms(step, k, 0, stream)  # clocks of the capped regime
        sustained = {"steps": len(sus) + k,
                     "first20_ms": round(float(np.mean(sus[:k])), 4),
                     "last20_ms": round(float(np.mean(tail)), 4),
                     "first20_GB_per_s": round(n * L / np.mean(sus[:k]) / 1e6, 1),
                     "last20_GB_per_s": round(n * L / np.mean(tail) / 1e6, 1),
                     "last20_clocks": sclk.summary()}
    read_gbs = read_probe_gbs(buf, stream)
    per_launch_ms = float(np.mean(step_ms))
    peak, peak_src = _peaks()
    alg_bytes = n * L + n * DIGEST_BYTES
    achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9
    ncu = _ncu_summary().get("bench_kernel", {})
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": ncu.get("dram_bytes_per_launch"),
            "traffic_source": ncu.get("source"),
            "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg_bytes,
            "kernel": None, "kernels_per_step": None,
            "frac_of_nominal_8000": round(achieved / 8000.0, 4),
            "read_ceiling_measured_gbs": round(read_gbs, 1),
            "frac_of_measured_read_ceiling": round(achieved / read_gbs, 4)}
    ir = introof.launch_roof(introof.highway_mix(L, 64), n)
    if ir:
        ir["frac_canonical"] = round(ir["t_int_canonical_ms"] / per_launch_ms, 4)
        ir["frac_balanced"] = round(ir["t_int_balanced_ms"] / per_launch_ms, 4)
        ir["frac_slot"] = round(ir["t_int_slot_ms"] / per_launch_ms, 4)
        roof["int_pipe"] = ir
        t_hbm = alg_bytes / (read_gbs * 1e9) * 1e3
        roof["t_roof_ms"] = round(max(t_hbm, ir["t_int_balanced_ms"]), 4)
        roof["frac_of_max_read_ceiling_or_int"] = round(roof["t_roof_ms"] / per_launch_ms, 4)

    gather = None
    if ws > 1:
        gather = gather_digests_timed(plane, out, dev)
        if args.peer_gather:  # opt-in: maps rank 0's buffer into every rank (CUDA IPC)
            gather["peer_stores"] = peer_store_steps(args, plane, key, msgs, start, n, stream)
    e2e = run_e2e(args, plane, key, dev, start, n)
    result = None
    if rank == 0:
        result = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_max / args.steps, 4), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (counter generator seed 1, generated in HBM; rank r holds "
                    "messages [start_r, stop_r) of one global batch)",
            "config": config_dict(ws, args.scaling, n),
            "msgs_per_s": round(s["bytes_per_step"] / L * args.steps / (t_max / 1e3), 1),
            **({"steps_ms": [round(x, 3) for x in step_ms]} if args.dump_steps else {}),
            "step_ms": {"min": round(float(np.min(step_ms)), 4),
                        "median": round(float(np.median(step_ms)), 4),
                        "max": round(float(np.max(step_ms)), 4)},
            "regimes": {"burst": {"steps": args.steps, "ms": round(per_launch_ms, 4),
                                  "GB_per_s": round(n * L / per_launch_ms / 1e6, 1)},
                        "sustained": sustained},
            "roofline": roof,
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "checksum": [f"{x:016x}" for x in folds],
            "e2e": e2e,
            **({"gather": gather} if gather else {}),
        }
    if args.scaling == "strong":
        strong = strong_cfg4(args, plane, key, dev)
        if rank == 0:
            result["strong_cfg4"] = strong
    calls = [("headline", step)] if rank == 0 else []
    if rank == 0 and ws == 1:
        if not args.no_configs:
            from scripts import bench_configs

            result["configs"] = bench_configs.run_all(dev, args.config_steps, 3,
                                                      cpu_seconds=args.config_cpu_seconds,
                                                      calls=calls)
        if not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline_headline(args.cpu_seconds)
    if rank == 0:
        # The kernels each timed call launches (one CUPTI session, at the end).
        kn = kernels_of_many(calls)
        head = kn.get("headline", [])
        roof["kernel"] = head[0] if head else None
        roof["kernels_per_step"] = len(head)
        result["gpu_launches"] = len(head) * args.steps
        for row in result.get("configs", []):
            row["kernels"] = kn.get(row["workload"], [])
            row["launches_per_call"] = len(row["kernels"])
    del buf, msgs, out
    torch.cuda.empty_cache()
    plane.barrier()
    if rank == 0:
        print(json.dumps(result), flush=True)
    plane.close()
    return 0


def cpu_baseline_headline(min_seconds: float):
    """The oracle port on every host thread over the first 2^22 messages
    (4 GiB) of the headline batch, repeated for >= min_seconds; plus one core."""
    from oracle import oracle as orc
    from paper_1612_06257_b200 import synth

    threads = _threads()
    n = 1 << 22
    msgs = orc.synth_fill(n * MSG_BYTES, DATA_SEED, nthreads=threads).reshape(n, MSG_BYTES)
    key = synth.key256()
    orc.batch_fixed(orc.ALG_HIGHWAY, key, msgs[: n // 8], 64, 4, nthreads=threads)
    gbs, passes, secs = cpu_rate(
        lambda: orc.batch_fixed(orc.ALG_HIGHWAY, key, msgs, 64, 4, nthreads=threads),
        msgs.nbytes, min_seconds)
    one = msgs[: 1 << 15]
    g1, p1, s1 = cpu_rate(lambda: orc.batch_fixed(orc.ALG_HIGHWAY, key, one, 64, 4, nthreads=1),
                          one.nbytes, 1.0)
    return {"value": round(gbs, 3), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{passes} passes x {n} msgs x {MSG_BYTES} B (first messages of the bench "
                      f"batch), oracle/lh_oracle.c, {threads} threads, {secs:.2f} s",
            "single_core": {"value": round(g1, 3), "unit": UNIT,
                            "sample": f"{p1} passes x {len(one)} msgs, 1 thread, {s1:.2f} s"},
            "host": _host_info()}


def gather_digests_timed(plane: Plane, out, dev):
    """SURVEY §8e's end-of-run exchange, outside the timed region: every
    rank's digest slice all-gathered into one (n_total,) tensor on every
    device (shard.gather_digests: NCCL all-gather over NVLink), timed on the
    device with CUDA events, max over ranks."""
    import torch

    from paper_1612_06257_b200 import shard

    n_total = int(plane.sum(out.shape[0]))
    shard.gather_digests(out, n_total)  # warm-up (communicator setup)
    torch.cuda.synchronize()
    plane.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    full = shard.gather_digests(out, n_total)
    b.record()
    torch.cuda.synchronize()
    ms = plane.max(a.elapsed_time(b))
    nbytes = full.numel() * full.element_size()
    del full
    return {"what": "all-gather of every rank's digests to every rank (shard.gather_digests)",
            "bytes_per_rank_out": nbytes, "ms": round(ms, 4),
            "GB_per_s_per_rank": round(nbytes / ms / 1e6, 1)}


def peer_store_steps(args, plane: Plane, key, msgs, start: int, n: int, stream):
    """The same step with the gather fused in (peer.py): every rank's kernel
    stores its digests straight into rank 0's buffer (CUDA IPC, NVLink).
    Max-over-ranks ms per step, to compare with ms_per_step + the NCCL
    all-gather above."""
    import torch

    from paper_1612_06257_b200 import engine, peer

    n_total = int(plane.sum(n))
    buf = peer.shared_digest_buffer(n_total, 1, root=0)
    mine = buf[start:start + n]  # this rank's messages [start, start + n) of the global batch
    fn = lambda: engine.highway_batch(key, msgs, 64, 4, out=mine)  # noqa: E731
    plane.barrier()
    ms = _event_ms(fn, max(3, args.steps // 2), 2, stream)
    peer.fence()
    t = plane.max(float(np.mean(ms)))
    del mine, buf
    peer.fence()
    return {"what": "each rank's kernel stores its digests into rank 0's buffer (peer.py)",
            "ms_per_step": round(t, 4)}


def run_e2e(args, plane: Plane, key, dev, start: int, n_rank: int):
    """The metric through the public API (engine.highway_batch on a pinned
    host batch): every step copies the inputs H2D and the digests D2H.  N=1:
    the whole headline batch (same config as the kernel and reference arms);
    N>1: --e2e-msgs-multi per rank (host RAM).  Aggregate over ranks: bytes
    all ranks hashed / max-over-ranks wall time."""
    import torch

    from paper_1612_06257_b200 import engine, synth

    n = min(n_rank, args.e2e_msgs if plane.ws == 1 else args.e2e_msgs_multi)
    L = MSG_BYTES
    host = torch.empty((n, L), dtype=torch.uint8, pin_memory=True)
    tmp = torch.empty(n * L, dtype=torch.uint8, device=dev)
    synth.fill_device(tmp, DATA_SEED, word_offset=start * L // 8)
    host.view(-1).copy_(tmp)
    del tmp
    torch.cuda.empty_cache()
    for _ in range(max(1, min(args.warmup, 2))):
        engine.highway_batch(key, host, 64)
    steps = max(1, min(args.steps, args.e2e_steps))
    plane.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        d = engine.highway_batch(key, host, 64)
    dt = time.perf_counter() - t0
    assert d.shape == (n,)
    dt_max = plane.max(dt)
    total = plane.sum(n * L)
    del host
    return {"value": round(total * steps / dt_max / 1e9, 2), "unit": UNIT,
            "h2d_bytes_per_step": int(total), "d2h_bytes_per_step": int(total // L * DIGEST_BYTES),
            "steps": steps, "messages_per_step": int(total // L), "ranks": plane.ws,
            "path": "paper_1612_06257_b200.engine.highway_batch(key, pinned host (n,1024) uint8)"}


def strong_cfg4(args, plane: Plane, key, dev):
    """cfg4 (16,384 x 1 MiB, HighwayHash-256) split by message index across
    the ranks: value = 16 GiB per step / max-over-ranks time."""
    import torch

    from paper_1612_06257_b200 import engine, shard, synth

    n_all, L = 16384, 1 << 20
    a, b = shard.fixed_shard(n_all, plane.ws, plane.rank)
    buf = torch.empty((b - a) * L, dtype=torch.uint8, device=dev)
    synth.fill_device(buf, 5, word_offset=a * L // 8)
    m = buf.view(b - a, L)
    o = torch.empty((b - a, 4), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    steps = max(3, args.steps // 2)
    plane.barrier()
    ms = _event_ms(lambda: engine.highway_batch(key, m, 256, out=o), steps, 2, stream)
    t = plane.max(sum(ms))
    del buf, m, o
    torch.cuda.empty_cache()
    return {"workload": "cfg4 16384 x 1 MiB hh256, strong (fixed global batch)",
            "messages_per_rank": b - a, "ms": round(t / steps, 4),
            "GB_per_s": round(n_all * L * steps / (t / 1e3) / 1e9, 1)}


# ---------------------------------------------------------------------------
# Process launch
# ---------------------------------------------------------------------------

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawned(rank, argv, world, port, entry):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
                       "RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world)})
    sys.exit(entry(parse(argv)) or 0)


def spawn(args, argv, entry=None):
    """--gpus N > 1 without torchrun: one process per GPU, ranks 0..N-1."""
    import torch.multiprocessing as mp

    mp.start_processes(_spawned, args=(argv, args.gpus, _free_port(), entry or run_ours),
                       nprocs=args.gpus, start_method="spawn")
    return 0


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--msgs", type=int, default=N_MSGS)
    ap.add_argument("--e2e-msgs", type=int, default=N_MSGS)
    ap.add_argument("--e2e-msgs-multi", type=int, default=1 << 22)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sustained-steps", type=int, default=150)
    ap.add_argument("--config-steps", type=int, default=20)
    ap.add_argument("--config-cpu-seconds", type=float, default=1.0)
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--peer-gather", action="store_true",
                    help="N > 1: also time the step with digests stored into rank 0 (peer.py)")
    ap.add_argument("--no-sustained", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clock-sampler", action="store_true")
    ap.add_argument("--dump-steps", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    return args


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)
    if "RANK" in os.environ:
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        if ws != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch with "
                             f"torchrun --nproc-per-node {args.gpus}, or without torchrun")
    elif args.gpus > 1:
        return spawn(args, argv)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
