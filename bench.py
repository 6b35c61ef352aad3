#!/usr/bin/env python
"""Benchmark of the B200 keyed-hash engine (one JSON line on rank 0).

Workload (BASELINE.json metric "HighwayHash GB/s hashed (1 KiB msgs)"):
HighwayHash-64 over 2^24 messages x 1,024 bytes (16 GiB) per GPU — the
roofline batch of SURVEY.md §8d, cfg1's message shape scaled up.  Inputs are
generated in HBM by the seeded counter generator (seed 1; rank r holds
messages [r*2^24, (r+1)*2^24) of the global batch), so they are resident
before timing and 130x larger than L2 (no flush needed).  One step = one
pass of the hot path over the whole per-GPU batch (one kernel launch).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference algorithm's CPU implementation on the
host cores (the oracle port oracle/lh_oracle.c with every available
thread; the reference package itself is Python/numba and does not travel to
the GPU box) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
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
CPU_SAMPLE_MSGS = 1 << 18  # 256 MiB per CPU step (~70 ms on 16 host threads)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_summary.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return j.get("bench_kernel", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def _int_peak():
    p = os.path.join(ROOT, "profiles", "int_peak.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


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


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline(steps: int, warmup: int = 1, nthreads=None, min_seconds: float = 0.0):
    """Time the oracle port (all host threads) on CPU_SAMPLE_MSGS x 1 KiB of
    the same workload (the first messages of rank 0's shard)."""
    from oracle import oracle as orc
    from paper_1612_06257_b200 import synth

    threads = len(os.sched_getaffinity(0)) if nthreads is None else nthreads
    msgs = synth.counter_bytes(DATA_SEED, CPU_SAMPLE_MSGS * MSG_BYTES).reshape(CPU_SAMPLE_MSGS,
                                                                               MSG_BYTES)
    key = synth.key256()
    for _ in range(max(warmup, 1)):  # untimed warm-up passes
        orc.batch_fixed(orc.ALG_HIGHWAY, key, msgs, 64, 4, nthreads=threads)
    times = []
    t_start = time.perf_counter()
    while len(times) < steps or time.perf_counter() - t_start < min_seconds:
        t0 = time.perf_counter()
        orc.batch_fixed(orc.ALG_HIGHWAY, key, msgs, 64, 4, nthreads=threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    gbs = len(times) * CPU_SAMPLE_MSGS * MSG_BYTES / total / 1e9
    # One core on a smaller slice, for the per-core figure SURVEY.md §8d asks for.
    one = msgs[:CPU_SAMPLE_MSGS // 8]
    t1, n1 = 0.0, 0
    while t1 < 1.0:
        t0 = time.perf_counter()
        orc.batch_fixed(orc.ALG_HIGHWAY, key, one, 64, 4, nthreads=1)
        t1 += time.perf_counter() - t0
        n1 += 1
    return {
        "value": round(gbs, 3), "unit": UNIT, "cores": threads, "kind": "port",
        "sample": f"{len(times)} passes x {CPU_SAMPLE_MSGS} msgs x {MSG_BYTES} B "
                  f"(first messages of the bench batch), oracle/lh_oracle.c, {threads} threads, "
                  f"{total:.2f} s",
        "seconds": total,
        "single_core": {"value": round(n1 * one.nbytes / t1 / 1e9, 3), "unit": UNIT,
                        "sample": f"{n1} passes x {len(one)} msgs, 1 thread, {t1:.2f} s"},
        "host": _host_info(),
    }


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


def len_or(k):
    return max(1, k)


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    cb = cpu_baseline(args.steps, warmup=args.warmup)
    secs = cb["seconds"]
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / len_or(args.steps) * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (counter generator seed 1)",
        "config": {"workload": f"hh64 over {CPU_SAMPLE_MSGS} x 1 KiB per step (bounded sample of "
                               f"the 2^24 x 1 KiB batch)", "messages_per_step": CPU_SAMPLE_MSGS,
                   "msg_bytes": MSG_BYTES, "digest_bits": 64},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                             "single_core", "host")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1612_06257_b200 import _lib, engine, synth

    ws, rank, local = _dist_env()
    distributed = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # launched by torchrun
    if distributed:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    key = synth.key256()
    n, L = args.msgs, MSG_BYTES
    buf = torch.empty(n * L, dtype=torch.uint8, device=dev)
    synth.fill_device(buf, DATA_SEED, word_offset=rank * n * L // 8)
    msgs = buf.view(n, L)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    def step():
        engine.highway_batch(key, msgs, 64, 4, out=out)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(torch.cuda.current_device(), enabled=not args.no_clock_sampler) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            step()
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max = float(t.item())

    # checksum of checksums (validation only, outside the timed region)
    fold_u = np.bitwise_xor.reduce(engine.to_u64(out))
    fold = torch.tensor([int(np.array([fold_u], np.uint64).view(np.int64)[0])],
                        dtype=torch.int64, device=dev)
    folds = [fold.clone() for _ in range(ws)]
    if distributed:
        dist.all_gather(folds, fold)

    payload = n * L
    value = ws * payload * args.steps / (total_ms_max / 1e3) / 1e9
    per_launch_ms = float(np.mean(step_ms))
    peak, peak_src = _peaks()
    alg_bytes = payload + n * DIGEST_BYTES
    achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": _traffic(),
            "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg_bytes,
            "kernel": "k_tma_fixed<Highway,512,3,1>",
            # north_star's nominal 8.0 TB/s HBM figure, reported beside the measured peak
            "frac_of_nominal_8000": round(achieved / 8000.0, 4)}
    intp = _int_peak()
    if intp and intp.get("ops_per_s"):
        ops = (80 * (L // 32 + 4) + 4) * n
        int_t = ops / intp["ops_per_s"]
        roof["int_pipe"] = {"canonical_ops_per_launch": ops, "peak_ops_per_s": intp["ops_per_s"],
                            "t_int_ms": round(int_t * 1e3, 3),
                            "frac": round(int_t / (per_launch_ms / 1e3), 4),
                            "peak_source": "measured (profiles/int_peak.json, tools/intpeak.cu)"}
        read_ceiling = 7260.0  # GB/s, TMA ring with a null consumer (profiles/r1_membench.txt)
        roof["t_roof_ms"] = round(max(int_t, alg_bytes / (read_ceiling * 1e9)) * 1e3, 3)
        roof["frac_of_max_hbm_read_or_int"] = round(roof["t_roof_ms"] / per_launch_ms, 4)

    result = None
    if rank == 0:
        result = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (counter generator seed 1, generated in HBM; rank r holds "
                    "messages [r*2^24,(r+1)*2^24) of one global batch)",
            "config": {"workload": "hh64_2^24x1KiB (HighwayHash-64, 2^24 messages x 1,024 B "
                                   "per GPU, SURVEY §8d roofline batch)",
                       "messages_per_gpu": n, "msg_bytes": L, "digest_bits": 64, "rounds": 4,
                       "parallelism": f"dp{ws} (message-index shards, no collective)",
                       "l2": "inputs 16 GiB per GPU >> 126 MB L2; no flush needed"},
            "msgs_per_s": round(ws * n * args.steps / (total_ms_max / 1e3), 1),
            **({"steps_ms": [round(x, 3) for x in step_ms]} if args.dump_steps else {}),
            "step_ms": {"min": round(float(np.min(step_ms)), 4),
                        "median": round(float(np.median(step_ms)), 4),
                        "max": round(float(np.max(step_ms)), 4)},
            "roofline": roof,
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "checksum": [f"{int(x.item()) & ((1 << 64) - 1):016x}" for x in folds],
        }
    # e2e through the public API with host buffers (pinned), rank-local
    e2e = run_e2e(args, key, dev, rank)
    if distributed:
        dist.barrier()
    if rank == 0:
        result["e2e"] = e2e
        if ws == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = {k: v for k, v in cpu_baseline(
                1, warmup=1, min_seconds=args.cpu_seconds).items() if k != "seconds"}
        print(json.dumps(result), flush=True)
    if distributed:
        dist.destroy_process_group()
    return 0


def run_e2e(args, key, dev, rank):
    """Same metric through engine.highway_batch() on a host-pinned batch:
    every step copies the step's inputs H2D and the digests D2H."""
    import torch

    from paper_1612_06257_b200 import engine, synth

    n, L = args.e2e_msgs, MSG_BYTES
    host = torch.empty((n, L), dtype=torch.uint8, pin_memory=True)
    tmp = torch.empty(n * L, dtype=torch.uint8, device=dev)
    synth.fill_device(tmp, DATA_SEED, word_offset=rank * N_MSGS * L // 8)
    host.view(-1).copy_(tmp)
    del tmp
    torch.cuda.empty_cache()
    for _ in range(max(1, min(args.warmup, 2))):
        engine.highway_batch(key, host, 64)
    steps = max(1, min(args.steps, args.e2e_steps))
    t0 = time.perf_counter()
    for _ in range(steps):
        d = engine.highway_batch(key, host, 64)
    dt = time.perf_counter() - t0
    assert d.shape == (n,)
    return {"value": round(n * L * steps / dt / 1e9, 2), "unit": UNIT,
            "h2d_bytes_per_step": n * L, "d2h_bytes_per_step": n * DIGEST_BYTES,
            "steps": steps, "messages_per_step": n,
            "path": "paper_1612_06257_b200.engine.highway_batch(key, pinned host (n,1024) uint8)"}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--msgs", type=int, default=N_MSGS)
    ap.add_argument("--e2e-msgs", type=int, default=1 << 21)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clock-sampler", action="store_true")
    ap.add_argument("--dump-steps", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
