"""One process, several GPUs: host batches split by message index across
devices ("one Python process with one host thread and one
stream per device").

Each device hashes a contiguous shard of the batch (``shard.fixed_shard``
for fixed-length rows, byte-balanced ``shard.ragged_cuts`` for ragged
batches) in its own host thread: the engine's ctypes calls and torch's
copies release the GIL, so the shards' H2D copies (one PCIe link per GPU),
kernels and D2H copies run concurrently.  Digests land directly in their
slice of one host array: no collective, and the gather is the final copy.
The multi-process form (torchrun, one rank per GPU, NCCL all-gather) is
``shard.gather_digests`` / bench.py.
"""
from __future__ import annotations

import threading
from typing import Optional, Sequence

import numpy as np
import torch

from . import engine, shard


def _devices(devices: Optional[Sequence[int]]):
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    if not devices:
        raise engine._lib.EngineError("no CUDA device: the B200 engine has no CPU fallback")
    return list(devices)


def _run_threads(jobs):
    engine._lib.lib()  # load the library once, before the threads
    errors = []

    def wrap(fn):
        def run():
            try:
                fn()
            except BaseException as e:  # surfaced in the caller's thread
                errors.append(e)
        return run

    threads = [threading.Thread(target=wrap(j)) for j in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]


def highway_batch(key, messages, width: int = 64, rounds: int = 4,
                  devices: Optional[Sequence[int]] = None) -> np.ndarray:
    """HighwayHash of every row of a host (n, L) uint8 batch over several
    GPUs; returns numpy uint64 (n,) or (n, width/64)."""
    return _fixed("hh", key, messages, width, rounds, 0, devices)


def sip_batch(key, messages, c: int = 2, d: int = 4, tree: bool = False,
              devices: Optional[Sequence[int]] = None) -> np.ndarray:
    return _fixed("sip", key, messages, c, d, tree, devices)


def _fixed(kind, key, messages, p1, p2, tree, devices):
    devs = _devices(devices)
    m = engine._as_u8_2d(messages)
    if m.is_cuda:
        raise ValueError("multi-GPU batches take host arrays")
    n = m.shape[0]
    lanes = p1 // 64 if kind == "hh" else 1
    out = np.empty((n, lanes) if lanes > 1 else (n,), np.uint64)
    jobs = []
    for r, dev in enumerate(devs):
        a, b = shard.fixed_shard(n, len(devs), r)
        if b <= a:
            continue

        def job(a=a, b=b, dev=dev):
            with torch.cuda.device(dev):
                if kind == "hh":
                    out[a:b] = engine.highway_batch(key, m[a:b], p1, p2)
                else:
                    out[a:b] = engine.sip_batch(key, m[a:b], p1, p2, tree)
        jobs.append(job)
    _run_threads(jobs)
    return out


def highway_ragged(key, buf, offsets, lengths=None, width: int = 64, rounds: int = 4,
                   devices: Optional[Sequence[int]] = None) -> np.ndarray:
    """Ragged host batch over several GPUs, cut at byte quantiles."""
    devs = _devices(devices)
    off = np.ascontiguousarray(offsets).astype(np.uint64, copy=False)
    lens = None if lengths is None else np.ascontiguousarray(lengths).astype(np.uint32,
                                                                             copy=False)
    n = len(off) - 1 if lens is None else len(off)
    lanes = width // 64
    out = np.empty((n, lanes) if lanes > 1 else (n,), np.uint64)
    cuts = shard.ragged_cuts(off, lens, len(devs))
    jobs = []
    for r, dev in enumerate(devs):
        a, b = int(cuts[r]), int(cuts[r + 1])
        if b <= a:
            continue

        def job(a=a, b=b, dev=dev):
            with torch.cuda.device(dev):
                if lens is None:
                    out[a:b] = engine.highway_ragged(key, buf, off[a:b + 1], None, width, rounds)
                else:
                    out[a:b] = engine.highway_ragged(key, buf, off[a:b], lens[a:b], width, rounds)
        jobs.append(job)
    _run_threads(jobs)
    return out
