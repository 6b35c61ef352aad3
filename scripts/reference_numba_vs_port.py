#!/usr/bin/env python
"""The reference's own CPU fast path vs the oracle port, same inputs, same box.

BASELINE.md §2 names the reference's numba batch kernel
(`lanehash._kernels.hash_batch`, S/_kernels.py:268-274) as the primary CPU
baseline; bench.py's reference arm times the oracle port
(oracle/lh_oracle.c) because the reference package is not part of the repo.
This script shows the two are the same speed class: it imports the
reference as installed into the git-ignored `baseline/_ref`
(`pip install --no-index --no-deps --target baseline/_ref /root/reference/pkg`)
and times, on a 2^18 x 1 KiB sample of the headline batch (seed 1):

* numba `hash_batch(0, key, msgs, 4, 0)` on 1 core (warm JIT), and on all
  cores with a process pool sharded by message index;
* the oracle port on 1 thread and on all threads;
* the same for SipHash-2-4 (`hash_batch(1, ...)`).

Digests are compared between the two (bit-exact).  Prints one JSON object.
Not part of any test or bench (TEST/MEASUREMENT INFRASTRUCTURE ONLY).
"""
from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, ROOT)

_MSGS = None


def _init(nbytes_per_row, n):
    global _MSGS
    sys.path.insert(0, REF)
    from oracle import oracle as orc

    _MSGS = orc.synth_fill(n * nbytes_per_row, 1, nthreads=1).reshape(n, nbytes_per_row)
    from lanehash import _kernels

    _kernels.hash_batch(0, np.zeros(4, np.uint64), _MSGS[:2], 4, 0)  # JIT warm-up
    _kernels.hash_batch(1, np.zeros(4, np.uint64), _MSGS[:2], 2, 4)


def _shard(args):
    algo, key, a, b, p1, p2 = args
    from lanehash import _kernels

    t0 = time.perf_counter()
    out = _kernels.hash_batch(algo, key, _MSGS[a:b], p1, p2)
    return time.perf_counter() - t0, out


def main():
    if not os.path.isdir(os.path.join(REF, "lanehash")):
        print(json.dumps({"unavailable": f"reference not installed in {REF}"}))
        return 0
    sys.path.insert(0, REF)
    from lanehash import _kernels

    from oracle import oracle as orc
    from paper_1612_06257_b200 import synth

    threads = len(os.sched_getaffinity(0))
    n, L = 1 << 18, 1024
    msgs = orc.synth_fill(n * L, 1, nthreads=threads).reshape(n, L)
    key = synth.key256()
    res = {"sample": f"{n} x {L} B (first messages of the bench batch, seed 1)", "cores": threads,
           "cpu_model": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0]
           .strip(" :\t")}
    for name, algo, p1, p2, oalg, op1, op2, k in (
            ("highway64", 0, 4, 0, orc.ALG_HIGHWAY, 64, 4, key),
            ("siphash24", 1, 2, 4, orc.ALG_SIPHASH, 2, 4, np.concatenate([key[:2], [0, 0]]).astype(np.uint64))):
        _kernels.hash_batch(algo, k, msgs[:16], p1, p2)  # JIT
        one = msgs[: n // 8]
        t0 = time.perf_counter()
        ref1 = _kernels.hash_batch(algo, k, one, p1, p2)
        t_ref1 = time.perf_counter() - t0
        t0 = time.perf_counter()
        port1 = orc.batch_fixed(oalg, k, one, op1, op2, nthreads=1)
        t_port1 = time.perf_counter() - t0
        assert np.array_equal(ref1, port1), name
        # all cores: process pool sharded by message index (each process has the sample)
        with ProcessPoolExecutor(threads, initializer=_init, initargs=(L, n)) as pool:
            cuts = np.linspace(0, n, threads + 1).astype(int)
            jobs = [(algo, k, int(cuts[i]), int(cuts[i + 1]), p1, p2) for i in range(threads)]
            list(pool.map(_shard, jobs))  # warm
            t0 = time.perf_counter()
            parts = list(pool.map(_shard, jobs))
            t_refN = time.perf_counter() - t0
        refN = np.concatenate([p[1] for p in parts])
        t0 = time.perf_counter()
        portN = orc.batch_fixed(oalg, k, msgs, op1, op2, nthreads=threads)
        t_portN = time.perf_counter() - t0
        assert np.array_equal(refN, portN), name
        extra = {}
        if algo == 0:  # the reference's numpy backend (S/_highway_np.py:116-130), 1 core
            from lanehash import _highway_np
            from lanehash.highway import Key256

            k256 = Key256([int(x) for x in key])
            t0 = time.perf_counter()
            npd = _highway_np.hash64_batch(k256, one)
            extra["numpy_backend_1core_GBps"] = round(one.nbytes / (time.perf_counter() - t0) / 1e9,
                                                      3)
            assert np.array_equal(npd, port1), name
        res[name] = {
            **extra,
            "numba_1core_GBps": round(one.nbytes / t_ref1 / 1e9, 3),
            "port_1thread_GBps": round(one.nbytes / t_port1 / 1e9, 3),
            "numba_pool_GBps": round(msgs.nbytes / t_refN / 1e9, 3),
            "port_all_threads_GBps": round(msgs.nbytes / t_portN / 1e9, 3),
            "digests_equal": True,
        }
    print(json.dumps(res))
    return 0


if __name__ == "__main__":
    sys.exit(main())
