"""Per-size GPU throughput sweep (§8f row 4; the reference's S/bench.py).

The reference times single CPU invocations per size (interleaved sizes,
mode/median estimator, S/bench.py:72-182) for the paper's Table 1 / Fig. 1
(PRESETS, S/bench.py:24-31).  On the GPU the unit is a batch: for each size
L, a device-resident batch of n equal-length messages (about ``batch_bytes``
of payload, at least 2^16 messages) is hashed in one launch, timed with CUDA
events over ``steps`` launches after warm-up, median per launch.  Rows carry
ns/byte and bytes/ns like the reference's report plus GB/s and messages/s.
Digests of every launch are folded into a checksum (the DigestSink idea,
S/bench.py:57-69) so the work is observable.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np

PRESETS: Dict[str, Tuple[int, ...]] = {
    "table1": (8, 31, 32, 63, 64, 1024),  # S/bench.py:26
    "fig1": tuple(sorted(32 * i + off for i in range(13) for off in (0, 9, 18, 27)
                         if 32 * i + off > 0)),  # S/bench.py:28-30
}


@dataclass
class SizeRow:
    algo: str
    size: int
    messages: int
    ms_per_launch: float
    ns_per_byte: float
    bytes_per_ns: float
    msgs_per_s: float
    digest_fold: int  # XOR of every digest word of the last launch


def sweep(algo_name: str, sizes: Sequence[int], batch_bytes: int = 1 << 30,
          steps: int = 10, warmup: int = 3, seed: int = 0, runs: int = 1) -> List[SizeRow]:
    """One row per size.  `runs` repeats the timed block per size; the row
    reports the median over runs of the per-run median launch time (the
    reference's estimator shape, S/bench.py:161-182)."""
    import torch

    from . import engine, synth
    from .registry import get_algorithm

    if steps < 1 or runs < 1:
        raise ValueError("steps and runs must be >= 1")
    algo = get_algorithm(algo_name)
    if algo.engine is None:
        raise ValueError(f"{algo_name} is a harness control, not an engine hash")
    alg, p1, p2 = algo.engine
    dev = torch.device("cuda", torch.cuda.current_device())
    key = synth.key256() if algo.key_size == 32 else synth.key128()
    rows = []
    for L in sizes:
        n = max(1 << 16, min(1 << 26, batch_bytes // max(L, 1)))
        buf = torch.empty(max(1, n * L), dtype=torch.uint8, device=dev)
        synth.fill_device(buf, seed + L)
        m = buf[: n * L].view(n, L)
        lanes = algo.digest_size // 8
        out = torch.empty((n, lanes) if lanes > 1 else (n,), dtype=torch.int64, device=dev)
        if alg == engine.ALG_HIGHWAY:
            def step():
                engine.highway_batch(key, m, p1, p2, out=out)
        else:
            def step():
                engine.sip_batch(key, m, p1, p2, alg == engine.ALG_SIPTREE, out=out)
        for _ in range(warmup):
            step()
        st = torch.cuda.current_stream(dev)
        run_ms = []
        for _ in range(runs):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
            ev[0].record(st)
            for i in range(steps):
                step()
                ev[i + 1].record(st)
            torch.cuda.synchronize()
            run_ms.append(float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(steps)])))
        ms = float(np.median(run_ms))
        fold = int(np.bitwise_xor.reduce(engine.to_u64(out).reshape(-1)))
        nbytes = n * L
        rows.append(SizeRow(algo_name, L, n, ms, ms * 1e6 / nbytes if nbytes else float("nan"),
                            nbytes / (ms * 1e6) if ms else float("inf"), n / ms * 1e3, fold))
        del buf, out
    return rows


def format_rows(rows: List[SizeRow], machine_readable: bool = False) -> str:
    if machine_readable:
        return "\n".join(f"{r.algo},{r.size},{r.ns_per_byte:.6f},{r.bytes_per_ns:.3f},"
                         f"{r.msgs_per_s:.0f},{r.messages}" for r in rows)
    lines = [f"{'algo':>10} {'size':>6} {'ns/byte':>10} {'bytes/ns':>10} {'Gmsg/s':>8} "
             f"{'batch':>9}"]
    for r in rows:
        lines.append(f"{r.algo:>10} {r.size:>6} {r.ns_per_byte:>10.5f} {r.bytes_per_ns:>10.1f} "
                     f"{r.msgs_per_s / 1e9:>8.3f} {r.messages:>9}")
    return "\n".join(lines)
