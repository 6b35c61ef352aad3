#!/usr/bin/env python
"""The reference's quality acceptance criteria (T/test_acceptance.py:142-213)
at their stated scale, run on the GPU engine; prints JSON with timings.
Reference runtimes: pkg/test_output.txt (avalanche 532 s)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1612_06257_b200 import quality  # noqa: E402


def main():
    out = {}
    quality.avalanche_counts(0, [1, 2, 3, 4], (1000, 8), 4, 0)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    worst = {}
    passed = True
    hashes = 0
    for name in ("highway64", "siphash24", "siphash13", "siptree24"):
        rep = quality.run_avalanche(quality.HashUnderTest.from_name(name), range(4, 33),
                                    iterations=20_000, samples=5)
        worst[name] = max(v.median_max_bias for v in rep.verdicts)
        passed = passed and rep.passed
        hashes += sum(5 * 20_000 * (8 * s + 1) for s in range(4, 33))
    dt = time.perf_counter() - t0
    out["avalanche_5x20000_sizes4-32"] = {"worst_median_max_bias": worst, "passed_1pct": passed,
                                          "seconds": round(dt, 3), "hashes": hashes,
                                          "reference_seconds": 532}
    t0 = time.perf_counter()
    fin = {r: quality.finalization_bias_experiment(r, inputs=2**20, seed=9) for r in (2, 3, 4)}
    dt = time.perf_counter() - t0
    out["finalization_2^20_seed9"] = {
        f"r{r}": {"max_bias": f.max_bias, "mean_bias": f.mean_bias} for r, f in fin.items()}
    out["finalization_2^20_seed9"]["ratio_2r_3r"] = fin[2].max_bias / fin[3].max_bias
    out["finalization_2^20_seed9"]["seconds"] = round(dt, 3)
    t0 = time.perf_counter()
    ex = {r: quality.finalization_bias_experiment(r, exhaustive=True, seed=9) for r in (1, 2, 3, 4)}
    dt = time.perf_counter() - t0
    out["finalization_exhaustive_2^24"] = {
        f"r{r}": {"max_bias": f.max_bias, "mean_bias": f.mean_bias} for r, f in ex.items()}
    out["finalization_exhaustive_2^24"]["seconds_4_rounds"] = round(dt, 3)
    out["finalization_exhaustive_2^24"]["hashes"] = 4 * 25 * 2**24
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
