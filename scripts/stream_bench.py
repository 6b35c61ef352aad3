#!/usr/bin/env python
"""Streaming (incremental) hashing throughput on the device vs the one-shot
batch over the same bytes: n messages appended in equal fixed-layout chunks.
CUDA-event median of whole passes (init + appends + finish)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import torch  # noqa: E402

from paper_1612_06257_b200 import engine, synth  # noqa: E402
from ragged_ab import med  # noqa: E402


def main():
    key = synth.key256()
    for n, chunk, k in ((1 << 16, 4096, 16), (1 << 20, 1024, 4), (1 << 14, 65536, 4),
                        (1 << 20, 1000, 4)):
        total = n * chunk * k
        chunks = [torch.empty((n, chunk), dtype=torch.uint8, device="cuda") for _ in range(k)]
        for j, c in enumerate(chunks):
            synth.fill_device(c.view(-1), 10 + j)

        def streamed():
            sb = engine.StreamBatch(engine.ALG_HIGHWAY, key, n)
            for c in chunks:
                sb.append(c)
            return sb.finish()

        whole = torch.cat(chunks, dim=1).contiguous()
        ms_s = med(streamed, steps=5, warmup=2)
        ms_o = med(lambda: engine.highway_batch(key, whole, 64), steps=5, warmup=2)
        same = bool(torch.equal(streamed(), engine.highway_batch(key, whole, 64)))
        print(json.dumps({"n": n, "chunk": chunk, "appends": k, "GiB": total / 2**30,
                          "stream_ms": round(ms_s, 3), "stream_GBs": round(total / ms_s / 1e6, 1),
                          "oneshot_ms": round(ms_o, 3), "oneshot_GBs": round(total / ms_o / 1e6, 1),
                          "same_digests": same}), flush=True)
        del chunks, whole
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
