import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1612_06257_b200 import engine, synth
n, L = 1 << 21, 1024
host = torch.empty((n, L), dtype=torch.uint8, pin_memory=True)
dev = torch.empty((n, L), dtype=torch.uint8, device="cuda")
host.view(-1)[:] = 7
for _ in range(3): dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()
print("raw H2D single copy: %.1f GB/s" % (5 * n * L / (time.perf_counter() - t) / 1e9))
key = synth.key256()
for chunk in (32, 64, 128, 256, 512):
    engine.HOST_CHUNK_BYTES = chunk << 20
    engine.highway_batch(key, host, 64)
    t = time.perf_counter()
    for _ in range(5): engine.highway_batch(key, host, 64)
    print("e2e chunk %d MiB: %.1f GB/s" % (chunk, 5 * n * L / (time.perf_counter() - t) / 1e9))
