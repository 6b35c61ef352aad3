"""Child process for tests/test_gpu_bounds.py: every kernel reads a batch
that ends exactly at (or starts exactly at) an unmapped virtual page.

The buffer is placed with the CUDA virtual-memory API (cuMemAddressReserve +
cuMemCreate + cuMemMap of one granule out of a two-granule reservation), so
a single byte read past the batch's last byte (or before its first) is an
illegal-address fault, not a silent read of allocator slack.  The digests
are also checked against the CPU oracle.  Exit 0 = no fault and every digest
matched; a fault surfaces as a CUDA error (the process then exits non-zero).

usage: python tests/_guard_child.py {end|start|control}
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1612_06257_b200 import _lib, synth  # noqa: E402
from paper_1612_06257_b200.engine import (KERNEL_DIRECT, KERNEL_RING, KERNEL_SPLIT,  # noqa: E402
                                          KERNEL_STAGED, KERNEL_TMA)

cu = ctypes.CDLL("libcuda.so.1")
u64, sz, vp = ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p


class Location(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("id", ctypes.c_int)]


class AllocFlags(ctypes.Structure):
    _fields_ = [("compressionType", ctypes.c_ubyte), ("gpuDirectRDMACapable", ctypes.c_ubyte),
                ("usage", ctypes.c_ushort), ("reserved", ctypes.c_ubyte * 4)]


class AllocProp(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("requestedHandleTypes", ctypes.c_int),
                ("location", Location), ("win32HandleMetaData", vp), ("allocFlags", AllocFlags)]


class AccessDesc(ctypes.Structure):
    _fields_ = [("location", Location), ("flags", ctypes.c_int)]


def ck(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: CUresult {rc}")


def guarded(nbytes: int, at_end: bool):
    """Device pointer p with [p, p + nbytes) mapped and the neighbouring page
    (after the end if at_end, else before the start) unmapped."""
    prop = AllocProp()
    prop.type = 1  # CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = 1  # CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = torch.cuda.current_device()
    gran = sz()
    ck(cu.cuMemGetAllocationGranularity(ctypes.byref(gran), ctypes.byref(prop), 0), "granularity")
    g = gran.value
    size = -(-max(nbytes, 1) // g) * g
    base = u64()
    ck(cu.cuMemAddressReserve(ctypes.byref(base), sz(2 * size), sz(g), u64(0), u64(0)), "reserve")
    h = u64()
    ck(cu.cuMemCreate(ctypes.byref(h), sz(size), ctypes.byref(prop), u64(0)), "create")
    mapped = base.value if at_end else base.value + size
    ck(cu.cuMemMap(u64(mapped), sz(size), sz(0), h, u64(0)), "map")
    acc = AccessDesc()
    acc.location.type = 1
    acc.location.id = prop.location.id
    acc.flags = 3  # READWRITE
    ck(cu.cuMemSetAccess(u64(mapped), sz(size), ctypes.byref(acc), sz(1)), "access")
    return mapped + size - nbytes if at_end else mapped


def put(host: np.ndarray, at_end: bool) -> int:
    host = np.ascontiguousarray(host, dtype=np.uint8)
    p = guarded(host.nbytes, at_end)
    if host.nbytes:
        ck(cu.cuMemcpyHtoD_v2(u64(p), host.ctypes.data_as(vp), sz(host.nbytes)), "copy")
    return p


def main(mode: str) -> int:
    at_end = mode != "start"
    torch.cuda.init()
    torch.zeros(1, device="cuda")  # primary context current on this thread
    lib = _lib.lib()
    key = synth.key256()
    k4 = (ctypes.c_uint64 * 4)(*[int(x) for x in key])
    k2 = (ctypes.c_uint64 * 2)(*[int(x) for x in synth.key128()])
    st = torch.cuda.current_stream().cuda_stream
    bad = 0
    if mode == "control":
        # Positive control: one 64-byte row past the mapped end must fault.
        m = synth.counter_bytes(3, 64 * 64).reshape(64, 64)
        p = put(m, True)
        out = torch.empty(65, dtype=torch.int64, device="cuda")
        rc = lib.lh_highway_fixed_kernel(p, 65, 64, k4, 64, 4, out.data_ptr(), st, KERNEL_DIRECT)
        torch.cuda.synchronize()  # raises on the illegal-address fault
        print(f"control: no fault (rc={rc})", flush=True)
        return 0

    def run(name, fn, n, lanes, want):
        nonlocal bad
        out = torch.empty(max(n, 1) * lanes, dtype=torch.int64, device="cuda")
        rc = fn(out.data_ptr())
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint64)[: n * lanes]
        ok = rc == 0 and np.array_equal(got, np.asarray(want).reshape(-1))
        bad += not ok
        print(f"{mode} {name}: {'ok' if ok else f'MISMATCH rc={rc}'}", flush=True)

    # Fixed-length batches (TMA, direct, split) whose last byte is the page's last.
    for n, L in ((300, 1024), (257, 48), (20, 4096), (7, 33)):
        m = synth.counter_bytes(L + 1, n * L).reshape(n, L)
        p = put(m, at_end)
        want = oracle.batch_fixed(oracle.ALG_HIGHWAY, key, m, 256, 4)
        kernels = [KERNEL_DIRECT, KERNEL_RING] + ([KERNEL_TMA] if L % 16 == 0 else []) + \
            ([KERNEL_SPLIT] if L % 128 == 0 else []) + ([KERNEL_STAGED] if L <= 64 else [])
        for kern in kernels:
            run(f"hh256 n={n} L={L} k={kern}",
                lambda o: lib.lh_highway_fixed_kernel(p, n, L, k4, 256, 4, o, st, kern), n, 4, want)
        want = oracle.batch_fixed(oracle.ALG_SIPTREE, synth.key128(), m, 2, 4)
        for kern in [KERNEL_DIRECT, KERNEL_RING] + ([KERNEL_TMA] if L % 16 == 0 else []):
            run(f"tree24 n={n} L={L} k={kern}",
                lambda o: lib.lh_siphash_fixed_kernel(p, n, L, k2, 2, 4, 1, o, st, kern), n, 1,
                want)
    # Ragged batches: short keys, the 0..1023 sweep, unaligned last messages.
    rng = np.random.default_rng(7)
    for name, lens in (("short", rng.integers(0, 65, 3000)), ("sweep", np.arange(1024)),
                       ("long", rng.integers(0, 3000, 500)),
                       ("odd_tail", np.array([5, 64, 63, 1, 37, 31, 33, 1023, 7]))):
        lens = lens.astype(np.uint32)
        off = np.zeros(len(lens) + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        buf = synth.counter_bytes(int(lens.sum()) % 97, int(off[-1]))
        p = put(buf, at_end)
        d_off = torch.from_numpy(off.view(np.int64)).cuda()
        n = len(lens)
        for kern in (KERNEL_STAGED, KERNEL_RING):
            want = oracle.batch_ragged(oracle.ALG_HIGHWAY, key, buf, off, None, 64, 4)
            run(f"ragged hh64 {name} k={kern}",
                lambda o: lib.lh_highway_ragged_kernel(p, d_off.data_ptr(), None, n, k4, 64, 4, o,
                                                       st, kern), n, 1, want)
        want = oracle.batch_ragged(oracle.ALG_SIPHASH, synth.key128(), buf, off, None, 1, 3)
        for kern in (KERNEL_RING, KERNEL_STAGED):
            run(f"ragged sip13 {name} k={kern}",
                lambda o: lib.lh_siphash_ragged_kernel(p, d_off.data_ptr(), None, n, k2, 1, 3, 0, o,
                                                       st, kern), n, 1, want)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
