"""Reference-side binding: a ``CudaBackend`` for lanehash's backend protocol
(S/backends.py:22-80) over the C ABI, as a lanehash maintainer would add it.

Plain ctypes + the CUDA runtime; no torch.  Register it in
``available_backends()`` (S/backends.py:83-94) and list "cuda" first in
``select_backend`` (:103).  tests/test_gpu_integration.py runs it.
"""
import ctypes
import ctypes.util
import glob
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("LANEHASH_B200_SO",
                     os.path.join(os.path.dirname(_HERE), "paper_1612_06257_b200", "libb200hash.so"))


def _load_cudart():
    cands = [ctypes.util.find_library("cudart")]
    try:  # the CUDA runtime that ships with torch, if present
        import importlib.util

        spec = importlib.util.find_spec("nvidia.cuda_runtime")
        if spec and spec.submodule_search_locations:
            for d in spec.submodule_search_locations:
                cands += glob.glob(os.path.join(d, "lib", "libcudart.so*"))
    except Exception:
        pass
    cands += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    for c in cands:
        if c:
            try:
                return ctypes.CDLL(c)
            except OSError:
                continue
    raise OSError("libcudart not found")


_so = ctypes.CDLL(_SO)
_cudart = _load_cudart()
vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
_so.lh_highway_fixed.argtypes = [vp, u64, u64, vp, i32, i32, vp, vp]
_so.lh_highway_fixed.restype = i32
_so.lh_strerror.argtypes = [i32]
_so.lh_strerror.restype = ctypes.c_char_p
_cudart.cudaMalloc.argtypes = [ctypes.POINTER(vp), ctypes.c_size_t]
_cudart.cudaFree.argtypes = [vp]
_cudart.cudaMemcpy.argtypes = [vp, vp, ctypes.c_size_t, ctypes.c_int]
H2D, D2H = 1, 2


def _check(rc):
    if rc:  # LH_EINVAL / LH_EALIGN / LH_ETOOBIG -> ValueError, as the reference raises
        msg = _so.lh_strerror(rc).decode()
        raise (ValueError if rc in (-1, -2, -5) else RuntimeError)(msg)


class CudaBackend:
    name = "cuda"

    def _run(self, key, messages, width, rounds):
        msgs = np.ascontiguousarray(messages, dtype=np.uint8)
        n, L = msgs.shape
        lanes = width // 64
        d_in, d_out = vp(), vp()
        if _cudart.cudaMalloc(ctypes.byref(d_in), max(1, msgs.nbytes)) or \
                _cudart.cudaMalloc(ctypes.byref(d_out), max(8, n * lanes * 8)):
            raise RuntimeError("cudaMalloc failed")
        try:
            _cudart.cudaMemcpy(d_in, msgs.ctypes.data, msgs.nbytes, H2D)
            k = (ctypes.c_uint64 * 4)(*key.lanes)
            _check(_so.lh_highway_fixed(d_in, n, L, k, width, rounds, d_out, None))
            out = np.empty((n, lanes), np.uint64)
            _cudart.cudaMemcpy(out.ctypes.data, d_out, out.nbytes, D2H)  # synchronises
        finally:
            _cudart.cudaFree(d_in)
            _cudart.cudaFree(d_out)
        return out

    def hash64(self, key, message, rounds=4):  # S/backends.py:28-29
        row = np.frombuffer(bytes(message), np.uint8).reshape(1, -1)
        return int(self._run(key, row, 64, rounds)[0, 0])

    def hash256(self, key, message, rounds=4):  # S/backends.py:32-33
        row = np.frombuffer(bytes(message), np.uint8).reshape(1, -1)
        return tuple(int(x) for x in self._run(key, row, 256, rounds)[0])

    def hash64_batch(self, key, messages, rounds=4):  # S/backends.py:52-53
        return self._run(key, messages, 64, rounds)[:, 0]
