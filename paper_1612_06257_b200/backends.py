"""Backend protocol of the reference, with the CUDA engine as the only backend.

Mirrors ``lanehash.backends`` (S/backends.py:22-118): duck-typed backend
objects with ``name``, ``hash64(key, message, rounds=4)``,
``hash256(key, message, rounds=4)`` and ``hash64_batch(key, messages,
rounds=4)``, plus ``available_backends`` / ``select_backend`` /
``get_backend``.  The reference silently falls back to a scalar backend
when an accelerator fails to import (S/backends.py:83-94); this engine has
no CPU fallback by design (BASELINE.json north_star), so the only backend
is ``"cuda"`` and a missing library or device raises instead.
"""
from __future__ import annotations

from typing import Dict, Optional

from . import engine
from .highway import as_key256


class CudaBackend:
    """B200 engine: every call is a CUDA kernel launch (csrc/lh_engine.cu)."""

    name = "cuda"

    def __init__(self):
        from . import _lib

        _lib.lib()  # load now: an unusable engine fails at selection time

    def hash64(self, key, message: bytes, rounds: int = 4) -> int:
        return int(engine.hash_one(as_key256(key), message, 64, rounds)[0])

    def hash128(self, key, message: bytes, rounds: int = 4):
        out = engine.hash_one(as_key256(key), message, 128, rounds)
        return (int(out[0]), int(out[1]))

    def hash256(self, key, message: bytes, rounds: int = 4):
        out = engine.hash_one(as_key256(key), message, 256, rounds)
        return tuple(int(x) for x in out)

    def hash64_batch(self, key, messages, rounds: int = 4):
        """(n, L) uint8 -> (n,) digests; numpy in -> numpy uint64 out (as
        S/_highway_np.py:116-130), CUDA tensor in -> CUDA int64 tensor out."""
        return engine.highway_batch(key, messages, 64, rounds)

    def hash_batch(self, key, messages, width: int = 64, rounds: int = 4):
        return engine.highway_batch(key, messages, width, rounds)

    def hash_ragged(self, key, buf, offsets, lengths=None, width: int = 64, rounds: int = 4):
        return engine.highway_ragged(key, buf, offsets, lengths, width, rounds)

    def siphash_batch(self, key, messages, c: int = 2, d: int = 4, tree: bool = False):
        return engine.sip_batch(key, messages, c, d, tree)

    def prf64(self, key, start: int, n: int, rounds: int = 4):
        return engine.prf64(key, start, n, rounds)


def available_backends() -> Dict[str, object]:
    """{"cuda": CudaBackend()} — raises if the engine cannot load."""
    return {"cuda": CudaBackend()}


_selected = None


def select_backend(name: Optional[str] = None):
    """Pick the backend (only "cuda" exists) and cache it (S/backends.py:100-113)."""
    global _selected
    if name is not None and name != "cuda":
        raise ValueError(f"unknown or unavailable backend: {name!r}")
    _selected = available_backends()["cuda"]
    return _selected


def get_backend():
    """Currently selected backend, choosing it on first use (S/backends.py:116-118)."""
    return _selected if _selected is not None else select_backend()
