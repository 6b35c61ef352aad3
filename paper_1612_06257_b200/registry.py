"""Catalog of named hash algorithms for the CLI, vector file and harnesses.

The reference's registry (S/registry.py:23-204) with the same names, fields
and byte conventions, so callers of ``lanehash.registry`` port by changing
the import:

* ``Algorithm(name, key_size, digest_size, hash64, digest, make_hasher,
  kernel, control)`` -- ``hash64`` is a ``(key bytes, message bytes) -> int``
  callable or None (256/128-bit digests), ``digest`` returns the
  little-endian byte image (lane 0 first, S/registry.py:54-55,
  S/highway.py:288-295), ``make_hasher(key)`` returns a streaming hasher whose
  ``finish()`` is an int (64-bit digests) or a tuple of lanes (256-bit), and
  ``kernel`` is the reference's jit spec ``(algo id, p1, p2)``
  (S/_kernels.py:237-244: 0 = HighwayHash-64 with p1 = rounds, 1 = SipHash,
  2 = SipTreeHash with p1, p2 = c, d), used by the quality harness.
* ``ALGORITHMS``, ``VECTOR_ALGORITHMS``, ``get_algorithm`` (ValueError for an
  unknown name), ``finalization_variant(rounds)``, ``RandomOracle``.

Every real hash runs on the GPU engine: one-shot calls through the backend
/ sip facade, lists of messages as one ragged GPU batch (``digest_batch``,
added here; the vector file and ``verify`` use it).  ``highway128`` (lanes
0-1 of the 256-bit lane sum; derived) is the one addition.  The two
controls ``first8bytes`` and ``constant`` (S/registry.py:162-183) are
deliberately degenerate "hashes" that calibrate the quality harness; they
are not on the hash path, have no kernel spec and are computed on the host
exactly as the reference does (``control=True``, excluded from the vector
file).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Callable, Dict, Optional, Sequence, Tuple

import numpy as np

from . import _lib

#: (kernel algo id, p1, p2), S/registry.py:18-19.
KernelSpec = Tuple[int, int, int]
#: Engine batch spec: (engine ALG_* id, p1, p2) -- HighwayHash (width,
#: rounds), Sip family (c, d).
EngineSpec = Tuple[int, int, int]


def _le64(value: int) -> bytes:
    return struct.pack("<Q", value & 0xFFFFFFFFFFFFFFFF)


@dataclass(frozen=True)
class Algorithm:
    """One keyed hash exposed under a stable name (S/registry.py:23-38)."""

    name: str
    key_size: int
    digest_size: int
    hash64: Optional[Callable[[bytes, bytes], int]]
    digest: Callable[[bytes, bytes], bytes]
    make_hasher: Callable[[bytes], object]
    kernel: Optional[KernelSpec] = None
    #: Controls are intentionally weak/degenerate and excluded from vectors.
    control: bool = False
    #: How the GPU engine batches this algorithm (None for the controls).
    engine: Optional[EngineSpec] = None

    def digest_hex(self, key: bytes, message: bytes) -> str:
        return self.digest(key, message).hex()

    def digest_batch(self, key: bytes, messages: Sequence[bytes]) -> np.ndarray:
        """(n, digest_size) uint8 digest images of a list of messages: one
        ragged GPU batch (controls: their host definition)."""
        key = bytes(key)
        if len(key) != self.key_size:
            raise ValueError(f"{self.name} needs a {self.key_size}-byte key")
        if self.engine is None:
            rows = [self.digest(key, bytes(m)) for m in messages]
            return np.frombuffer(b"".join(rows), np.uint8).reshape(len(rows), self.digest_size)
        from . import engine

        alg, p1, p2 = self.engine
        lanes = np.frombuffer(key, np.uint64).copy()
        lens = np.array([len(m) for m in messages], dtype=np.uint32)
        off = np.zeros(len(messages), np.uint64)
        if len(messages) > 1:
            off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
        buf = np.frombuffer(b"".join(bytes(m) for m in messages) or b"\0", np.uint8)
        if alg == _lib.ALG_HIGHWAY:
            d = engine.highway_ragged(lanes, buf, off, lens, p1, p2)
        else:
            d = engine.sip_ragged(lanes, buf, off, lens, p1, p2, tree=alg == _lib.ALG_SIPTREE)
        d = np.ascontiguousarray(np.asarray(d).reshape(len(messages), -1).astype("<u8"))
        return d.view(np.uint8).reshape(len(messages), self.digest_size)


# ---------------------------------------------------------------------------
# Real hashes: every call goes to the GPU engine
# ---------------------------------------------------------------------------

def _highway64(key: bytes, message: bytes) -> int:
    from .backends import get_backend
    from .highway import Key256

    return get_backend().hash64(Key256.from_bytes(key), message)


def _highway_lanes(width: int):
    def fn(key: bytes, message: bytes) -> Tuple[int, ...]:
        from .backends import get_backend
        from .highway import Key256

        b = get_backend()
        k = Key256.from_bytes(key)
        return b.hash256(k, message) if width == 256 else b.hash128(k, message)

    return fn


def _sip_fn(c: int, d: int, tree: bool) -> Callable[[bytes, bytes], int]:
    def fn(key: bytes, message: bytes) -> int:
        from . import sip

        f = sip.siptreehash if tree else sip.siphash
        return f(sip.Key128.from_bytes(key), message, sip.SipParams(c, d))

    return fn


class _WideStream:
    """StreamingHasher finishing at a fixed width (S/registry.py:83-95):
    finish() returns the lanes as a tuple."""

    def __init__(self, key: bytes, width: int):
        from .highway import Key256, StreamingHasher

        self._inner = StreamingHasher(Key256.from_bytes(key))
        self._width = width

    def append(self, chunk):
        self._inner.append(chunk)
        return self

    def finish(self):
        return self._inner.finish(self._width)


def _highway64_hasher(key: bytes):
    from .highway import Key256, StreamingHasher

    return StreamingHasher(Key256.from_bytes(key))


def _sip_hasher(c: int, d: int, tree: bool):
    def make(key: bytes):
        from . import sip

        cls = sip.SipTreeHasher if tree else sip.SipHasher
        return cls(sip.Key128.from_bytes(key), sip.SipParams(c, d))

    return make


# ---------------------------------------------------------------------------
# Harness controls (S/registry.py:58-103, 162-183): host-side by design
# ---------------------------------------------------------------------------

def _first8(key: bytes, message: bytes) -> int:
    head = bytes(message[:8])
    return int.from_bytes(head + bytes(8 - len(head)), "little")


class _First8Hasher:
    """Keeps the first 8 bytes; a maximally linear 'hash'."""

    def __init__(self):
        self._head = b""

    def append(self, chunk: bytes) -> "_First8Hasher":
        if len(self._head) < 8:
            self._head = (self._head + bytes(chunk))[:8]
        return self

    def finish(self) -> int:
        return _first8(b"", self._head)


class _ConstantHasher:
    def append(self, chunk: bytes) -> "_ConstantHasher":
        return self

    def finish(self) -> int:
        return 0


class RandomOracle:
    """A fresh random 64-bit output per query (message ignored): the
    avalanche noise-floor calibrator of S/registry.py:76-90 (numpy Philox,
    not a deterministic function of its inputs)."""

    def __init__(self, seed: int = 0):
        self._rng = np.random.Generator(np.random.Philox(seed))

    def __call__(self, key: bytes, message: bytes) -> int:
        return int(self._rng.integers(0, 1 << 64, dtype=np.uint64))


def _algorithms() -> Dict[str, Algorithm]:
    out: Dict[str, Algorithm] = {}

    def add(a: Algorithm) -> None:
        out[a.name] = a

    add(Algorithm("highway64", 32, 8, _highway64, lambda k, m: _le64(_highway64(k, m)),
                  _highway64_hasher, kernel=(0, 4, 0), engine=(_lib.ALG_HIGHWAY, 64, 4)))
    for w in (128, 256):
        fn = _highway_lanes(w)
        add(Algorithm(f"highway{w}", 32, w // 8, None,
                      lambda k, m, fn=fn, w=w: struct.pack(f"<{w // 64}Q", *fn(k, m)),
                      lambda k, w=w: _WideStream(k, w), engine=(_lib.ALG_HIGHWAY, w, 4)))
    for name, c, d, tree in (("siphash24", 2, 4, False), ("siphash13", 1, 3, False),
                             ("siptree24", 2, 4, True), ("siptree13", 1, 3, True)):
        fn = _sip_fn(c, d, tree)
        alg = _lib.ALG_SIPTREE if tree else _lib.ALG_SIPHASH
        add(Algorithm(name, 16, 8, fn, lambda k, m, fn=fn: _le64(fn(k, m)),
                      _sip_hasher(c, d, tree), kernel=(2 if tree else 1, c, d),
                      engine=(alg, c, d)))
    add(Algorithm("first8bytes", 16, 8, _first8, lambda k, m: _le64(_first8(k, m)),
                  lambda k: _First8Hasher(), control=True))
    add(Algorithm("constant", 16, 8, lambda k, m: 0, lambda k, m: _le64(0),
                  lambda k: _ConstantHasher(), control=True))
    return out


ALGORITHMS = _algorithms()

#: S/registry.py:190 -- deterministic, non-control algorithms of the vector file.
VECTOR_ALGORITHMS = ("highway64", "highway256", "siphash24", "siphash13", "siptree24",
                     "siptree13")


def get_algorithm(name: str) -> Algorithm:
    try:
        return ALGORITHMS[name]
    except KeyError:
        raise ValueError(f"unknown algorithm: {name!r}") from None


def finalization_variant(rounds: int) -> Callable[[bytes, bytes], int]:
    """HighwayHash-64 with a non-default finalization depth
    (S/registry.py:200-204), through the selected backend."""
    from .backends import get_backend
    from .highway import Key256

    if rounds < 0:
        raise ValueError("rounds must be >= 0")
    return lambda key, msg: get_backend().hash64(Key256.from_bytes(key), msg, rounds)
