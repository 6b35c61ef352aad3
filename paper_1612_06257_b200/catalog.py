"""Algorithm catalog for the vector file, CLI and harnesses.

Same names, key sizes and digest byte images as the reference registry
(S/registry.py:106-190): ``highway64``, ``highway256``, ``siphash24``,
``siphash13``, ``siptree24``, ``siptree13``, plus ``highway128`` (lanes 0-1
of the 256-bit lane sum; derived, not in the reference).  Digests are the
little-endian byte image, lane 0 first (S/registry.py:54-55,
S/highway.py:288-295).  Every digest is computed on the GPU in batches; the
control hashes of the reference (``first8bytes``, ``constant``,
S/registry.py:162-183) calibrate its quality harness and are not part of
the hash path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Sequence

import numpy as np

from . import _lib


@dataclass(frozen=True)
class Algorithm:
    name: str
    key_size: int
    digest_size: int
    alg: int
    p1: int  # width (HighwayHash) or c (Sip family)
    p2: int  # rounds (HighwayHash) or d

    def _key(self, key: bytes):
        if len(key) != self.key_size:
            raise ValueError(f"{self.name} needs a {self.key_size}-byte key")
        return np.frombuffer(bytes(key), np.uint64).copy()

    def digest_batch(self, key: bytes, messages: Sequence[bytes]) -> np.ndarray:
        """(n, digest_size) uint8 digest images of a list of messages, one
        ragged GPU batch."""
        from . import engine

        k = self._key(key)
        lens = np.array([len(m) for m in messages], dtype=np.uint32)
        off = np.zeros(len(messages), np.uint64)
        if len(messages) > 1:
            off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
        buf = np.frombuffer(b"".join(bytes(m) for m in messages) or b"\0", np.uint8)
        if self.alg == _lib.ALG_HIGHWAY:
            d = engine.highway_ragged(k, buf, off, lens, self.p1, self.p2)
        else:
            d = engine.sip_ragged(k, buf, off, lens, self.p1, self.p2,
                                  tree=self.alg == _lib.ALG_SIPTREE)
        d = np.ascontiguousarray(d.reshape(len(messages), -1).astype("<u8"))
        return d.view(np.uint8).reshape(len(messages), self.digest_size)

    def digest(self, key: bytes, message: bytes) -> bytes:
        return self.digest_batch(key, [message])[0].tobytes()

    def digest_hex(self, key: bytes, message: bytes) -> str:
        return self.digest(key, message).hex()

    def make_hasher(self, key: bytes):
        """Streaming hasher whose finish() returns the digest image bytes."""
        return _Stream(self, self._key(key))


class _Stream:
    def __init__(self, algo: Algorithm, key):
        from . import engine

        self._algo = algo
        if algo.alg == _lib.ALG_HIGHWAY:
            self._sb = engine.StreamBatch(algo.alg, key, 1, width=256, rounds=algo.p2)
        else:
            self._sb = engine.StreamBatch(algo.alg, key[:2], 1, c=algo.p1, d=algo.p2)

    def append(self, chunk: bytes):
        if chunk:
            self._sb.append(np.frombuffer(bytes(chunk), np.uint8).reshape(1, -1))
        return self

    def finish(self) -> bytes:
        from . import engine

        width = self._algo.p1 if self._algo.alg == _lib.ALG_HIGHWAY else None
        d = engine.to_u64(self._sb.finish(width) if width else self._sb.finish())
        return np.ascontiguousarray(d.reshape(-1).astype("<u8")).tobytes()


def _algorithms() -> Dict[str, Algorithm]:
    a = {}
    for w in (64, 128, 256):
        a[f"highway{w}"] = Algorithm(f"highway{w}", 32, w // 8, _lib.ALG_HIGHWAY, w, 4)
    for name, alg, c, d in (("siphash24", _lib.ALG_SIPHASH, 2, 4),
                            ("siphash13", _lib.ALG_SIPHASH, 1, 3),
                            ("siptree24", _lib.ALG_SIPTREE, 2, 4),
                            ("siptree13", _lib.ALG_SIPTREE, 1, 3)):
        a[name] = Algorithm(name, 16, 8, alg, c, d)
    return a


ALGORITHMS = _algorithms()

#: S/registry.py:190 — the algorithms of the conformance vector file.
VECTOR_ALGORITHMS = ("highway64", "highway256", "siphash24", "siphash13", "siptree24",
                     "siptree13")


def get_algorithm(name: str) -> Algorithm:
    try:
        return ALGORITHMS[name]
    except KeyError:
        raise ValueError(f"unknown algorithm: {name!r}") from None


def finalization_variant(rounds: int):
    """HighwayHash-64 with a non-default finalization depth, as a
    ``(key bytes, message bytes) -> int`` callable (S/registry.py:200-204),
    through the selected backend."""
    from .backends import get_backend
    from .highway import Key256

    if rounds < 0:
        raise ValueError("rounds must be >= 0")
    return lambda key, msg: get_backend().hash64(Key256.from_bytes(key), msg, rounds)
