"""SipHash-c-d and SipTreeHash types and one-shot API on the B200 engine.

Mirrors ``lanehash.sip`` (S/sip.py): ``Key128`` (:24-50), ``SipParams``
(:53-66) with ``SIPHASH_24`` / ``SIPHASH_13`` (:69-70), ``siphash`` (:89-108)
and ``siptreehash`` (:124-128), same argument meaning and errors.  Digests
are computed by the CUDA library (csrc/lh_device.cuh: Sip / SipTree).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Tuple

_MASK64 = 0xFFFFFFFFFFFFFFFF


class Key128:
    """128-bit SipHash key as two little-endian 64-bit words."""

    __slots__ = ("k0", "k1")

    def __init__(self, k0: int, k1: int):
        self.k0 = int(k0) & _MASK64
        self.k1 = int(k1) & _MASK64

    @classmethod
    def from_bytes(cls, raw: bytes) -> "Key128":
        if len(raw) != 16:
            raise ValueError("Key128 requires exactly 16 bytes")
        return cls(*struct.unpack("<2Q", raw))

    @classmethod
    def from_hex(cls, text: str) -> "Key128":
        return cls.from_bytes(bytes.fromhex(text))

    def to_bytes(self) -> bytes:
        return struct.pack("<2Q", self.k0, self.k1)

    @property
    def lanes(self):
        return (self.k0, self.k1)

    def __eq__(self, other: object) -> bool:
        return isinstance(other, Key128) and (self.k0, self.k1) == (other.k0, other.k1)

    def __hash__(self) -> int:
        return hash((self.k0, self.k1))

    def __repr__(self) -> str:
        return f"Key128({self.to_bytes().hex()})"


def as_key128(key) -> Key128:
    if isinstance(key, Key128):
        return key
    if isinstance(key, (bytes, bytearray, memoryview)):
        return Key128.from_bytes(bytes(key))
    k = [int(x) for x in key]
    if len(k) != 2:
        raise ValueError("Key128 requires exactly 2 words")
    return Key128(*k)


@dataclass(frozen=True)
class SipParams:
    """Round counts: c per message word, d during finalization."""

    c: int = 2
    d: int = 4

    def __post_init__(self):
        if self.c < 1 or self.d < 1:
            raise ValueError("round counts must be positive")


SIPHASH_24 = SipParams(2, 4)
SIPHASH_13 = SipParams(1, 3)


def sip_round(state: Tuple[int, int, int, int]) -> Tuple[int, int, int, int]:
    """One SipRound (S/sip.py:73-86) on the GPU engine (lh::sip_round)."""
    from . import engine
    import numpy as np

    if len(state) != 4:
        raise ValueError("state is four 64-bit words")
    st = np.array([[x & _MASK64 for x in state]], dtype=np.uint64)
    return tuple(int(x) for x in engine.sip_round_states(st, 1)[0])


def deinterleave(message: bytes) -> Tuple[bytes, bytes, bytes, bytes]:
    """SipTreeHash's lane split (S/sip.py:111-121): zero-pad to a multiple
    of 32 bytes (empty stays empty); lane j gets words 4i + j.  A byte-layout
    helper: the engine reads lanes straight from the message (lh::SipTree)."""
    message = bytes(message)
    if message and len(message) % 32:
        message += bytes(32 - len(message) % 32)
    lanes = [bytearray(), bytearray(), bytearray(), bytearray()]
    for i in range(0, len(message), 8):
        lanes[(i // 8) % 4] += message[i:i + 8]
    return tuple(bytes(x) for x in lanes)


def siphash(key, message: bytes, params: SipParams = SIPHASH_24) -> int:
    """SipHash-c-d 64-bit digest (S/sip.py:89-108) on the GPU."""
    from . import engine

    return engine.sip_one(as_key128(key), message, params.c, params.d, tree=False)


def siptreehash(key, message: bytes, params: SipParams = SIPHASH_24) -> int:
    """4-lane interleaved tree SipHash (S/sip.py:124-128) on the GPU."""
    from . import engine

    return engine.sip_one(as_key128(key), message, params.c, params.d, tree=True)


class _SipStream:
    def __init__(self, alg, key, params: SipParams):
        from . import engine

        self._engine = engine
        self._sb = engine.StreamBatch(alg, as_key128(key), 1, c=params.c, d=params.d)

    def append(self, chunk: bytes):
        import numpy as np

        if self._sb._finished:
            raise RuntimeError("cannot append after finish")
        raw = bytes(chunk)
        if raw:
            self._sb.append(np.frombuffer(raw, np.uint8).reshape(1, -1))
        return self

    def finish(self) -> int:
        return int(self._engine.to_u64(self._sb.finish()).reshape(-1)[0])


class SipHasher(_SipStream):
    """Incremental SipHash-c-d (S/sip.py:131-169) on the GPU engine."""

    def __init__(self, key, params: SipParams = SIPHASH_24):
        from . import engine

        super().__init__(engine.ALG_SIPHASH, key, params)


class SipTreeHasher(_SipStream):
    """Incremental 4-lane tree hash (S/sip.py:172-203) on the GPU engine."""

    def __init__(self, key, params: SipParams = SIPHASH_24):
        from . import engine

        super().__init__(engine.ALG_SIPTREE, key, params)
