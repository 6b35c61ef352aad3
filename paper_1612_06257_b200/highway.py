"""HighwayHash types and one-shot API, computed on the B200 engine.

Mirrors the reference module ``lanehash.highway`` (S/highway.py): the same
``Key256`` type, constants, digest byte images and ``hash64`` / ``hash256``
signatures (S/highway.py:43-70, 20-38, 247-254, 288-295), plus ``hash128``
(lanes 0-1 of the 256-bit lane sum; the reference defines no 128-bit width,
S/highway.py:228-229 — derived).  Every digest is computed by
the CUDA library; there is no Python arithmetic path.
"""
from __future__ import annotations

import struct
from typing import Iterable, Sequence, Tuple

_MASK64 = 0xFFFFFFFFFFFFFFFF

#: S/highway.py:20-31 (lane 0 first).  The engine carries its own copy in
#: csrc/lh_engine.cu; tests/test_host.py checks both against the reference.
INIT0: Tuple[int, int, int, int] = (
    0xDBE6D5D5FE4CCE2F,
    0xA4093822299F31D0,
    0x13198A2E03707344,
    0x243F6A8885A308D3,
)
INIT1: Tuple[int, int, int, int] = (
    0x3BD39E10CB0EF593,
    0xC0ACF169B5F18A8C,
    0xBE5466CF34E90C6C,
    0x452821E638D01377,
)
#: S/highway.py:35-38; realised on the GPU as 5 PRMT per lane pair
#: (csrc/lh_device.cuh: zipper).
ZIPPER_OFFSETS: Tuple[int, ...] = (
    0x3, 0xC, 0x2, 0x5, 0xE, 0x1, 0xF, 0x0,
    0xB, 0x4, 0xA, 0xD, 0x9, 0x6, 0x8, 0x7,
)

WIDTHS = (64, 128, 256)


class Key256:
    """256-bit key held as four 64-bit little-endian lanes (S/highway.py:43-70)."""

    __slots__ = ("lanes",)

    def __init__(self, lanes: Sequence[int]):
        if len(lanes) != 4:
            raise ValueError("Key256 requires exactly 4 lanes")
        self.lanes = tuple(int(lane) & _MASK64 for lane in lanes)

    @classmethod
    def from_bytes(cls, raw: bytes) -> "Key256":
        if len(raw) != 32:
            raise ValueError("Key256 requires exactly 32 bytes")
        return cls(struct.unpack("<4Q", raw))

    @classmethod
    def from_hex(cls, text: str) -> "Key256":
        return cls.from_bytes(bytes.fromhex(text))

    def to_bytes(self) -> bytes:
        return struct.pack("<4Q", *self.lanes)

    def __eq__(self, other: object) -> bool:
        return isinstance(other, Key256) and self.lanes == other.lanes

    def __hash__(self) -> int:
        return hash(self.lanes)

    def __repr__(self) -> str:
        return f"Key256({self.to_bytes().hex()})"


def as_key256(key) -> Key256:
    """Accept a Key256, 32 raw bytes, or 4 integer lanes (numpy array ok)."""
    if isinstance(key, Key256):
        return key
    if isinstance(key, (bytes, bytearray, memoryview)):
        return Key256.from_bytes(bytes(key))
    return Key256([int(x) for x in key])


def _check_width(width: int) -> None:
    if width not in WIDTHS:
        raise ValueError("width must be 64, 128 or 256")


def hash64(key, message: bytes, rounds: int = 4) -> int:
    """One-shot 64-bit HighwayHash (S/highway.py:247-249) on the GPU."""
    from . import engine

    return int(engine.hash_one(as_key256(key), message, 64, rounds)[0])


def hash128(key, message: bytes, rounds: int = 4) -> Tuple[int, int]:
    """One-shot 128-bit HighwayHash: lanes 0-1 of the 256-bit lane sum."""
    from . import engine

    out = engine.hash_one(as_key256(key), message, 128, rounds)
    return (int(out[0]), int(out[1]))


def hash256(key, message: bytes, rounds: int = 4) -> Tuple[int, int, int, int]:
    """One-shot 256-bit HighwayHash as four lanes (S/highway.py:252-254)."""
    from . import engine

    out = engine.hash_one(as_key256(key), message, 256, rounds)
    return tuple(int(x) for x in out)


#: (v0, v1, mul0, mul1), four lanes each (S/highway.py:40).
State = Tuple[Tuple[int, int, int, int], ...]


def _rot32(x: int) -> int:
    return ((x >> 32) | (x << 32)) & _MASK64


def initialize(key) -> State:
    """Key expansion (S/highway.py:122-127): v0 = k ^ INIT0,
    v1 = rot32(k) ^ INIT1, mul0 = INIT0, mul1 = INIT1.  Key-only, so it is
    host logic (the engine expands the key once per batch, lh_host.cuh)."""
    k = as_key256(key).lanes
    return (tuple(k[i] ^ INIT0[i] for i in range(4)),
            tuple(_rot32(k[i]) ^ INIT1[i] for i in range(4)), INIT0, INIT1)


def _state_op(state: State, packet: Sequence[int], inverse: bool) -> State:
    from . import engine
    import numpy as np

    if len(packet) != 4:
        raise ValueError("packet is four 64-bit lanes")
    pk = np.array([[x & _MASK64 for x in packet]], dtype=np.uint64)
    return _unflat(engine.update_states(_flat(state), pk, inverse)[0])


def update(state: State, packet: Sequence[int]) -> State:
    """One Update step (S/highway.py:130-150) on the GPU engine."""
    return _state_op(state, packet, False)


def update_inverse(state: State, packet: Sequence[int]) -> State:
    """Exact inverse of :func:`update` (S/highway.py:153-173) on the GPU."""
    return _state_op(state, packet, True)


def _flat(state: State):
    import numpy as np

    if len(state) != 4 or any(len(x) != 4 for x in state):
        raise ValueError("state is four 4-lane tuples")
    return np.array([[x & _MASK64 for lanes in state for x in lanes]], dtype=np.uint64)


def _unflat(row) -> State:
    out = [int(x) for x in row]
    return tuple(tuple(out[i:i + 4]) for i in range(0, 16, 4))


def update_remainder(state: State, tail: bytes) -> State:
    """Absorb the final 1..31 bytes plus the length injection
    (S/highway.py:182-199), on the GPU engine (lh::Highway::remainder)."""
    from . import engine
    import numpy as np

    tail = bytes(tail)
    if not 1 <= len(tail) <= 31:
        raise ValueError("remainder length must be in 1..31")
    t = np.zeros((1, 32), np.uint8)
    t[0, :len(tail)] = np.frombuffer(tail, np.uint8)
    return _unflat(engine.remainder_states(_flat(state), t, [len(tail)])[0])


def finalize(state: State, width: int = 64, rounds: int = 4):
    """`rounds` PermuteAndUpdates and the lane sums (S/highway.py:223-234),
    on the GPU engine: an int for width 64, a tuple of width/64 lanes
    otherwise (128 is this library's derived width)."""
    from . import engine

    _check_width(width)
    out = engine.finalize_states(_flat(state), width, rounds)
    return int(out[0]) if width == 64 else tuple(int(x) for x in out[0])


# Byte-layout helpers of the reference module.  They only rearrange bytes
# and never feed the engine, which builds packets in registers
# (lh_device.cuh); they exist so code written against lanehash.highway runs.

def packet_lanes(packet: bytes) -> Tuple[int, int, int, int]:
    """32 bytes as four little-endian 64-bit lanes (S/highway.py:115-119)."""
    if len(packet) != 32:
        raise ValueError("packet must be exactly 32 bytes")
    return struct.unpack("<4Q", bytes(packet))


def remainder_packet(tail: bytes) -> bytes:
    """The 32-byte packet of a 1..31 byte remainder (S/highway.py:206-220):
    whole 4-byte groups first, the 0..3 leftover bytes at bytes 28..31."""
    r = len(tail)
    if not 1 <= r <= 31:
        raise ValueError("remainder length must be in 1..31")
    whole = r & ~3
    packet = bytearray(32)
    packet[:whole] = bytes(tail[:whole])
    packet[28:28 + r - whole] = bytes(tail[whole:])
    return bytes(packet)


def permute_lanes(v: Sequence[int]) -> Tuple[int, int, int, int]:
    """PermuteAndUpdate's packet (S/highway.py:176-179)."""
    a, b, c, d = v
    return (_rot32(c), _rot32(d), _rot32(a), _rot32(b))


def zipper_merge(half: bytes) -> bytes:
    """ZIPPER_OFFSETS applied to one 16-byte lane pair (S/highway.py:73-77)."""
    if len(half) != 16:
        raise ValueError("zipper_merge operates on exactly 16 bytes")
    return bytes(half[off] for off in ZIPPER_OFFSETS)


def mul32(a: int, b: int) -> int:
    """Low 32 bits of a times low 32 bits of b (S/highway.py:80-82)."""
    return ((a & 0xFFFFFFFF) * (b & 0xFFFFFFFF)) & _MASK64


class StreamingHasher:
    """Incremental HighwayHash (S/highway.py:257-285) on the GPU engine.

    Same contract as the reference: only len mod 32 affects padding; append
    after finish and a second finish raise RuntimeError.  Each append ships
    the chunk to the device and advances the state there (engine.StreamBatch
    with n = 1): nothing but the device record (state, <= 31 pending bytes,
    length) is retained.  Use engine.StreamBatch to stream many messages."""

    def __init__(self, key, rounds: int = 4):
        from . import engine

        self._engine = engine
        self._sb = engine.StreamBatch(engine.ALG_HIGHWAY, as_key256(key), 1, 256, rounds)

    def append(self, chunk: bytes) -> "StreamingHasher":
        import numpy as np

        if self._sb._finished:
            raise RuntimeError("cannot append after finish")
        raw = bytes(chunk)
        if raw:
            self._sb.append(np.frombuffer(raw, np.uint8).reshape(1, -1))
        return self

    def finish(self, width: int = 64):
        _check_width(width)
        out = [int(x) for x in self._engine.to_u64(self._sb.finish(width)).reshape(-1)]
        return out[0] if width == 64 else tuple(out)


def digest64_to_bytes(digest: int) -> bytes:
    """Little-endian byte image of a 64-bit digest (S/highway.py:288-290)."""
    return struct.pack("<Q", digest & _MASK64)


def digest128_to_bytes(digest: Iterable[int]) -> bytes:
    return struct.pack("<2Q", *(lane & _MASK64 for lane in digest))


def digest256_to_bytes(digest: Iterable[int]) -> bytes:
    """Lane 0 first, each lane little-endian (S/highway.py:293-295)."""
    return struct.pack("<4Q", *(lane & _MASK64 for lane in digest))
