"""ctypes wrapper over oracle/liblh_oracle.so (TEST INFRASTRUCTURE ONLY).

Mirrors the reference's batch oracle recipes:
HighwayHash-64/128/256 per message (S/highway.py:247-254), SipHash-c-d
(S/sip.py:89-108), SipTreeHash (S/sip.py:124-128), PRF = hash64 of LE
counters.  All inputs are numpy arrays; outputs are uint64 numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblh_oracle.so")
_lib = None

ALG_HIGHWAY, ALG_SIPHASH, ALG_SIPTREE = 0, 1, 2
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build() -> str:
    """Compile the oracle with its Makefile (gcc; seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "lh_oracle.c")
        ):
            build()
        l = ctypes.CDLL(_SO)
        vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        l.lh_ref_batch_fixed.argtypes = [i32, vp, vp, u64, u64, i32, i32, vp, i32]
        l.lh_ref_batch_ragged.argtypes = [i32, vp, vp, vp, vp, u64, i32, i32, vp, i32]
        l.lh_ref_prf64.argtypes = [vp, u64, u64, i32, vp, i32]
        l.lh_ref_highway.argtypes = [vp, vp, u64, i32, vp]
        l.lh_ref_siphash.argtypes = [vp, vp, u64, i32, i32]
        l.lh_ref_siphash.restype = u64
        l.lh_ref_siptree.argtypes = [vp, vp, u64, i32, i32]
        l.lh_ref_siptree.restype = u64
        l.lh_ref_sip_round.argtypes = [vp]
        l.lh_ref_zipper_bytes.argtypes = [u64, u64, vp, vp]
        l.lh_ref_hh_update.argtypes = [vp, vp]
        l.lh_ref_hh_update_inverse.argtypes = [vp, vp]
        l.lh_ref_hh_update_remainder.argtypes = [vp, vp, ctypes.c_uint]
        l.lh_ref_hh_finalize.argtypes = [vp, i32, vp]
        l.lh_ref_update_states.argtypes = [vp, vp, u64, i32]
        l.lh_ref_hh_init.argtypes = [vp, vp]
        l.lh_ref_hh_remainder_packet.argtypes = [vp, ctypes.c_uint, vp]
        l.lh_ref_avalanche_counts.argtypes = [i32, vp, vp, u64, ctypes.c_uint32, i32, i32, vp, i32]
        l.lh_ref_synth_fill.argtypes = [vp, u64, u64, u64, u64, i32]
        _lib = l
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _key(key, n) -> np.ndarray:
    k = np.zeros(4, np.uint64)
    k[:n] = np.asarray(key, dtype=np.uint64)[:n]
    return k


def _threads(nthreads):
    if nthreads is None or nthreads <= 0:
        return len(os.sched_getaffinity(0))
    return nthreads


def highway(key, msg: bytes, rounds: int = 4):
    """4 lane sums (HighwayHash-256); [0] is HighwayHash-64."""
    k = _key(key, 4)
    m = np.frombuffer(bytes(msg), np.uint8) if len(msg) else np.zeros(1, np.uint8)
    out = np.zeros(4, np.uint64)
    lib().lh_ref_highway(_ptr(k), _ptr(m), len(msg), rounds, _ptr(out))
    return tuple(int(x) for x in out)


def siphash(key, msg: bytes, c: int = 2, d: int = 4) -> int:
    k = _key(key, 2)
    m = np.frombuffer(bytes(msg), np.uint8) if len(msg) else np.zeros(1, np.uint8)
    return int(lib().lh_ref_siphash(_ptr(k), _ptr(m), len(msg), c, d))


def siptree(key, msg: bytes, c: int = 2, d: int = 4) -> int:
    k = _key(key, 2)
    m = np.frombuffer(bytes(msg), np.uint8) if len(msg) else np.zeros(1, np.uint8)
    return int(lib().lh_ref_siptree(_ptr(k), _ptr(m), len(msg), c, d))


def batch_fixed(alg, key, msgs: np.ndarray, p1: int, p2: int, nthreads=None):
    """msgs: (n, L) uint8 C-contiguous.  HH: p1=width, p2=rounds; Sip: c, d."""
    msgs = np.ascontiguousarray(msgs, dtype=np.uint8)
    n, L = msgs.shape
    w = p1 // 64 if alg == ALG_HIGHWAY else 1
    out = np.zeros(n * w, np.uint64)
    k = _key(key, 4 if alg == ALG_HIGHWAY else 2)
    buf = msgs if msgs.size else np.zeros(1, np.uint8)
    lib().lh_ref_batch_fixed(alg, _ptr(k), _ptr(buf), n, L, p1, p2, _ptr(out), _threads(nthreads))
    return out.reshape(n, w) if w > 1 else out


def batch_ragged(alg, key, buf: np.ndarray, offsets: np.ndarray, lengths=None,
                 p1: int = 64, p2: int = 4, nthreads=None):
    """offsets: uint64 (n+1 if lengths is None else n); lengths: uint32 or None."""
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = len(offsets) - 1 if lengths is None else len(offsets)
    if lengths is not None:
        lengths = np.ascontiguousarray(lengths, dtype=np.uint32)
    w = p1 // 64 if alg == ALG_HIGHWAY else 1
    out = np.zeros(max(n, 1) * w, np.uint64)
    k = _key(key, 4 if alg == ALG_HIGHWAY else 2)
    b = buf if buf.size else np.zeros(1, np.uint8)
    lib().lh_ref_batch_ragged(alg, _ptr(k), _ptr(b), _ptr(offsets),
                              _ptr(lengths) if lengths is not None else None,
                              n, p1, p2, _ptr(out), _threads(nthreads))
    out = out[: n * w]
    return out.reshape(n, w) if w > 1 else out


def update_states(states: np.ndarray, packets: np.ndarray, inverse: bool = False) -> np.ndarray:
    """S/highway.py:130-173 on n raw states: (n,16) uint64 (v0, v1, mul0,
    mul1 lanes) and (n,4) uint64 packets; returns the new states."""
    st = np.array(states, dtype=np.uint64, order="C", copy=True).reshape(-1, 16)
    pk = np.ascontiguousarray(packets, dtype=np.uint64).reshape(-1, 4)
    if len(st) != len(pk):
        raise ValueError("states and packets differ in length")
    if len(st):
        lib().lh_ref_update_states(_ptr(st), _ptr(pk), len(st), int(bool(inverse)))
    return st


def prf64(key, start: int, n: int, rounds: int = 4, nthreads=None) -> np.ndarray:
    out = np.zeros(max(n, 1), np.uint64)
    k = _key(key, 4)
    lib().lh_ref_prf64(_ptr(k), start, n, rounds, _ptr(out), _threads(nthreads))
    return out[:n]


def avalanche_counts(alg, key, msgs: np.ndarray, p1: int, p2: int, nthreads=None) -> np.ndarray:
    """S/_kernels.py:247-265 restated: (8*size, 64) int64 flip tallies."""
    msgs = np.ascontiguousarray(msgs, dtype=np.uint8)
    iters, size = msgs.shape
    k = _key(key, 4 if alg == ALG_HIGHWAY else 2)
    out = np.zeros((8 * size, 64), np.int64)
    buf = msgs if msgs.size else np.zeros(1, np.uint8)
    rc = lib().lh_ref_avalanche_counts(alg, _ptr(k), _ptr(buf), iters, size, p1, p2, _ptr(out),
                                       _threads(nthreads))
    if rc:
        raise ValueError("size too large")
    return out


def synth_fill(nbytes: int, seed: int, word_offset: int = 0, stream: int = 0,
               nthreads=None, out: np.ndarray = None) -> np.ndarray:
    """Host twin of the engine's counter generator (synth.counter_bytes), on
    all host threads: the reference leg's input, no GPU involved."""
    buf = np.empty(max(nbytes, 1), np.uint8) if out is None else out
    if nbytes:
        lib().lh_ref_synth_fill(_ptr(buf), nbytes, seed, stream, word_offset, _threads(nthreads))
    return buf[:nbytes]
