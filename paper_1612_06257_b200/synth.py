"""Seeded synthetic inputs (bench / test harness, not a reference interface).

The reference benchmarks on synthetic random bytes (BASELINE.json configs,
SURVEY.md §8d); there is no dataset.  Two generators are frozen here:

* ``numpy_bytes(seed, shape)`` — ``np.random.default_rng(seed).integers(0,
  256, shape, uint8)``: cfg1 (4,096 x 1 KiB, seed 1) and the key
  (``default_rng(0)``, 4 x u64), exactly as SURVEY.md §8d records them.
* a counter-based generator with twin CUDA (csrc/lh_synth.cu) and numpy
  (below) implementations, used for the large configs so that multi-GiB
  batches are generated in HBM at memory speed and every GPU shard of a
  global batch is reproducible from (seed, word index):

      word(seed, stream, w) = mix64(k + (w + 1) * G)
      k = mix64(seed * G + stream + 1),  G = 0x9E3779B97F4A7C15 (mod 2^64)
      mix64 = SplitMix64 finalizer
      byte b of a buffer = byte (b & 7) of word(b >> 3), little-endian

tests/test_synth.py cross-checks the two implementations.
"""
from __future__ import annotations

import numpy as np

G = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1

KEY_SEED = 0


def key256() -> np.ndarray:
    """The frozen HighwayHash key: default_rng(0) -> 4 u64 lanes."""
    return np.random.default_rng(KEY_SEED).integers(0, 2**64, size=4, dtype=np.uint64)


def key128() -> np.ndarray:
    """The frozen SipHash key: the first two lanes of key256()."""
    return key256()[:2].copy()


def numpy_bytes(seed: int, shape) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, 256, shape, dtype=np.uint8)


def _mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def _mix64_int(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int = 0) -> int:
    return _mix64_int((seed * G + stream + 1) & _M64)


def words(seed: int, first: int, count: int, stream: int = 0) -> np.ndarray:
    """word(seed, stream, first .. first+count-1) as uint64."""
    k = np.uint64(stream_key(seed, stream))
    w = np.arange(first + 1, first + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = k + w * np.uint64(G)
    return _mix64_np(z)


def counter_bytes(seed: int, nbytes: int, word_offset: int = 0, stream: int = 0) -> np.ndarray:
    """numpy twin of lh_synth_fill."""
    nw = (nbytes + 7) // 8
    return words(seed, word_offset, nw, stream).view(np.uint8)[:nbytes].copy()


def lengths(seed: int, n: int, lo: int, hi: int, first: int = 0) -> np.ndarray:
    """numpy twin of lh_synth_lengths: lo + hi32(word) * (hi-lo+1) >> 32."""
    v = words(seed, first, n, 0) >> np.uint64(32)
    span = np.uint64(hi - lo + 1)
    return (np.uint64(lo) + ((v * span) >> np.uint64(32))).astype(np.uint32)


# ---------------------------------------------------------------------------
# Device-side generation (CUDA, via the engine library)
# ---------------------------------------------------------------------------

def fill_device(t, seed: int, word_offset: int = 0, stream: int = 0) -> None:
    """Fill a CUDA uint8 tensor with the counter stream (lh_synth_fill)."""
    import torch

    from . import _lib

    assert t.is_cuda and t.dtype == torch.uint8
    st = torch.cuda.current_stream(t.device).cuda_stream
    _lib.check(_lib.lib().lh_synth_fill(t.data_ptr(), t.numel(), seed, stream, word_offset, st),
               "lh_synth_fill")


def lengths_device(t, seed: int, lo: int, hi: int, first: int = 0) -> None:
    import torch

    from . import _lib

    assert t.is_cuda and t.dtype == torch.int32
    st = torch.cuda.current_stream(t.device).cuda_stream
    _lib.check(_lib.lib().lh_synth_lengths(t.data_ptr(), t.numel(), seed, first, lo, hi, st),
               "lh_synth_lengths")


def remainder_sweep_layout(max_len: int = 1024, per_len: int = 64):
    """cfg2 layout: for L = 0..max_len-1 (ascending), `per_len` messages:
    the first half random, then a quarter all-0x00, then a quarter all-0xFF.
    Returns (lengths u32, offsets u64[n+1], kind u8[n]: 0 random/1 zero/2 ff)."""
    lens = np.repeat(np.arange(max_len, dtype=np.uint32), per_len)
    kind = np.tile(
        np.concatenate([
            np.zeros(per_len // 2, np.uint8),
            np.ones(per_len // 4, np.uint8),
            np.full(per_len - per_len // 2 - per_len // 4, 2, np.uint8),
        ]),
        max_len,
    )
    offsets = np.zeros(len(lens) + 1, np.uint64)
    np.cumsum(lens, out=offsets[1:])
    return lens, offsets, kind


def remainder_sweep_bytes(seed: int = 2, max_len: int = 1024, per_len: int = 64):
    """cfg2 packed buffer: counter bytes (seed 2) with the zero / 0xFF
    messages overwritten.  Returns (buf, offsets u64[n+1], lengths u32)."""
    lens, offsets, kind = remainder_sweep_layout(max_len, per_len)
    total = int(offsets[-1])
    buf = counter_bytes(seed, total)
    starts = offsets[:-1].astype(np.int64)
    for k, val in ((1, 0x00), (2, 0xFF)):
        sel = np.nonzero(kind == k)[0]
        for i in sel:
            s = starts[i]
            buf[s:s + lens[i]] = val
    return buf, offsets, lens
