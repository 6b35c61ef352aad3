"""Same-signature stand-ins for the reference's numba batch entry points.

``lanehash._kernels`` (S/_kernels.py) is the reference's fast path: jit
functions over uint8 arrays with the key as a 4-lane uint64 array.  Callers
of it port by changing the import; every function here is one launch of the
engine's CUDA kernels (csrc/lh_engine.cu, csrc/lh_quality.cu):

  highway64(keylanes, msg, rounds)          S/_kernels.py:150-154
  highway256(keylanes, msg, rounds)         S/_kernels.py:157-166
  siphash(keylanes, msg, c, d)              S/_kernels.py:210-213
  siptreehash(keylanes, msg, c, d)          S/_kernels.py:216-234
  avalanche_counts(algo, keylanes, msgs, p1, p2)   S/_kernels.py:247-265
  hash_batch(algo, keylanes, msgs, p1, p2)  S/_kernels.py:268-274

``algo`` follows S/_kernels.py:237-244: 0 = HighwayHash-64 with p1 =
finalization rounds (p2 ignored), 1 = SipHash-p1-p2, 2 = SipTreeHash-p1-p2.
numpy in -> numpy uint64 out, as the reference; ``hash_batch`` also takes a
(n, L) uint8 CUDA tensor and then returns the int64 CUDA tensor of digests
without leaving the device.
"""
from __future__ import annotations

import numpy as np

from . import engine

_ALGOS = {0: engine.ALG_HIGHWAY, 1: engine.ALG_SIPHASH, 2: engine.ALG_SIPTREE}


def _algo(algo: int) -> int:
    try:
        return _ALGOS[int(algo)]
    except (KeyError, TypeError, ValueError):
        raise ValueError(f"unknown kernel algo id {algo!r} (0, 1 or 2)") from None


def _lanes(keylanes, n: int) -> np.ndarray:
    k = np.asarray(keylanes, dtype=np.uint64).reshape(-1)
    if k.size < n:
        raise ValueError(f"need at least {n} key lanes")
    return k[:n].copy()


def _row(msg) -> np.ndarray:
    return np.ascontiguousarray(msg, dtype=np.uint8).reshape(1, -1)


def hash_batch(algo, keylanes, msgs, p1, p2):
    """Hash every row of a (n, size) uint8 batch; returns (n,) uint64."""
    alg = _algo(algo)
    if alg == engine.ALG_HIGHWAY:
        return engine.highway_batch(_lanes(keylanes, 4), msgs, 64, int(p1))
    return engine.sip_batch(_lanes(keylanes, 2), msgs, int(p1), int(p2),
                            tree=alg == engine.ALG_SIPTREE)


def highway64(keylanes, msg, rounds) -> np.uint64:
    return np.uint64(hash_batch(0, keylanes, _row(msg), rounds, 0)[0])


def highway256(keylanes, msg, rounds):
    d = engine.highway_batch(_lanes(keylanes, 4), _row(msg), 256, int(rounds))
    return tuple(np.uint64(x) for x in np.asarray(d).reshape(-1))


def siphash(keylanes, msg, c, d) -> np.uint64:
    return np.uint64(hash_batch(1, keylanes, _row(msg), c, d)[0])


def siptreehash(keylanes, msg, c, d) -> np.uint64:
    return np.uint64(hash_batch(2, keylanes, _row(msg), c, d)[0])


def avalanche_counts(algo, keylanes, msgs, p1, p2) -> np.ndarray:
    """(8*size, 64) int64 flip tallies (csrc/lh_quality.cu).  Unlike the
    reference the message array is never modified (no in-place flips)."""
    from .quality import avalanche_counts as _counts

    lanes = np.zeros(4, np.uint64)
    k = np.asarray(keylanes, dtype=np.uint64).reshape(-1)[:4]
    lanes[: k.size] = k
    return _counts(_algo(algo), lanes, msgs, int(p1), int(p2))
