"""ctypes binding of the in-tree CUDA library ``libb200hash.so``.

The C ABI is declared in ``include/lanehash_b200.h``.  There is no CPU
fallback: if the library cannot be loaded, or no sm_100 device is present,
every hash call raises.
"""
from __future__ import annotations

import ctypes
import os
import re

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(_HERE), "include", "lanehash_b200.h")

LH_OK = 0
LH_EINVAL = -1
LH_EALIGN = -2
LH_ECUDA = -3
LH_ENODEV = -4
LH_ETOOBIG = -5

KERNEL_AUTO = 0
KERNEL_DIRECT = 1
KERNEL_TMA = 2
KERNEL_SPLIT = 3
KERNEL_STAGED = 4
KERNEL_RING = 5

ALG_HIGHWAY = 0
ALG_SIPHASH = 1
ALG_SIPTREE = 2

_lib = None


class EngineError(RuntimeError):
    """A CUDA-side failure reported by the engine (LH_ECUDA / LH_ENODEV)."""


def _declare(l):
    vp, u64, i32, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32
    l.lh_version.restype = ctypes.c_char_p
    l.lh_version.argtypes = []
    l.lh_strerror.restype = ctypes.c_char_p
    l.lh_strerror.argtypes = [i32]
    l.lh_highway_fixed.argtypes = [vp, u64, u64, vp, i32, i32, vp, vp]
    l.lh_highway_fixed_kernel.argtypes = [vp, u64, u64, vp, i32, i32, vp, vp, i32]
    l.lh_highway_ragged.argtypes = [vp, vp, vp, u64, vp, i32, i32, vp, vp]
    l.lh_highway_ragged_kernel.argtypes = [vp, vp, vp, u64, vp, i32, i32, vp, vp, i32]
    l.lh_siphash_fixed.argtypes = [vp, u64, u64, vp, i32, i32, i32, vp, vp]
    l.lh_siphash_fixed_kernel.argtypes = [vp, u64, u64, vp, i32, i32, i32, vp, vp, i32]
    l.lh_siphash_ragged.argtypes = [vp, vp, vp, u64, vp, i32, i32, i32, vp, vp]
    l.lh_siphash_ragged_kernel.argtypes = [vp, vp, vp, u64, vp, i32, i32, i32, vp, vp, i32]
    l.lh_highway_prf64.argtypes = [u64, u64, vp, i32, vp, vp]
    l.lh_stream_state_bytes.argtypes = [i32]
    l.lh_stream_state_bytes.restype = ctypes.c_size_t
    l.lh_stream_init.argtypes = [i32, vp, u64, vp, i32, i32, vp]
    l.lh_stream_update.argtypes = [i32, vp, u64, vp, vp, vp, u64, vp]
    l.lh_stream_finish.argtypes = [i32, vp, u64, vp, i32, vp]
    l.lh_avalanche_counts.argtypes = [i32, vp, vp, u64, ctypes.c_uint32, i32, i32, vp, vp]
    l.lh_synth_fill.argtypes = [vp, u64, u64, u64, u64, vp]
    l.lh_synth_lengths.argtypes = [vp, u64, u64, u64, u32, u32, vp]
    l.lh_highway_update_states.argtypes = [vp, vp, u64, i32, vp]
    l.lh_highway_bijectivity.argtypes = [u64, u64, vp, vp]
    l.lh_highway_remainder_states.argtypes = [vp, vp, vp, u64, vp]
    l.lh_highway_finalize_states.argtypes = [vp, u64, i32, i32, vp, vp]
    l.lh_sip_round_states.argtypes = [vp, u64, i32, vp]
    l.lh_ragged_plan.argtypes = [vp, vp, u64, u64, u64, vp, vp, vp, vp]
    l.lh_read_probe.argtypes = [vp, u64, vp, vp]
    l.lh_ragged_plan_stats.argtypes = [vp, vp, u64, u64, u64, vp, vp, vp, vp, u32, u32, vp]
    l.lh_ragged_order.argtypes = [vp, vp, u64, u32, vp, vp, vp]
    l.lh_highway_ragged_ordered.argtypes = [vp, vp, vp, u64, vp, vp, i32, i32, vp, vp]
    l.lh_siphash_ragged_ordered.argtypes = [vp, vp, vp, u64, vp, vp, i32, i32, i32, vp, vp]
    for name in (
        "lh_highway_fixed", "lh_highway_fixed_kernel", "lh_highway_ragged",
        "lh_highway_ragged_kernel", "lh_siphash_fixed", "lh_siphash_fixed_kernel",
        "lh_siphash_ragged", "lh_siphash_ragged_kernel",
        "lh_highway_prf64", "lh_synth_fill", "lh_synth_lengths",
        "lh_stream_init", "lh_stream_update", "lh_stream_finish", "lh_avalanche_counts",
        "lh_highway_update_states", "lh_highway_bijectivity",
        "lh_highway_remainder_states", "lh_highway_finalize_states", "lh_sip_round_states",
        "lh_ragged_plan", "lh_read_probe", "lh_ragged_plan_stats", "lh_ragged_order",
        "lh_highway_ragged_ordered", "lh_siphash_ragged_ordered",
    ):
        getattr(l, name).restype = i32


def lib(build_if_missing: bool = True):
    """Load (building first if the .so is missing) the engine library."""
    global _lib
    if _lib is None:
        path = os.environ.get("LH_LIBRARY")  # A/B tuning runs load an alternate build
        if not path:
            path = _build.SO
            if not os.path.exists(path):
                if not build_if_missing:
                    raise EngineError(f"engine library not built: {path}")
                _build.build()
        l = ctypes.CDLL(path)
        _declare(l)
        _lib = l
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map an LH_* status to the reference's exception types."""
    if rc == LH_OK:
        return
    msg = lib().lh_strerror(rc).decode()
    if what:
        msg = f"{what}: {msg}"
    if rc in (LH_EINVAL, LH_EALIGN, LH_ETOOBIG):
        raise ValueError(msg)
    raise EngineError(msg)


def version() -> str:
    return lib().lh_version().decode()


def declared_symbols() -> list:
    """Function names declared in include/lanehash_b200.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(lh_\w+)\s*\(", text, re.M)))
