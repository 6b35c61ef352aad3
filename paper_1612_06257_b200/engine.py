"""Batch API of the B200 engine (the hot path behind the reference interface).

All functions take either CUDA tensors (zero-copy: the call is a single
asynchronous kernel launch on the current stream; results stay in HBM) or
host arrays (numpy / CPU torch tensors; the call streams the batch through
the GPU in chunks — H2D, kernel and D2H overlapped on two CUDA streams —
and returns host numpy ``uint64`` digests).

Digests are 64-bit words stored in ``torch.int64`` tensors on the device
(bit-identical to uint64; ``to_u64`` converts to numpy ``uint64``).  Layout:
width 64 -> shape (n,), 128 -> (n, 2), 256 -> (n, 4), lane 0 first.

Reference correspondence (S = /root/reference/pkg/src/lanehash):
  highway_batch  <- NumpyBackend.hash64_batch (S/backends.py:52-53,
                    S/_highway_np.py:116-130), _kernels.hash_batch algo 0
                    (S/_kernels.py:268-274), widths 64/128/256
  highway_ragged <- per-message hash64/hash256 over unequal lengths
  sip_batch      <- _kernels.hash_batch algo 1/2 (S/_kernels.py:237-244),
                    sip.siphash / sip.siptreehash (S/sip.py:89-128)
  prf64          <- hash64(key, le64(ctr)) (S/highway.py:247-249)
"""
from __future__ import annotations

import ctypes
import warnings
from typing import Optional

import numpy as np
import torch

from . import _lib
from .highway import Key256, _check_width
from .highway import as_key256 as _as_key256
from .sip import Key128
from .sip import as_key128 as _as_key128

KERNEL_AUTO = _lib.KERNEL_AUTO
KERNEL_DIRECT = _lib.KERNEL_DIRECT
KERNEL_TMA = _lib.KERNEL_TMA
KERNEL_SPLIT = _lib.KERNEL_SPLIT
KERNEL_STAGED = _lib.KERNEL_STAGED
KERNEL_RING = _lib.KERNEL_RING

#: Host-path chunk size (bytes of message payload per H2D copy).
HOST_CHUNK_BYTES = 128 << 20
# Ragged batches whose mean message length (buffer bytes / messages) reaches
# this use the register-ring kernel (KERNEL_RING): several packets in flight
# per thread; shorter ones the warp-staged short-key kernel.
RING_MIN_MEAN_BYTES = 128
# Sip-family ragged batches below this mean length use the warp-staged kernel
# (cfg3-shaped SipHash-1-3 2.10 -> 1.70 ms); at a 128-B mean it loses to the ring.
SIP_STAGED_MAX_MEAN_BYTES = 64


# Per-call host work matters for small, launch-bound batches (cfg1: a 3.5 us
# kernel): device objects, the raw stream handle and the ctypes key arrays
# are cached; the device context is only switched when it differs.
_DEVICES: dict = {}
_CUDA_CHECKED = False
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _require_cuda() -> torch.device:
    global _CUDA_CHECKED
    if not _CUDA_CHECKED:
        if not torch.cuda.is_available():
            raise _lib.EngineError("no CUDA device: the B200 engine has no CPU fallback")
        _CUDA_CHECKED = True
    i = torch.cuda.current_device()
    d = _DEVICES.get(i)
    if d is None:
        d = _DEVICES[i] = torch.device("cuda", i)
    return d


def _stream_ptr(device) -> int:
    if _raw_stream is not None:
        return _raw_stream(device.index if device.index is not None else
                           torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


_KEYS: dict = {}
_KEY_OBJS: dict = {}


def _cached_key(key, conv):
    """Key256/Key128 of a key given as a numpy array or raw bytes, memoised on
    its bytes (the conversion and validation cost more than a small launch)."""
    if isinstance(key, (Key256, Key128)):
        return conv(key)
    if isinstance(key, np.ndarray):
        tag = (conv, key.dtype.str, key.tobytes())
    elif isinstance(key, (bytes, bytearray)):
        tag = (conv, bytes(key))
    else:
        return conv(key)
    k = _KEY_OBJS.get(tag)
    if k is None:
        if len(_KEY_OBJS) > 256:
            _KEY_OBJS.clear()
        k = _KEY_OBJS[tag] = conv(key)
    return k


def as_key256(key) -> Key256:
    return _cached_key(key, _as_key256)


def as_key128(key) -> Key128:
    return _cached_key(key, _as_key128)


def _key_array(lanes: tuple):
    a = _KEYS.get(lanes)
    if a is None:
        if len(_KEYS) > 256:
            _KEYS.clear()
        a = _KEYS[lanes] = (ctypes.c_uint64 * len(lanes))(*lanes)
    return a


def _key4(key: Key256):
    return _key_array(key.lanes)


def _key2(key: Key128):
    return _key_array((key.k0, key.k1))


class _on_device:
    """torch.cuda.device(d) only when d is not already current."""

    __slots__ = ("ctx",)

    def __init__(self, device):
        self.ctx = None if device.index == torch.cuda.current_device() else \
            torch.cuda.device(device)

    def __enter__(self):
        if self.ctx is not None:
            self.ctx.__enter__()

    def __exit__(self, *exc):
        if self.ctx is not None:
            return self.ctx.__exit__(*exc)
        return False


def to_u64(t) -> np.ndarray:
    """Digest tensor/array -> numpy uint64 (bit-preserving)."""
    if isinstance(t, torch.Tensor):
        t = t.detach().cpu().numpy()
    return np.asarray(t).view(np.uint64)


def _host_view(a: np.ndarray) -> torch.Tensor:
    """Zero-copy torch view of a host array the engine only reads.  Read-only
    arrays (np.frombuffer(bytes), read-only np.memmap) are fine: torch warns
    that writes through the view would be undefined, and there are none."""
    a = np.ascontiguousarray(a)
    if a.flags.writeable:
        return torch.from_numpy(a)
    with warnings.catch_warnings():
        warnings.filterwarnings("ignore", message=".*not writable.*", category=UserWarning)
        return torch.from_numpy(a)


def _as_u8_2d(msgs):
    if isinstance(msgs, torch.Tensor):
        if msgs.dtype != torch.uint8 or msgs.dim() != 2:
            raise ValueError("messages must be a 2-D uint8 tensor (n, length)")
        return msgs
    a = np.asarray(msgs)
    if a.dtype != np.uint8 or a.ndim != 2:
        raise ValueError("messages must be a 2-D uint8 array (n, length)")
    return _host_view(a)


def _out_shape(n: int, lanes: int):
    return (n,) if lanes == 1 else (n, lanes)


_PEER_OK: dict = {}


def _peer_ok(device, other) -> bool:
    """Can kernels on `device` store to memory on `other` (NVLink / P2P)?"""
    key = (device.index, other.index)
    v = _PEER_OK.get(key)
    if v is None:
        v = _PEER_OK[key] = bool(torch.cuda.can_device_access_peer(device.index, other.index))
    return v


def _check_out(out: torch.Tensor, n: int, lanes: int, device) -> torch.Tensor:
    """A caller-supplied digest tensor must be exactly what the kernels write:
    n * lanes contiguous 64-bit words, on the launch device or on a GPU the
    launch device can store to directly (peer access: the digests then go
    straight into that GPU's memory, see peer.py); else the launch would
    write out of bounds or scramble digests."""
    if not isinstance(out, torch.Tensor):
        raise ValueError("out must be a torch tensor")
    if not out.is_cuda or (out.device != device and not _peer_ok(device, out.device)):
        raise ValueError(f"out must be a CUDA tensor on {device} (or a peer-accessible "
                         f"GPU), got {out.device}")
    if out.dtype not in (torch.int64, torch.uint64):
        raise ValueError(f"out must be int64 (or uint64), got {out.dtype}")
    if tuple(out.shape) != _out_shape(n, lanes) or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous tensor of shape {_out_shape(n, lanes)}, "
                         f"got {tuple(out.shape)}")
    return out


# ---------------------------------------------------------------------------
# Fixed-length batches
# ---------------------------------------------------------------------------

def _launch_fixed(kind, key, d_msgs: torch.Tensor, n: int, L: int, p1: int, p2: int,
                  tree: int, d_out: torch.Tensor, kernel: int, device) -> None:
    st = _stream_ptr(device)
    ptr = d_msgs.data_ptr() if d_msgs.numel() else 0
    if kind == "hh":
        rc = _lib.lib().lh_highway_fixed_kernel(ptr, n, L, _key4(key), p1, p2,
                                                d_out.data_ptr(), st, kernel)
        _lib.check(rc, "lh_highway_fixed")
    else:
        rc = _lib.lib().lh_siphash_fixed_kernel(ptr, n, L, _key2(key), p1, p2, tree,
                                                d_out.data_ptr(), st, kernel)
        _lib.check(rc, "lh_siphash_fixed")


def _fixed(kind, key, msgs, p1, p2, tree, lanes, kernel, out=None):
    # Fast path for the common small-batch call (a contiguous uint8 CUDA
    # tensor on the current device): one ctypes call, no device switch.
    if (isinstance(msgs, torch.Tensor) and msgs.is_cuda and msgs.dtype is torch.uint8
            and msgs.dim() == 2 and msgs.is_contiguous()):
        idx = msgs.get_device()
        if _CUDA_CHECKED and idx == torch.cuda.current_device():
            n, L = msgs.shape
            if out is None:
                out = torch.empty(_out_shape(n, lanes), dtype=torch.int64, device=msgs.device)
            elif (out.device != msgs.device or out.dtype is not torch.int64
                  or out.shape != _out_shape(n, lanes) or not out.is_contiguous()):
                _check_out(out, n, lanes, msgs.device)
            if n:
                st = _raw_stream(idx) if _raw_stream is not None else \
                    torch.cuda.current_stream(idx).cuda_stream
                ptr = msgs.data_ptr() if L else 0
                if kind == "hh":
                    rc = _lib.lib().lh_highway_fixed_kernel(ptr, n, L, _key4(key), p1, p2,
                                                            out.data_ptr(), st, kernel)
                else:
                    rc = _lib.lib().lh_siphash_fixed_kernel(ptr, n, L, _key2(key), p1, p2, tree,
                                                            out.data_ptr(), st, kernel)
                if rc:
                    _lib.check(rc, "lh_highway_fixed" if kind == "hh" else "lh_siphash_fixed")
            return out
    device = _require_cuda()
    m = _as_u8_2d(msgs)
    n, L = m.shape
    if m.is_cuda:
        m = m.contiguous()
        if out is None:
            out = torch.empty(_out_shape(n, lanes), dtype=torch.int64, device=m.device)
        else:
            _check_out(out, n, lanes, m.device)
        if n:
            with _on_device(m.device):
                _launch_fixed(kind, key, m, n, L, p1, p2, tree, out, kernel, m.device)
        return out
    if out is not None:
        raise ValueError("out= is only accepted with CUDA input (host batches return numpy)")
    return _fixed_host(kind, key, m.contiguous(), p1, p2, tree, lanes, kernel, device)


def _fixed_host(kind, key, m: torch.Tensor, p1, p2, tree, lanes, kernel, device):
    """Stream a host (n, L) batch through the GPU: per chunk, H2D -> kernel ->
    D2H on alternating streams so copies overlap the other chunk's kernel."""
    n, L = m.shape
    out_host = torch.empty(_out_shape(n, lanes), dtype=torch.int64,
                           pin_memory=torch.cuda.is_available())
    if n == 0:
        return to_u64(out_host)
    rows = n if L == 0 else max(1, min(n, HOST_CHUNK_BYTES // L))
    if rows < n and rows >= 128:
        rows -= rows % 128
    streams = [torch.cuda.Stream(device), torch.cuda.Stream(device)]
    cur = torch.cuda.current_stream(device)
    nbuf = 2 if rows < n else 1
    dbuf = [torch.empty((rows, L), dtype=torch.uint8, device=device) for _ in range(nbuf)]
    dout = [torch.empty(_out_shape(rows, lanes), dtype=torch.int64, device=device)
            for _ in range(nbuf)]
    for s in streams:
        s.wait_stream(cur)
    for k, r0 in enumerate(range(0, n, rows)):
        r1 = min(n, r0 + rows)
        s = streams[k % 2]
        b = k % nbuf
        with torch.cuda.stream(s):
            db = dbuf[b][: r1 - r0]
            db.copy_(m[r0:r1], non_blocking=True)
            do = dout[b][: r1 - r0]
            _launch_fixed(kind, key, db, r1 - r0, L, p1, p2, tree, do, kernel, device)
            out_host[r0:r1].copy_(do, non_blocking=True)
    for s in streams:
        s.synchronize()
    return to_u64(out_host)


def highway_batch(key, messages, width: int = 64, rounds: int = 4,
                  kernel: int = KERNEL_AUTO, out: Optional[torch.Tensor] = None):
    """HighwayHash-64/128/256 of every row of an (n, L) uint8 batch."""
    _check_width(width)
    if rounds < 0:
        raise ValueError("rounds must be >= 0")
    return _fixed("hh", as_key256(key), messages, width, rounds, 0, width // 64, kernel, out)


def sip_batch(key, messages, c: int = 2, d: int = 4, tree: bool = False,
              kernel: int = KERNEL_AUTO, out: Optional[torch.Tensor] = None):
    """SipHash-c-d (tree=False) or SipTreeHash (tree=True) of every row."""
    if c < 1 or d < 1:
        raise ValueError("round counts must be positive")
    return _fixed("sip", as_key128(key), messages, c, d, int(bool(tree)), 1, kernel, out)


# ---------------------------------------------------------------------------
# Ragged batches
# ---------------------------------------------------------------------------

def _to_device(x, dtype, device):
    if isinstance(x, torch.Tensor):
        if x.dtype != dtype:
            raise ValueError(f"expected {dtype}, got {x.dtype}")
        return x.to(device, non_blocking=True).contiguous()
    return _host_view(np.ascontiguousarray(x).view(
        {torch.uint8: np.uint8, torch.int64: np.int64, torch.int32: np.int32}[dtype])
    ).to(device).contiguous()


def _ragged_kernel(kind, kernel, span_bytes, n):
    """Kernel for a ragged launch.  HighwayHash: the register ring when the
    mean message length reaches RING_MIN_MEAN_BYTES, else the warp-staged
    short-key kernel.  Sip: warp-staged below SIP_STAGED_MAX_MEAN_BYTES,
    else the register ring."""
    allowed = (KERNEL_DIRECT, KERNEL_RING, KERNEL_STAGED)
    if kernel != KERNEL_AUTO:
        if kernel not in allowed:
            raise ValueError(f"ragged {kind} batches take KERNEL_AUTO or one of {allowed}")
        return kernel
    if kind != "hh":  # Sip: warp-staged keys below 64 B on average, else the ring
        return KERNEL_STAGED if n and span_bytes < SIP_STAGED_MAX_MEAN_BYTES * n else KERNEL_RING
    if n and span_bytes >= RING_MIN_MEAN_BYTES * n:
        return KERNEL_RING
    return KERNEL_STAGED


def _launch_ragged(kind, key, buf_ptr, off_ptr, len_ptr, n, p1, p2, tree, out, device,
                   kernel=KERNEL_AUTO, order=None):
    st = _stream_ptr(device)
    if order is not None:  # length-class schedule (register-ring kernel)
        if kind == "hh":
            rc = _lib.lib().lh_highway_ragged_ordered(buf_ptr, off_ptr, len_ptr, n,
                                                      order.data_ptr(), _key4(key), p1, p2,
                                                      out.data_ptr(), st)
        else:
            rc = _lib.lib().lh_siphash_ragged_ordered(buf_ptr, off_ptr, len_ptr, n,
                                                      order.data_ptr(), _key2(key), p1, p2, tree,
                                                      out.data_ptr(), st)
    elif kind == "hh":
        rc = _lib.lib().lh_highway_ragged_kernel(buf_ptr, off_ptr, len_ptr, n, _key4(key), p1,
                                                 p2, out.data_ptr(), st, kernel)
    else:
        rc = _lib.lib().lh_siphash_ragged_kernel(buf_ptr, off_ptr, len_ptr, n, _key2(key), p1,
                                                 p2, tree, out.data_ptr(), st, kernel)
    _lib.check(rc, "ragged batch")


# Work units of one message for the lane-balance statistic (lh_ragged_plan_stats):
# (unit_shift, fixed_units) = 32-byte packets + 5 Updates of finalization and
# remainder for HighwayHash; 8-byte words + 3 compressions for the Sip family.
_WORK_UNITS = {"hh": (5, 5), "sip": (3, 3)}
# Cost model of the automatic schedule (scripts/ragged_balance_bench.py, B200):
# the ring kernels retire about 164 G HighwayHash lane-packets/s and 324 G
# SipHash-2-4 lane-words/s; ordering costs ~15 us + 12 ps per message; an
# ordered batch runs at ~0.93 warp efficiency.
BALANCE_ORDERED_EFFICIENCY = 0.93
BALANCE_COST_S = (15e-6, 12e-12)
BALANCE_MARGIN = 1.2


def _unit_seconds(kind, p1):
    """Seconds per lane-step of the ring kernels (kind "sip": p1 = c rounds)."""
    return 1 / 164e9 if kind == "hh" else (1.45e-12 * max(int(p1), 1) + 0.2e-12)


def balance_gain(kind, p1, n, wsum, wmax32):
    """(estimated seconds saved by the length-class schedule, its cost)."""
    if not wmax32:
        return 0.0, BALANCE_COST_S[0]
    eff = wsum / wmax32
    saved = wmax32 * _unit_seconds(kind, p1) * max(0.0, 1 - eff / BALANCE_ORDERED_EFFICIENCY)
    return saved, BALANCE_COST_S[0] + BALANCE_COST_S[1] * n


def _plan(d_off, d_len, n: int, chunk_msgs: int, buf_len: int, device, stats_kind=None):
    """lh_ragged_plan: per-chunk byte spans [lo, hi) and the invalid-message
    count of a device-resident layout, in one launch and one small D2H
    (csrc/lh_plan.cu).  Raises ValueError for an invalid layout.  With
    ``stats_kind`` ("hh" or "sip") also returns (sum of work, sum over
    32-message groups of 32 * max work) of the natural order; their ratio is
    its warp efficiency."""
    nchunks = -(-n // chunk_msgs)
    res = torch.empty(2 * nchunks + 3, dtype=torch.int64, device=device)
    shift, fixed = _WORK_UNITS.get(stats_kind, (0, 0))
    rc = _lib.lib().lh_ragged_plan_stats(
        d_off.data_ptr(), None if d_len is None else d_len.data_ptr(), n, chunk_msgs,
        buf_len & 0xFFFFFFFFFFFFFFFF, res.data_ptr(), res[nchunks:].data_ptr(),
        res[2 * nchunks:].data_ptr(), res[2 * nchunks + 1:].data_ptr() if stats_kind else None,
        shift, fixed, _stream_ptr(device))
    _lib.check(rc, "lh_ragged_plan")
    r = res.cpu().numpy().view(np.uint64)
    if r[2 * nchunks]:
        raise ValueError(f"invalid ragged layout: {int(r[2 * nchunks])} of {n} messages have "
                         f"decreasing offsets, a wrapping length or end past the {buf_len}-byte "
                         "buffer")
    if stats_kind:
        return r[:nchunks], r[nchunks:2 * nchunks], (int(r[2 * nchunks + 1]), int(r[2 * nchunks + 2]))
    return r[:nchunks], r[nchunks:2 * nchunks]


def ragged_order(d_off, d_len, n: int, kind: str = "hh"):
    """lh_ragged_order: the batch as (n, 4) int32 schedule records {offset lo,
    offset hi, length, message index} grouped by length class, longest first,
    for the ordered ragged launches."""
    device = d_off.device
    sched = torch.empty((n, 4), dtype=torch.int32, device=device)
    scratch = torch.empty(1024, dtype=torch.int32, device=device)
    rc = _lib.lib().lh_ragged_order(d_off.data_ptr(), None if d_len is None else d_len.data_ptr(),
                                    n, _WORK_UNITS["hh" if kind == "hh" else "sip"][0],
                                    sched.data_ptr(), scratch.data_ptr(), _stream_ptr(device))
    _lib.check(rc, "lh_ragged_order")
    return sched


def _check_schedule(schedule, n, device):
    if not (isinstance(schedule, torch.Tensor) and schedule.is_cuda and schedule.device == device
            and schedule.dtype is torch.int32 and tuple(schedule.shape) == (n, 4)
            and schedule.is_contiguous()):
        raise ValueError(f"schedule must be the ({n}, 4) int32 tensor ragged_order returned "
                         f"for this layout, on {device}")
    return schedule


def _schedule(kind, p1, d_off, d_len, n, buf_len, device, kern, check, balance, schedule=None):
    """Layout validation and the lane-balance decision of one device-resident
    ragged launch.  Returns the schedule tensor or None.  balance=None: order
    the batch when the validation pass (check=True) measures a natural order
    whose estimated loss exceeds BALANCE_MARGIN x the cost of ordering
    (balance_gain); True: always (ring-kernel launches); False: never."""
    ring = kern in (KERNEL_RING, KERNEL_DIRECT) and n < (1 << 32)
    capturing = torch.cuda.is_current_stream_capturing()
    sk = "hh" if kind == "hh" else "sip"
    if schedule is not None:  # the caller's own (ragged_order of this layout, reused)
        if not ring:
            raise ValueError("schedule= applies to register-ring launches (kernel=KERNEL_RING)")
        _check_schedule(schedule, n, device)
        if check and not capturing:
            _plan(d_off, d_len, n, n, buf_len, device)
        return schedule
    auto = balance is None and ring
    want = balance is True and ring
    if check and not capturing:
        r = _plan(d_off, d_len, n, n, buf_len, device, sk if auto else None)
        if auto:
            saved, cost = balance_gain(sk, p1, n, *r[2])
            want = saved > BALANCE_MARGIN * cost
    return ragged_order(d_off, d_len, n, sk) if want else None


def _ragged_host_pipelined(kind, key, buf, offsets, lengths, p1, p2, tree, lanes, device,
                           kernel=KERNEL_AUTO):
    """Host ragged batch streamed through the GPU in message-range chunks of
    about HOST_CHUNK_BYTES.  The offsets/lengths go to the device first (one
    copy each); one lh_ragged_plan launch validates the layout and reduces
    each chunk's byte span [min start, max end), read back once for all
    chunks; then per chunk the span goes H2D, the kernel runs and the digests
    come back D2H, alternating two streams so copies overlap the other
    chunk's kernel.  Offsets are not rebased: the kernel gets d_span -
    span_start as its buffer base (span_start 16-aligned), so buf +
    offsets[i] lands inside the copied span.  Returns None when the spans are
    too scattered (caller falls back to one copy)."""
    buf_t = buf if isinstance(buf, torch.Tensor) else _host_view(
        np.ascontiguousarray(buf, dtype=np.uint8))
    buf_t = buf_t.reshape(-1)
    off_t = offsets if isinstance(offsets, torch.Tensor) else _host_view(
        np.ascontiguousarray(offsets).astype(np.uint64, copy=False).view(np.int64))
    len_t = None
    if lengths is not None:
        len_t = lengths if isinstance(lengths, torch.Tensor) else _host_view(
            np.ascontiguousarray(lengths).astype(np.uint32, copy=False).view(np.int32))
    n = off_t.numel() - 1 if len_t is None else off_t.numel()
    if n <= 0 or (len_t is not None and len_t.numel() != n):
        return None
    d_off = off_t.to(device, non_blocking=True).contiguous()
    d_len = None if len_t is None else len_t.to(device, non_blocking=True).contiguous()
    # Chunk count from the buffer size (packed batches: span ~ buffer / chunks).
    nchunks = max(1, min(256, -(-max(buf_t.numel(), 1) // HOST_CHUNK_BYTES)))
    cnt = -(-n // nchunks)
    los, his = _plan(d_off, d_len, n, cnt, buf_t.numel(), device)
    spans = []
    for k, (lo, hi) in enumerate(zip(los.tolist(), his.tolist())):
        a, b = k * cnt, min(n, (k + 1) * cnt)
        lo &= ~15
        if hi - lo > 4 * HOST_CHUNK_BYTES + 4096:
            return None  # scattered offsets: no compact span per chunk
        spans.append((a, b, lo, max(hi, lo)))
    out_host = torch.empty(_out_shape(n, lanes), dtype=torch.int64,
                           pin_memory=torch.cuda.is_available())
    streams = [torch.cuda.Stream(device), torch.cuda.Stream(device)]
    cur = torch.cuda.current_stream(device)
    for s in streams:
        s.wait_stream(cur)
    for k, (a, b, lo, hi) in enumerate(spans):
        s = streams[k % 2]
        with torch.cuda.stream(s):
            d_span = buf_t[lo:hi].to(device, non_blocking=True) if hi > lo else \
                torch.empty(16, dtype=torch.uint8, device=device)
            d_o = d_off[a:b + 1] if d_len is None else d_off[a:b]
            d_l = None if d_len is None else d_len[a:b]
            d_out = torch.empty(_out_shape(b - a, lanes), dtype=torch.int64, device=device)
            _launch_ragged(kind, key, (d_span.data_ptr() - lo) & 0xFFFFFFFFFFFFFFFF,
                           d_o.data_ptr(), None if d_l is None else d_l.data_ptr(), b - a,
                           p1, p2, tree, d_out, device, _ragged_kernel(kind, kernel, hi - lo, b - a))
            out_host[a:b].copy_(d_out, non_blocking=True)
    for s in streams:
        s.synchronize()
    return to_u64(out_host)


def _ragged_fast(kind, key, buf, offsets, lengths, p1, p2, tree, lanes, out, kernel, check,
                 balance=None, schedule=None):
    """The common launch-bound call -- contiguous CUDA tensors of the right
    dtypes on the current device -- in one ctypes call (the general path's
    conversions cost more than a small kernel).  None if not applicable."""
    if not (isinstance(buf, torch.Tensor) and isinstance(offsets, torch.Tensor) and _CUDA_CHECKED
            and buf.is_cuda and offsets.is_cuda and buf.dtype is torch.uint8
            and offsets.dtype is torch.int64 and buf.is_contiguous() and offsets.is_contiguous()):
        return None
    idx = buf.get_device()
    if idx != torch.cuda.current_device() or offsets.get_device() != idx:
        return None
    if lengths is not None and not (isinstance(lengths, torch.Tensor) and lengths.is_cuda
                                    and lengths.dtype is torch.int32 and lengths.is_contiguous()
                                    and lengths.get_device() == idx):
        return None
    if buf.dim() != 1 or offsets.dim() != 1 or kernel not in (KERNEL_AUTO, KERNEL_DIRECT,
                                                               KERNEL_RING, KERNEL_STAGED):
        return None
    n = offsets.numel() - 1 if lengths is None else offsets.numel()
    if n < 0 or (lengths is not None and lengths.numel() != n):
        return None
    device = buf.device
    if out is None:
        out = torch.empty(_out_shape(n, lanes), dtype=torch.int64, device=device)
    elif (out.device != device or out.dtype is not torch.int64
          or out.shape != _out_shape(n, lanes) or not out.is_contiguous()):
        _check_out(out, n, lanes, device)
    if n:
        kern = _ragged_kernel(kind, kernel, buf.numel(), n)
        order = _schedule(kind, p1, offsets, lengths, n, buf.numel(), device, kern, check, balance,
                          schedule)
        bp = buf.data_ptr() if buf.numel() else offsets.data_ptr()
        _launch_ragged(kind, key, bp, offsets.data_ptr(),
                       None if lengths is None else lengths.data_ptr(), n, p1, p2, tree, out,
                       device, kern, order)
    return out


def _ragged(kind, key, buf, offsets, lengths, p1, p2, tree, lanes, out=None,
            kernel=KERNEL_AUTO, check=True, balance=None, schedule=None):
    r = _ragged_fast(kind, key, buf, offsets, lengths, p1, p2, tree, lanes, out, kernel, check,
                     balance, schedule)
    if r is not None:
        return r
    device = _require_cuda()
    _ragged_kernel(kind, kernel, 0, 0)  # validate before any work
    host = not (isinstance(buf, torch.Tensor) and buf.is_cuda)
    if host and out is None and not any(isinstance(x, torch.Tensor) and x.is_cuda
                                        for x in (offsets, lengths)):
        r = _ragged_host_pipelined(kind, key, buf, offsets, lengths, p1, p2, tree, lanes, device,
                                   kernel)
        if r is not None:
            return r
    if isinstance(offsets, np.ndarray):
        offsets = offsets.astype(np.uint64, copy=False).view(np.int64)
    if isinstance(lengths, np.ndarray):
        lengths = lengths.astype(np.uint32, copy=False).view(np.int32)
    if isinstance(buf, np.ndarray):
        buf = buf.astype(np.uint8, copy=False).reshape(-1)
    d_buf = _to_device(buf, torch.uint8, device)
    d_off = _to_device(offsets, torch.int64, device)
    d_len = None if lengths is None else _to_device(lengths, torch.int32, device)
    n = d_off.numel() - 1 if d_len is None else d_off.numel()
    if d_len is not None and d_len.numel() != n:
        raise ValueError("offsets and lengths disagree on the message count")
    if n < 0:
        raise ValueError("offsets must hold n+1 entries when lengths is None")
    if out is None:
        out = torch.empty(_out_shape(n, lanes), dtype=torch.int64, device=device)
    else:
        _check_out(out, n, lanes, device)
    if n:
        # Host inputs are always checked (one extra sync is noise there).  A
        # layout being captured into a CUDA graph cannot be read back: trusted.
        kern = _ragged_kernel(kind, kernel, d_buf.numel(), n)
        order = _schedule(kind, p1, d_off, d_len, n, d_buf.numel(), device, kern, check or host,
                          balance, schedule)
        bp = d_buf.data_ptr() if d_buf.numel() else d_off.data_ptr()
        lp = d_len.data_ptr() if d_len is not None else None
        _launch_ragged(kind, key, bp, d_off.data_ptr(), lp, n, p1, p2, tree, out, device, kern,
                       order)
    if host:
        return to_u64(out)
    return out


def highway_ragged(key, buf, offsets, lengths=None, width: int = 64, rounds: int = 4,
                   out: Optional[torch.Tensor] = None, kernel: int = KERNEL_AUTO,
                   check: bool = True, balance: Optional[bool] = None,
                   schedule: Optional[torch.Tensor] = None):
    """HighwayHash over a packed ragged buffer.  Message i is
    buf[offsets[i] : offsets[i] + len_i] with len_i = lengths[i] when given,
    else offsets[i+1] - offsets[i] (offsets then holds n+1 entries).
    kernel: KERNEL_AUTO picks by mean length (RING_MIN_MEAN_BYTES);
    KERNEL_RING (or KERNEL_DIRECT) forces the register-ring kernel,
    KERNEL_STAGED the warp-staged short-key kernel.
    check: validate the layout first (lh_ragged_plan: offsets non-decreasing,
    no wrapping length, every message inside buf; ValueError otherwise).  It
    costs one metadata pass and a sync; check=False skips it for CUDA inputs
    the caller has validated (the C ABI's contract: offsets are trusted).
    Host inputs are always checked; calls captured into a CUDA graph are not
    (nothing can be read back during capture).
    balance: the lane schedule of register-ring launches.  One message per
    lane means a warp runs until its longest message is done; None (default)
    lets the validation pass measure the natural order's warp efficiency and,
    when the estimated loss outweighs the cost of ordering (balance_gain),
    hashes the messages grouped by length class (lh_ragged_order; digests
    stay in message order).  True always orders,
    False never; with check=False nothing is measured, so None means False.
    schedule: a schedule built once with ragged_order(offsets, lengths, n, "hh")
    and reused for every batch of the same layout (only the bytes change):
    the ordering launches are then paid once (cfg2: 15.3 -> 13.1 us)."""
    _check_width(width)
    if rounds < 0:
        raise ValueError("rounds must be >= 0")
    return _ragged("hh", as_key256(key), buf, offsets, lengths, width, rounds, 0,
                   width // 64, out, kernel, check, balance, schedule)


def sip_ragged(key, buf, offsets, lengths=None, c: int = 2, d: int = 4, tree: bool = False,
               out: Optional[torch.Tensor] = None, kernel: int = KERNEL_AUTO,
               check: bool = True, balance: Optional[bool] = None,
               schedule: Optional[torch.Tensor] = None):
    """SipHash-c-d / SipTreeHash over a packed ragged buffer (layout,
    ``check``, ``balance`` and ``schedule`` as highway_ragged; build the
    schedule with ragged_order(..., "sip"))."""
    if c < 1 or d < 1:
        raise ValueError("round counts must be positive")
    return _ragged("sip", as_key128(key), buf, offsets, lengths, c, d, int(bool(tree)), 1, out,
                   kernel, check, balance, schedule)


# ---------------------------------------------------------------------------
# PRF mode and one-shot helpers
# ---------------------------------------------------------------------------

def prf64(key, start: int, n: int, rounds: int = 4, out: Optional[torch.Tensor] = None):
    """out[i] = HighwayHash-64(key, le64(start + i)) for i < n (device tensor)."""
    device = _require_cuda()
    if n < 0 or rounds < 0:
        raise ValueError("n and rounds must be >= 0")
    if out is None:
        out = torch.empty((n,), dtype=torch.int64, device=device)
    else:
        _check_out(out, n, 1, device)
    if n:
        rc = _lib.lib().lh_highway_prf64(start, n, _key4(as_key256(key)), rounds,
                                         out.data_ptr(), _stream_ptr(device))
        _lib.check(rc, "lh_highway_prf64")
    return out


def update_states(states, packets, inverse: bool = False):
    """update (S/highway.py:130-150) or update_inverse (:153-173) of n raw
    states: (n,16) lanes v0, v1, mul0, mul1 and (n,4) packets, uint64 numpy
    or int64 CUDA tensors.  CUDA tensors are updated in place and returned;
    host arrays come back as a new numpy uint64 array."""
    device = _require_cuda()
    host = not (isinstance(states, torch.Tensor) and states.is_cuda)
    if host:
        st = np.ascontiguousarray(states, dtype=np.uint64).reshape(-1, 16)
        pk = np.ascontiguousarray(packets, dtype=np.uint64).reshape(-1, 4)
        d_st = torch.from_numpy(st.view(np.int64).copy()).to(device)
        d_pk = _host_view(pk.view(np.int64)).to(device)
    else:
        d_st, d_pk = states, packets
        if not isinstance(d_pk, torch.Tensor) or not d_pk.is_cuda:
            raise ValueError("states and packets must both be CUDA tensors (or both host)")
        if d_st.dtype != torch.int64 or d_pk.dtype != torch.int64:
            raise ValueError("CUDA states and packets must be int64 tensors")
        if not (d_st.is_contiguous() and d_pk.is_contiguous()):
            raise ValueError("CUDA states and packets must be contiguous")
    n = d_st.numel() // 16
    if d_st.numel() != 16 * n or d_pk.numel() != 4 * n:
        raise ValueError("need (n,16) states and (n,4) packets")
    if n:
        rc = _lib.lib().lh_highway_update_states(d_st.data_ptr(), d_pk.data_ptr(), n,
                                                 int(bool(inverse)), _stream_ptr(device))
        _lib.check(rc, "lh_highway_update_states")
    return to_u64(d_st).reshape(n, 16) if host else d_st


def remainder_states(states, tails, r):
    """update_remainder (S/highway.py:182-199) of n raw states with tails
    (n, 32) uint8 (bytes beyond r[i] ignored) and r (n,) in 1..31.  Host
    arrays only; returns the new (n, 16) uint64 states."""
    device = _require_cuda()
    st = np.ascontiguousarray(states, dtype=np.uint64).reshape(-1, 16)
    tl = np.ascontiguousarray(tails, dtype=np.uint8).reshape(-1, 32)
    rr = np.ascontiguousarray(r, dtype=np.uint32).reshape(-1)
    n = len(st)
    if len(tl) != n or len(rr) != n:
        raise ValueError("need (n,16) states, (n,32) tails and (n,) lengths")
    if n and (rr.min() < 1 or rr.max() > 31):
        raise ValueError("remainder length must be in 1..31")
    if not n:
        return st.copy()
    d_st = torch.from_numpy(st.view(np.int64).copy()).to(device)
    d_tl = _host_view(tl).to(device)
    d_r = _host_view(rr.view(np.int32)).to(device)
    rc = _lib.lib().lh_highway_remainder_states(d_st.data_ptr(), d_tl.data_ptr(), d_r.data_ptr(),
                                                n, _stream_ptr(device))
    _lib.check(rc, "lh_highway_remainder_states")
    return to_u64(d_st).reshape(n, 16)


def finalize_states(states, width: int = 64, rounds: int = 4) -> np.ndarray:
    """finalize (S/highway.py:223-234) of n raw (n, 16) states: numpy
    uint64 (n,) for width 64, else (n, width/64)."""
    _check_width(width)
    if rounds < 0:
        raise ValueError("rounds must be >= 0")
    device = _require_cuda()
    st = np.ascontiguousarray(states, dtype=np.uint64).reshape(-1, 16)
    n = len(st)
    lanes = width // 64
    out = torch.empty(_out_shape(n, lanes), dtype=torch.int64, device=device)
    if n:
        d_st = _host_view(st.view(np.int64)).to(device)
        rc = _lib.lib().lh_highway_finalize_states(d_st.data_ptr(), n, width, rounds,
                                                   out.data_ptr(), _stream_ptr(device))
        _lib.check(rc, "lh_highway_finalize_states")
    return to_u64(out)


def sip_round_states(states, rounds: int = 1) -> np.ndarray:
    """`rounds` SipRounds (S/sip.py:73-86) of n (n, 4) uint64 host states;
    returns the new states."""
    if rounds < 0:
        raise ValueError("rounds must be >= 0")
    device = _require_cuda()
    st = np.ascontiguousarray(states, dtype=np.uint64).reshape(-1, 4)
    if not len(st):
        return st.copy()
    d_st = torch.from_numpy(st.view(np.int64).copy()).to(device)
    rc = _lib.lib().lh_sip_round_states(d_st.data_ptr(), len(st), rounds, _stream_ptr(device))
    _lib.check(rc, "lh_sip_round_states")
    return to_u64(d_st).reshape(-1, 4)


def bijectivity(seed: int, n: int):
    """Device self-test: (failures, fold) over n synthetic (state, packet)
    cases, case i = words 20i..20i+19 of synth stream (seed, 0)."""
    device = _require_cuda()
    if n < 0:
        raise ValueError("n must be >= 0")
    res = torch.zeros(2, dtype=torch.int64, device=device)
    rc = _lib.lib().lh_highway_bijectivity(seed, n, res.data_ptr(), _stream_ptr(device))
    _lib.check(rc, "lh_highway_bijectivity")
    r = to_u64(res)
    return int(r[0]), int(r[1])


def _one(message):
    device = _require_cuda()
    raw = bytes(message)
    t = torch.frombuffer(bytearray(raw or b"\0"), dtype=torch.uint8)
    return t.to(device)[: len(raw)].reshape(1, len(raw)), device


def hash_one(key: Key256, message, width: int, rounds: int) -> np.ndarray:
    _check_width(width)
    if rounds < 0:
        raise ValueError("rounds must be >= 0")
    m, device = _one(message)
    out = torch.empty((width // 64,), dtype=torch.int64, device=device)
    _launch_fixed("hh", key, m, 1, m.shape[1], width, rounds, 0, out, KERNEL_AUTO, device)
    return to_u64(out)


def sip_one(key: Key128, message, c: int, d: int, tree: bool) -> int:
    if c < 1 or d < 1:
        raise ValueError("round counts must be positive")
    m, device = _one(message)
    out = torch.empty((1,), dtype=torch.int64, device=device)
    _launch_fixed("sip", key, m, 1, m.shape[1], c, d, int(bool(tree)), out, KERNEL_AUTO, device)
    return int(to_u64(out)[0])


# ---------------------------------------------------------------------------
# Batched streaming (incremental) hashing — csrc/lh_stream.cu
# ---------------------------------------------------------------------------

ALG_HIGHWAY = _lib.ALG_HIGHWAY
ALG_SIPHASH = _lib.ALG_SIPHASH
ALG_SIPTREE = _lib.ALG_SIPTREE


class StreamBatch:
    """n messages hashed incrementally on the device.

    The batch form of StreamingHasher / SipHasher / SipTreeHasher
    (S/highway.py:257-285, S/sip.py:131-203): ``append`` one chunk per
    message (an (n, Lc) uint8 tensor, or a ragged ``(buf, offsets[, lengths])``
    triple), any number of times; ``finish`` returns the digests of
    everything appended.  Appending after ``finish`` or finishing twice raises
    RuntimeError, as the reference's hashers do (S/highway.py:269-281)."""

    def __init__(self, alg: int, key, n: int, width: int = 64, rounds: int = 4,
                 c: int = 2, d: int = 4):
        self.device = _require_cuda()
        if n < 0:
            raise ValueError("n must be >= 0")
        self.alg, self.n = alg, n
        if alg == ALG_HIGHWAY:
            _check_width(width)
            k, p1, p2, self.lanes = _key4(as_key256(key)), width, rounds, width // 64
        elif alg in (ALG_SIPHASH, ALG_SIPTREE):
            if c < 1 or d < 1:
                raise ValueError("round counts must be positive")
            k, p1, p2, self.lanes = _key2(as_key128(key)), c, d, 1
        else:
            raise ValueError(f"unknown algorithm id {alg}")
        rec = _lib.lib().lh_stream_state_bytes(alg)
        self.state = torch.empty(max(1, n) * rec, dtype=torch.uint8, device=self.device)
        self._finished = False
        _lib.check(_lib.lib().lh_stream_init(alg, self.state.data_ptr(), n, k, p1, p2,
                                             _stream_ptr(self.device)), "lh_stream_init")

    def append(self, chunks, offsets=None, lengths=None) -> "StreamBatch":
        if self._finished:
            raise RuntimeError("cannot append after finish")
        st = _stream_ptr(self.device)
        if offsets is None:
            m = _as_u8_2d(chunks)
            if m.shape[0] != self.n:
                raise ValueError("one chunk per message expected")
            m = m.to(self.device).contiguous()
            ptr = m.data_ptr() if m.numel() else 0
            rc = _lib.lib().lh_stream_update(self.alg, self.state.data_ptr(), self.n, ptr, None,
                                             None, m.shape[1], st)
            keep = (m,)
        else:
            d_buf = _to_device(chunks.reshape(-1) if isinstance(chunks, np.ndarray) else chunks,
                               torch.uint8, self.device)
            if isinstance(offsets, np.ndarray):
                offsets = offsets.astype(np.uint64, copy=False).view(np.int64)
            if isinstance(lengths, np.ndarray):
                lengths = lengths.astype(np.uint32, copy=False).view(np.int32)
            d_off = _to_device(offsets, torch.int64, self.device)
            d_len = None if lengths is None else _to_device(lengths, torch.int32, self.device)
            nn = d_off.numel() - 1 if d_len is None else d_off.numel()
            if nn != self.n:
                raise ValueError("one chunk per message expected")
            if nn and not torch.cuda.is_current_stream_capturing():
                _plan(d_off, d_len, nn, nn, d_buf.numel(), self.device)  # layout check
            bp = d_buf.data_ptr() if d_buf.numel() else d_off.data_ptr()
            rc = _lib.lib().lh_stream_update(self.alg, self.state.data_ptr(), self.n, bp,
                                             d_off.data_ptr(),
                                             d_len.data_ptr() if d_len is not None else None,
                                             0, st)
            keep = (d_buf, d_off, d_len)
        _lib.check(rc, "lh_stream_update")
        self._keep = keep  # inputs stay alive until the next call on this stream
        return self

    def finish(self, width: Optional[int] = None):
        """Digests (device tensor).  HighwayHash may pick the width here (the
        absorbed state is width-independent); default: the init width."""
        if self._finished:
            raise RuntimeError("finish may only be called once")
        lanes = self.lanes
        if width is not None:
            if self.alg != ALG_HIGHWAY:
                raise ValueError("width applies to HighwayHash only")
            _check_width(width)
            lanes = width // 64
        self._finished = True
        out = torch.empty(_out_shape(self.n, lanes), dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().lh_stream_finish(self.alg, self.state.data_ptr(), self.n,
                                               out.data_ptr(), lanes,
                                               _stream_ptr(self.device)), "lh_stream_finish")
        return out
