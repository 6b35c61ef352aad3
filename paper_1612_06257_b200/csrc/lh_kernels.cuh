// lh_kernels.cuh — the sm_100a hashing kernels and their launchers, shared
// by the translation units of libb200hash.so: lh_engine.cu (HighwayHash and
// the extern "C" boundary) and lh_sip_variant.cu (compiled once per Sip
// variant, so the instantiations build in parallel).  Everything here is in
// an anonymous namespace: each TU instantiates only what it launches.
//
// Kernels:
//   k_tma_fixed<H,ROWS,STAGES[,STREAM]>  fixed-length batch; one thread per
//       message; a producer warp streams ROWS x 128-byte boxes of the (n, len)
//       byte matrix into a STAGES-deep shared-memory ring with 2-D TMA
//       (SWIZZLE_128B, so each thread's 16-byte reads of its own row are
//       bank-conflict free); consumer threads run the hash on registers.
//       STREAM: the streaming append of whole-block chunks.
//   k_tma_split  HighwayHash of few long messages: the state split over a
//       thread pair, 3-D TMA boxes of 16 rows x 512 B per warp (also STREAM).
//   k_ragged_short  short keys (ragged, or fixed rows <= 64 B): warp-staged
//       byte spans, non-divergent Update slots; falls back to the direct
//       reader.
//   k_staged_any<H,WARPS,MPL>  the warp staging for the Sip family's short
//       keys (ragged, or fixed rows of 12..63 B), 4 keys per lane.
//   k_ragged_ring<H,D,16>  ragged batches of medium/long messages
//       (HighwayHash), every ragged Sip batch and fixed rows TMA does not
//       take: one thread per message, 16-byte word reads branch-free in the
//       alignment (lh_reader.cuh: absorb_ring128), D packets in flight.
//   k_direct<H>  any layout (fixed or ragged, any alignment/length); one
//       thread per message reading its bytes with 8-byte-aligned loads and
//       funnel shifts (small batches; LH_KERNEL_DIRECT).
//   k_prf        HighwayHash-64 of 8-byte LE counters (no input bytes).
// H is one of lh::Highway, lh::Sip<C,D>, lh::SipTree<C,D> (lh_device.cuh).
//
// Note on hash_direct: keep the reader inline in this shape.  A version
// split into lh_reader.cuh's absorb_blocks + load_tail made ptxas (CUDA
// 12.9, sm_100a) rematerialise a loop-carried state word of the
// finalization loop from the kernel-parameter constant bank -- wrong digests
// for rounds >= 1.  The parity tests cover rounds 0..5.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "../../include/lanehash_b200.h"
#include "lh_device.cuh"
#include "lh_reader.cuh"
#include "lh_host.cuh"
#include "lh_stream.cuh"
#include "lh_tma.cuh"

using namespace lh;


namespace {

template <class H>
__host__ __device__ inline int nout(const H&) {
  return 1;
}
template <>
__host__ __device__ inline int nout<Highway>(const Highway& h) {
  return h.width / 64;
}

// Prototype staging.  Every HighwayHash kernel starts each message from a
// copy of the shared-memory prototype (Highway::load_state: 8 volatile
// LDS.128) instead of `h = proto`.  Two reasons: `h = proto` costs 16
// LDCU.64 + 32 IMAD.U32 per message (the parameter lives in the constant
// bank), and ptxas (CUDA 12.9, sm_100a) has miscompiled finalization loops
// that start from a parameter copy: it replaced the loop-carried v0[0] with
// the parameter's c[0x0][0x380] (profiles/r2_depth1/).  A
// value loaded by volatile LDS cannot be rematerialised from the constant
// bank.  Other hashers copy the parameter as before.
struct ProtoSmem {
  u64 w[16];
};

__device__ __forceinline__ u32 stage_proto(const Highway& p, ProtoSmem& s) {
  if (threadIdx.x < 16) {
    const u32 t = threadIdx.x;
    const u64* src = t < 4 ? p.v0 : t < 8 ? p.v1 : t < 12 ? p.m0 : p.m1;
    s.w[t] = src[t & 3];
  }
  return smem_u32(&s);
}
template <class H>
__device__ __forceinline__ u32 stage_proto(const H&, ProtoSmem& s) {
  return smem_u32(&s);
}

__device__ __forceinline__ void init_state(Highway& h, const Highway& p, u32 sa) {
  h.load_state(sa, p);
}
template <class H>
__device__ __forceinline__ void init_state(H& h, const H& p, u32) {
  h = p;
}

// PF: prefetch the next packet while hashing the current one (worth it for
// messages of several packets; costs registers, so fixed batches of short
// messages use PF = false).
template <bool PF, class H>
__device__ __forceinline__ void hash_direct(H& h, const uint8_t* msg, u64 len, u64* out) {
  const u64 full = len & ~31ull;
  const u32 r = (u32)(len & 31);
  const uintptr_t a = (uintptr_t)msg;
  const u32 sh = (u32)(a & 7) * 8;
  const u64* w = (const u64*)(a & ~(uintptr_t)7);
  u64 t[4] = {0, 0, 0, 0};
  const u64 nb = full >> 5;
  if (sh == 0) {
    if ((a & 15) == 0) {
      // Next packet's loads are issued before this packet's Update (one
      // thread walks its message alone; hide the load latency in-thread).
      const ulonglong2* w2 = (const ulonglong2*)w;
      ulonglong2 x = {0, 0}, y = {0, 0};
      if (PF && nb) {
        x = __ldg(w2);
        y = __ldg(w2 + 1);
      }
      for (u64 b = 0; b < nb; ++b) {
        ulonglong2 xn = {0, 0}, yn = {0, 0};
        if (!PF) {
          x = __ldg(w2 + 2 * b);
          y = __ldg(w2 + 2 * b + 1);
        } else if (b + 1 < nb) {
          xn = __ldg(w2 + 2 * b + 2);
          yn = __ldg(w2 + 2 * b + 3);
        }
        const u64 p[4] = {x.x, x.y, y.x, y.y};
        h.absorb32(p);
        x = xn;
        y = yn;
      }
    } else {
      for (u64 b = 0; b < nb; ++b) {
        const u64 p[4] = {ldg64(w + 4 * b), ldg64(w + 4 * b + 1), ldg64(w + 4 * b + 2),
                          ldg64(w + 4 * b + 3)};
        h.absorb32(p);
      }
    }
    if (r) {
      const u64* tw = w + (full >> 3);
      const u32 nw = (r + 7) >> 3;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((u32)k < nw) t[k] = ldg64(tw + k);
      mask_tail(t, r);
    }
  } else {
    u64 cur = len ? ldg64(w) : 0;
    u64 n0 = 0, n1 = 0, n2 = 0, n3 = 0;
    if (PF && nb) {
      n0 = ldg64(w + 1);
      n1 = ldg64(w + 2);
      n2 = ldg64(w + 3);
      n3 = ldg64(w + 4);
    }
    for (u64 b = 0; b < nb; ++b) {
      u64 m0 = 0, m1 = 0, m2 = 0, m3 = 0;
      if (!PF) {
        const u64* q = w + 4 * b;
        n0 = ldg64(q + 1);
        n1 = ldg64(q + 2);
        n2 = ldg64(q + 3);
        n3 = ldg64(q + 4);
      } else if (b + 1 < nb) {  // prefetch the next packet's words
        const u64* q = w + 4 * b + 4;
        m0 = ldg64(q + 1);
        m1 = ldg64(q + 2);
        m2 = ldg64(q + 3);
        m3 = ldg64(q + 4);
      }
      const u64 p[4] = {funnel(cur, n0, sh), funnel(n0, n1, sh), funnel(n1, n2, sh),
                        funnel(n2, n3, sh)};
      cur = n3;
      h.absorb32(p);
      n0 = m0;
      n1 = m1;
      n2 = m2;
      n3 = m3;
    }
    if (r) {
      // words covering [a+full, a+full+r): cur plus `extra` more.
      const u64 first = (a + full) >> 3;
      const u32 extra = (u32)(((a + full + r - 1) >> 3) - first);
      const u64* q = w + (full >> 3);
      u64 W[5];
      W[0] = cur;
#pragma unroll
      for (int k = 1; k < 5; ++k) W[k] = ((u32)k <= extra) ? ldg64(q + k) : 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) t[k] = funnel(W[k], W[k + 1], sh);
      mask_tail(t, r);
    }
  }
  h.finish(t, r, len, out);
}

template <class H, bool PF>
__global__ void __launch_bounds__(256) k_direct(const H proto, const uint8_t* __restrict__ buf,
                                                const u64* __restrict__ offsets,
                                                const u32* __restrict__ lengths, u64 fixed_len,
                                                u64 n, u64* __restrict__ out) {
  const int W = nout(proto);
  __shared__ __align__(16) ProtoSmem sp;
  const u32 sa = stage_proto(proto, sp);
  __syncthreads();
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    const uint8_t* msg;
    u64 len;
    if (offsets) {
      const u64 off = offsets[i];
      len = lengths ? (u64)lengths[i] : offsets[i + 1] - off;
      msg = buf + off;
    } else {
      msg = buf + i * fixed_len;
      len = fixed_len;
    }
    H h;
    init_state(h, proto, sa);
    hash_direct<PF>(h, msg, len, out + i * W);
  }
}

// The ring readers (lh_reader.cuh) with WORD-byte loads, then finalization.
template <int D, int WORD, class H>
__device__ __forceinline__ void hash_ring_any(H& h, const uint8_t* msg, u64 len, u64* out) {
  static_assert(WORD == 16, "the ring reader loads 16-byte words");
  u64 t[4];
  absorb_ring128<D>(h, msg, len, t);
  h.finish(t, (u32)(len & 31), len, out);
}

template <class H, int D, int WORD>
__global__ void __launch_bounds__(128) k_ragged_ring(const H proto, const uint8_t* __restrict__ buf,
                                                     const u64* __restrict__ offsets,
                                                     const u32* __restrict__ lengths,
                                                     u64 fixed_len, u64 n,
                                                     u64* __restrict__ out,
                                                     const uint4* __restrict__ sched) {
  const int W = nout(proto);
  __shared__ __align__(16) ProtoSmem sp;
  const u32 sa = stage_proto(proto, sp);
  __syncthreads();
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (u64)gridDim.x * blockDim.x) {
    u64 i = t;
    u64 off, len;
    if (sched) {
      // Schedule record t (lh_ragged_order): {offset, length, message index},
      // grouped by length class, so the lanes of a warp hold messages of
      // nearly equal length.  A saturated length is re-read from the layout.
      const uint4 r = __ldg(sched + t);
      i = r.w;
      off = pack(r.x, r.y);
      len = r.z;
      if (r.z == 0xFFFFFFFFu) len = lengths ? (u64)lengths[i] : offsets[i + 1] - off;
    } else if (offsets) {
      off = offsets[i];
      len = lengths ? (u64)lengths[i] : offsets[i + 1] - off;
    } else {  // fixed layout: message i = buf[i*L : (i+1)*L]
      off = i * fixed_len;
      len = fixed_len;
    }
    H h;
    init_state(h, proto, sa);
    hash_ring_any<D, WORD>(h, buf + off, len, out + i * W);
  }
}

// --------------------------------------------------------------------------
// Ragged short-message kernel (cfg3: 2^26 keys of 8..64 bytes, finalization
// dominated).  Each warp takes 32 consecutive messages.  Fast path (every
// message <= 64 B and inside the kSpanCap-byte window that starts at lane
// 0's message): the warp copies the window into shared memory with
// coalesced 16-byte loads, each thread reads its message's little-endian
// 32-bit words from it with funnel shifts (bytes past the end are never
// used unmasked), and runs two non-divergent Update slots:
//   slot 0: block 0 if the message has one;
//   slot 1: block 1 (64-byte messages) or the remainder packet (r > 0),
// so lanes of different lengths share both Updates, and the remainder's
// length injection, done in slot 1 with r_eff = r or 0 (adding 0 / rotating
// by 0 is the identity), is the only one.  Any other warp (long messages, scattered
// offsets) takes the generic per-thread path (hash_direct).
// --------------------------------------------------------------------------
constexpr u32 kSpanCap = 2048;  // bytes of a warp's span staged in smem

// Shared-memory bounds checks for the staged kernels, compiled in only for
// the A/B build LH_NVCC_EXTRA=-DLH_DEBUG_BOUNDS (compute-sanitizer is not
// available on the GPU pool): an out-of-range stage index traps the kernel,
// which the random-layout parity tests then report as a CUDA error.
#ifdef LH_DEBUG_BOUNDS
#define LH_CHECK(cond) \
  do {                 \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define LH_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// Length injection of UpdateRemainder (S/highway.py:188-197); r = 0 is a no-op.
__device__ __forceinline__ void rem_tweak(Highway& h, u32 r) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h.v0[i] = pack(lo32(h.v0[i]) + r, hi32(h.v0[i]) + r);
    h.v1[i] = pack(__funnelshift_l(lo32(h.v1[i]), lo32(h.v1[i]), r),
                   __funnelshift_l(hi32(h.v1[i]), hi32(h.v1[i]), r));
  }
}

// Reader for the groups that fail the staged fast path (a message > 64 B or
// outside the window): the register-ring reader at depth 2, 1.3-1.7x the
// direct reader on mixed short/medium keys.  Depth 1 here
// produced wrong digests for scattered offsets (a ptxas hazard like the one
// noted above; the parity tests caught it), so it is not used.
#ifndef LH_FALLBACK_DEPTH
#define LH_FALLBACK_DEPTH 2
#endif
#define LH_STAGED_FALLBACK(h, p, l, o) hash_ring_any<LH_FALLBACK_DEPTH, 16>(h, p, l, o)

#ifndef LH_SHORT_MPL
#define LH_SHORT_MPL 4
#endif
// Staging copy of a warp's window: coalesced 16-byte chunks, global -> shared.
// Asynchronous copies (LDGSTS.128: no registers, every chunk in flight at
// once, one wait); the plain LDG -> STS loop runs in batches of 8 loads, each
// batch a round trip (cfg3 1.778 -> 1.747 ms; LH_SHORT_NO_LDGSTS is the A/B knob).
#ifndef LH_SHORT_NO_LDGSTS
#define LH_STAGE_COPY(dst, src, nch, lane)                                                     \
  do {                                                                                         \
    const u32 d0_ = smem_u32(dst);                                                             \
    for (u32 c = lane; c < nch; c += 32)                                                       \
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d0_ + 16 * c),            \
                   "l"((src) + c)                                                              \
                   : "memory");                                                                \
    asm volatile("cp.async.wait_all;" ::: "memory");                                           \
  } while (0)
#else
#define LH_STAGE_COPY(dst, src, nch, lane) \
  for (u32 c = lane; c < nch; c += 32) (dst)[c] = __ldg((src) + c)
#endif
// MPL messages per lane per warp iteration (a group of 32 * MPL consecutive
// messages staged together, hashed one after another by each lane).
// (No min-blocks bound: __launch_bounds__(64, 1) alone moved ptxas to 108
// registers and cfg3 to 1.885 ms; 11..13 blocks, 1.81-1.83 ms.)
#if defined(LH_SHORT_MINB)  // A/B: a minimum-blocks bound (register cap)
#define LH_SHORT_BOUNDS __launch_bounds__(WARPS * 32, LH_SHORT_MINB)
#elif defined(LH_SHORT_MAXNREG)  // A/B: an explicit register cap
#define LH_SHORT_BOUNDS __maxnreg__(LH_SHORT_MAXNREG)
#else
#define LH_SHORT_BOUNDS __launch_bounds__(WARPS * 32)
#endif
template <int WARPS, int MPL = LH_SHORT_MPL>
__global__ void LH_SHORT_BOUNDS k_ragged_short(const Highway proto,
                                                             const uint8_t* __restrict__ buf,
                                                             const u64* __restrict__ offsets,
                                                             const u32* __restrict__ lengths,
                                                             u64 fixed_len, u64 n,
                                                             u64* __restrict__ out) {
  constexpr u32 kSpan = kSpanCap * MPL;
  __shared__ __align__(16) uint4 stage[WARPS][kSpan / 16 + 8];
  __shared__ __align__(16) ProtoSmem sp;
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = proto.width / 64;
  const u32* S = reinterpret_cast<const u32*>(&stage[warp][0]);
  const u32 s_state_a = stage_proto(proto, sp);
  __syncthreads();
  for (u64 base = ((u64)blockIdx.x * WARPS + warp) * 32 * MPL; base < n;
       base += (u64)gridDim.x * WARPS * 32 * MPL) {
    u64 start[MPL], len[MPL];
#pragma unroll
    for (int m = 0; m < MPL; ++m) {
      const u64 i = base + 32 * m + lane;
      start[m] = 0;
      len[m] = 0;
      if (i < n) {
#ifdef LH_DIAG_NOLOAD  // timing diagnostic only: synthetic layout, no metadata or payload loads
        if (offsets) {
          start[m] = i * 36;
          len[m] = 8 + (u32)(i * 7) % 57;
        } else {
#else
        if (offsets) {
          start[m] = offsets[i];
          len[m] = lengths ? (u64)lengths[i] : offsets[i + 1] - start[m];
        } else {  // fixed layout: message i = buf[i*L : (i+1)*L]
#endif
          start[m] = i * fixed_len;
          len[m] = fixed_len;
        }
      }
    }
    // Fast-path test with 32-bit warp reductions: every message lies in the
    // window [s0, s0 + kSpan) that starts at the group's first message
    // (always valid) and is at most 64 bytes.  Packed batches always pass.
    const u64 s0 = __shfl_sync(0xffffffffu, start[0], 0);
    bool fits = true;
    u32 reach = 0;
#pragma unroll
    for (int m = 0; m < MPL; ++m) {
      const bool valid = base + 32 * m + lane < n;
      fits &= !valid || (len[m] <= 64 && start[m] >= s0 && start[m] + len[m] - s0 <= kSpan);
      if (valid) reach = max(reach, (u32)(start[m] + len[m] - s0));
    }
    if (__all_sync(0xffffffffu, fits)) {
      const u32 span = __reduce_max_sync(0xffffffffu, reach);
      const u64 lo = s0, hi = s0 + span;
      // Align on the absolute address: d_buf itself need not be 16-B aligned.
      const u64 bb = (u64)(uintptr_t)buf;
      const u64 lo_al = ((bb + lo) & ~15ull) - bb, hi_al = ((bb + hi + 15) & ~15ull) - bb;
      const u32 nch = (u32)((hi_al - lo_al) >> 4);
      const uint4* src = reinterpret_cast<const uint4*>(buf + lo_al);
      LH_CHECK(nch <= kSpan / 16 + 8);
#ifndef LH_DIAG_NOLOAD
      LH_STAGE_COPY(&stage[warp][0], src, nch, lane);
#endif
      __syncwarp();
#pragma unroll 1
      for (int m = 0; m < MPL; ++m) {
        const u64 i = base + 32 * m + lane;
        if (i >= n) break;
        const u32 o = (u32)(start[m] - lo_al), a = o >> 2, sh = (o & 3) * 8;
        const u32 L = (u32)len[m];
        const u32 nfull = L >> 5, r = L & 31;
        // Word k of the message (LE; bytes past L belong to other messages).
        auto word = [&](u32 k) {
          LH_CHECK(a + k + 1 < (kSpan / 16 + 8) * 4);
          return __funnelshift_r(S[a + k], S[a + k + 1], sh);
        };
        Highway h;
        h.load_state(s_state_a, proto);
        // Slot 0: block 0 if the message has one (32..64 bytes); no tweak.
        if (nfull) {
          u32 P[8];
#pragma unroll
          for (u32 j = 0; j < 8; ++j) P[j] = word(j);
          h.update(pack(P[0], P[1]), pack(P[2], P[3]), pack(P[4], P[5]), pack(P[6], P[7]));
        }
        // Slot 1: block 1 (64 bytes) or the remainder packet (r > 0) of the
        // words from b = 8 * [nfull >= 1] on (S/highway.py:206-220): whole
        // words j < q = r/4 in place, zeros, the r%4 leftover bytes of word q
        // in word 7; a full block is q = 8 (all words, word 7 unmasked).
        // The length injection is applied with r_eff = r or 0 (identity).
        if (r || nfull == 2) {
          const u32 b = nfull ? 8u : 0u;
          const u32 q = r ? (r >> 2) : 8u;
          const u32 nleft = r ? (r & 3u) : 4u;
          u32 P[8];
#pragma unroll
          for (u32 j = 0; j < 7; ++j) P[j] = j < q ? word(b + j) : 0u;
          const u32 lft = word(b + (q < 7 ? q : 7u));
          P[7] = lft & (nleft >= 4 ? 0xffffffffu : ((1u << (8 * nleft)) - 1u));
          rem_tweak(h, r);
          h.update(pack(P[0], P[1]), pack(P[2], P[3]), pack(P[4], P[5]), pack(P[6], P[7]));
        }
        h.finalize_out(out + i * W);
      }
      __syncwarp();
    } else {
#pragma unroll 1
      for (int m = 0; m < MPL; ++m) {
        const u64 i = base + 32 * m + lane;
        if (i < n) {
          // A parameter copy here, not load_state: measured 1.78 vs 1.87 ms
          // on cfg3 (the fallback's code shape moves the fast path's
          // schedule).  Ring depth 2 here is parity-tested at rounds 0..5;
          // the ptxas hazard of DESIGN.md §10 was seen at depth 1 only.
#ifdef LH_FALLBACK_LOAD_STATE  // A/B knob
          Highway h;
          h.load_state(s_state_a, proto);
#else
          Highway h = proto;
#endif
          LH_STAGED_FALLBACK(h, buf + start[m], len[m], out + i * W);
        }
      }
    }
  }
}

template <class H>
struct IsSipHash {
  static constexpr bool value = false;
};
template <int C, int D>
struct IsSipHash<Sip<C, D>> {
  static constexpr bool value = true;
};

// SipHash-c-d of a staged group of 32 * MPL short keys (<= 64 B), for
// k_staged_any.  SipHash's cost grows with every 8-byte word and the warp
// runs each round of its lanes until the round's longest key is done, so:
//  * one flat loop over a key's whole words, then its final word -- at
//    most 9 compressions per round (8 whole words + the length word)
//    instead of absorb32 blocks plus tail words (up to 12);
//  * (SORT: ragged launches) the group's keys are first ranked by length class (8-byte classes, or 16-byte
//    ones for SipHash-1-3; invalid slots last) with warp ballots and re-dealt to
//    the rounds through shared memory, so each round's lanes hash keys of
//    similar length.  cfg3-shaped SipHash-2-4 2.45 -> 2.19 ms (flat loop)
//    -> 2.00 ms (sorted).  Fixed rows (one length) keep the flat loop: the
//    sort costs them ~13% (and a runtime "one class?" test moved the
//    schedule enough to lose most of the ragged gain: a template flag).
// Digest of key `base + slot` goes to out[base + slot] as before.
template <int WARPS, int MPL, bool SORT, int C, int D>
__device__ __forceinline__ void hash_sip_group(const Sip<C, D>& proto, const u32* S,
                                               const u64 (&start)[MPL], const u64 (&len)[MPL],
                                               u64 base, u64 n, u64 lo_al, u32 lane, u32 warp,
                                               u64* __restrict__ out) {
  constexpr u32 G = 32 * MPL;
  auto hash_one = [&](u64 st, u32 L, u64 i) {
    const u32 o = (u32)(st - lo_al), a = o >> 2, sh = (o & 3) * 8;
    auto word = [&](u32 k) { return __funnelshift_r(S[a + k], S[a + k + 1], sh); };
    SipCore<C, D> v = proto.s;
    const u32 nw = L >> 3, tb = L & 7;
    for (u32 w = 0; w < nw; ++w) v.compress(pack(word(2 * w), word(2 * w + 1)), proto.c, proto.k);
    u64 last = 0;
    if (tb) last = pack(word(2 * nw), word(2 * nw + 1)) & ((1ull << (8 * tb)) - 1);
    out[i] = v.final(last | ((u64)(L & 0xFF) << 56), proto.c, proto.d, proto.k);
  };
  if constexpr (SORT) {
    __shared__ u64 s_start[WARPS][G];
    __shared__ u32 s_len[WARPS][G];
    __shared__ uint16_t s_slot[WARPS][G];
    // Length classes of one word for 2+ rounds per word, two words for
    // SipHash-1-3 (cfg3-shaped 2-4: 1.861 -> 1.810 ms with one-word classes;
    // 1-3: 1.335 -> 1.390, the extra ballots cost more than they save).
    constexpr u32 kSortShift = C == 1 ? 4 : 3;
    constexpr u32 kSortMax = 64u >> kSortShift;  // class of a 64-byte key
    u32 cls[MPL];
#pragma unroll
    for (int m = 0; m < MPL; ++m) {
      const u32 L = (u32)len[m];
      cls[m] = base + 32 * m + lane < n ? min(L >> kSortShift, kSortMax) : kSortMax + 1;
    }
    const u32 lt = (1u << lane) - 1u;
    u32 pos[MPL], next = 0;
#pragma unroll
    for (u32 c = 0; c < kSortMax + 2; ++c) {
#pragma unroll
      for (int m = 0; m < MPL; ++m) {
        const u32 b = __ballot_sync(0xffffffffu, cls[m] == c);
        if (cls[m] == c) pos[m] = next + __popc(b & lt);
        next += __popc(b);
      }
    }
#pragma unroll
    for (int m = 0; m < MPL; ++m) {
      s_start[warp][pos[m]] = start[m];
      s_len[warp][pos[m]] = (u32)len[m];
      s_slot[warp][pos[m]] = (uint16_t)(32 * m + lane);
    }
    __syncwarp();
#pragma unroll 1
    for (int m = 0; m < MPL; ++m) {
      const u32 p = 32 * m + lane;
      const u64 i = base + s_slot[warp][p];
      if (i < n) hash_one(s_start[warp][p], s_len[warp][p], i);
    }
  } else {
    (void)warp;
#pragma unroll 1
    for (int m = 0; m < MPL; ++m) {
      const u64 i = base + 32 * m + lane;
      if (i >= n) break;
      hash_one(start[m], (u32)len[m], i);
    }
  }
}

// --------------------------------------------------------------------------
// The same warp staging for any hasher (the Sip family's short keys): the
// window of 32 * MPL messages <= 64 B is staged once, then each lane hashes
// its MPL messages one after another, reading 32-bit words from the stage
// (absorb32 per whole block, the masked tail to finish).  Hashing several
// keys per lane also evens out the per-lane work: SipHash's cost grows with
// every 8-byte word, so lanes of one key each wait for the warp's longest.
// --------------------------------------------------------------------------
template <class H, int WARPS, int MPL, bool SORT = false>
__global__ void __launch_bounds__(WARPS * 32) k_staged_any(const H proto,
                                                           const uint8_t* __restrict__ buf,
                                                           const u64* __restrict__ offsets,
                                                           const u32* __restrict__ lengths,
                                                           u64 fixed_len, u64 n,
                                                           u64* __restrict__ out) {
  constexpr u32 kSpan = kSpanCap * MPL;
  __shared__ __align__(16) uint4 stage[WARPS][kSpan / 16 + 8];
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const u32* S = reinterpret_cast<const u32*>(&stage[warp][0]);
  for (u64 base = ((u64)blockIdx.x * WARPS + warp) * 32 * MPL; base < n;
       base += (u64)gridDim.x * WARPS * 32 * MPL) {
    u64 start[MPL], len[MPL];
#pragma unroll
    for (int m = 0; m < MPL; ++m) {
      const u64 i = base + 32 * m + lane;
      start[m] = 0;
      len[m] = 0;
      if (i < n) {
        if (offsets) {
          start[m] = offsets[i];
          len[m] = lengths ? (u64)lengths[i] : offsets[i + 1] - start[m];
        } else {
          start[m] = i * fixed_len;
          len[m] = fixed_len;
        }
      }
    }
    const u64 s0 = __shfl_sync(0xffffffffu, start[0], 0);
    bool fits = true;
    u32 reach = 0;
#pragma unroll
    for (int m = 0; m < MPL; ++m) {
      const bool valid = base + 32 * m + lane < n;
      fits &= !valid || (len[m] <= 64 && start[m] >= s0 && start[m] + len[m] - s0 <= kSpan);
      if (valid) reach = max(reach, (u32)(start[m] + len[m] - s0));
    }
    if (__all_sync(0xffffffffu, fits)) {
      const u32 span = __reduce_max_sync(0xffffffffu, reach);
      const u64 bb = (u64)(uintptr_t)buf;
      const u64 lo_al = ((bb + s0) & ~15ull) - bb, hi_al = ((bb + s0 + span + 15) & ~15ull) - bb;
      const u32 nch = (u32)((hi_al - lo_al) >> 4);
      const uint4* src = reinterpret_cast<const uint4*>(buf + lo_al);
      LH_CHECK(nch <= kSpan / 16 + 8);
      // cfg3-shaped SipHash-2-4 / -1-3: 2.000 -> 1.971 / 1.457 -> 1.391 ms vs LDG -> STS
      LH_STAGE_COPY(&stage[warp][0], src, nch, lane);
      if constexpr (IsSipHash<H>::value) {
        __syncwarp();
        hash_sip_group<WARPS, MPL, SORT>(proto, S, start, len, base, n, lo_al, lane, warp, out);
        __syncwarp();
        continue;
      }
      __syncwarp();
#pragma unroll 1
      for (int m = 0; m < MPL; ++m) {
        const u64 i = base + 32 * m + lane;
        if (i >= n) break;
        const u32 o = (u32)(start[m] - lo_al), a = o >> 2, sh = (o & 3) * 8;
        const u32 L = (u32)len[m];
        auto word = [&](u32 k) {
          LH_CHECK(a + k + 1 < (kSpan / 16 + 8) * 4);
          return __funnelshift_r(S[a + k], S[a + k + 1], sh);
        };
        H h = proto;
        const u32 nb = L >> 5, r = L & 31;
        for (u32 b = 0; b < nb; ++b) {
          const u64 p[4] = {pack(word(8 * b), word(8 * b + 1)), pack(word(8 * b + 2), word(8 * b + 3)),
                            pack(word(8 * b + 4), word(8 * b + 5)),
                            pack(word(8 * b + 6), word(8 * b + 7))};
          h.absorb32(p);
        }
        u64 t[4] = {0, 0, 0, 0};
        if (r) {
#pragma unroll
          for (u32 k = 0; k < 4; ++k) t[k] = pack(word(8 * nb + 2 * k), word(8 * nb + 2 * k + 1));
          mask_tail(t, r);
        }
        h.finish(t, r, L, out + i);
      }
      __syncwarp();
    } else {
#pragma unroll 1
      for (int m = 0; m < MPL; ++m) {
        const u64 i = base + 32 * m + lane;
        if (i < n) {
          H h = proto;
          LH_STAGED_FALLBACK(h, buf + start[m], len[m], out + i);
        }
      }
    }
  }
}

// --------------------------------------------------------------------------
// TMA-staged fixed-length kernel.
// Requirements (checked on the host): len % 16 == 0, d_msgs 16-B aligned.
// Shared ring: STAGES x [ROWS rows x BOX B].  BOX = 128 (the default) uses
// the 128-byte swizzle: 16-byte unit u of row t lives at
// t*128 + ((u ^ (t & 7)) << 4); BOX = 64 the 64-byte swizzle:
// t*64 + ((u ^ ((t >> 1) & 3)) << 4).  Either way the 8 rows a quarter-warp
// reads with LDS.128 hit distinct bank groups.  64-byte boxes halve the
// bytes per stage, so an INT-bound hash (SipHash) gets twice the stages --
// more slack between its fastest and slowest consumer warp -- in the same
// shared memory.
// --------------------------------------------------------------------------

constexpr int kBoxBytes = 128;

template <int BOX>
__device__ __forceinline__ u32 swz_unit(u32 u, u32 t) {
  return BOX == 128 ? (u ^ (t & 7)) : (u ^ ((t >> 1) & 3));
}

// Rows per TMA box (boxDim <= 256): ROWS itself, else the largest divisor
// of ROWS that is a multiple of 32 and <= 256.
constexpr int tma_box_rows(int rows) {
  if (rows <= 256) return rows;
  for (int r = 256; r >= 32; r -= 32)
    if (rows % r == 0) return r;
  return 32;
}

template <int ROWS, int STAGES, int BOX = kBoxBytes>
constexpr size_t tma_smem_bytes() {
  return 1024 /*alignment slack*/ + (size_t)STAGES * ROWS * BOX + 2 * STAGES * 8;
}

// STREAM: the streaming append of whole-block chunks (lh_stream_update):
// each row starts from its StreamRec's state instead of the prototype and
// stores the state back instead of finishing; a row with a pending tail
// (not block-aligned) takes the generic append from global memory.
template <class H, int ROWS, int STAGES, int MINB, bool STREAM = false, int BOX = kBoxBytes>
__global__ void __launch_bounds__(ROWS + 32, MINB)
    k_tma_fixed(const __grid_constant__ CUtensorMap tmap, const H proto, u64 n, u64 len,
                u64* __restrict__ out, u32 pf, StreamRec<H>* __restrict__ rec,
                const uint8_t* __restrict__ chunks) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  static_assert(BOX == 128 || BOX == 64, "box width");
  constexpr u32 kStageBytes = ROWS * BOX;
  constexpr u32 kUnits = BOX / 16, kPkts = BOX / 32;  // 16-B units / packets per row-chunk
  constexpr int kConsumerWarps = ROWS / 32;
  constexpr int kBoxRowsTma = tma_box_rows(ROWS);  // TMA box rows <= 256
  constexpr int kBoxesPerStage = ROWS / kBoxRowsTma;
  uint64_t* full_bar = (uint64_t*)(smem + STAGES * kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ __align__(16) ProtoSmem sp;
  const u32 sa = stage_proto(proto, sp);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const u64 ntiles = (n + ROWS - 1) / ROWS;
  const u32 nchunks = (u32)((len + BOX - 1) / BOX);

  if (warp == kConsumerWarps) {
    // ---- producer: one elected lane streams boxes into the ring ----
    if (lane == 0) {
      tma_prefetch_desc(&tmap);
      // L2 prefetch cursor, `pf` boxes ahead of the loads: the ring is only
      // STAGES deep, so the loads themselves would expose DRAM latency.
      u64 pf_tile = blockIdx.x;
      u32 pf_c = 0;
      for (u32 k = 0; k < pf && pf_tile < ntiles; ++k) {
        for (int b = 0; b < kBoxesPerStage; ++b)
          tma_prefetch_l2_2d(&tmap, (int32_t)(pf_c * BOX),
                             (int32_t)(pf_tile * ROWS + b * kBoxRowsTma));
        if (++pf_c == nchunks) { pf_c = 0; pf_tile += gridDim.x; }
      }
      // Every message tile restarts at stage 0 (the consumers unroll over
      // stages per tile); `used` bit s = parity of the uses of stage s.
      u32 used = 0;
      for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (u32 c = 0; c < nchunks; ++c) {
          const u32 s = c % STAGES, ph = (used >> s) & 1;
          used ^= 1u << s;
          mbar_wait(&empty_bar[s], ph ^ 1);
          mbar_arrive_expect_tx(&full_bar[s], kStageBytes);
#pragma unroll
          for (int b = 0; b < kBoxesPerStage; ++b)
            tma_load_2d(smem + s * kStageBytes + b * kBoxRowsTma * BOX, &tmap,
                        (int32_t)(c * BOX), (int32_t)(tile * ROWS + b * kBoxRowsTma),
                        &full_bar[s]);
          if (pf && pf_tile < ntiles) {
            for (int b = 0; b < kBoxesPerStage; ++b)
              tma_prefetch_l2_2d(&tmap, (int32_t)(pf_c * BOX),
                                 (int32_t)(pf_tile * ROWS + b * kBoxRowsTma));
            if (++pf_c == nchunks) { pf_c = 0; pf_tile += gridDim.x; }
          }
        }
      }
    }
    return;
  }

  // ---- consumers: thread t owns message row tile*ROWS + t ----
  const u32 t = threadIdx.x;
  // Shared addresses of this thread's swizzled 16-byte units in stage 0.
  const u32 row0 = smem_u32(smem) + t * BOX;
  // Kept live in registers (opaque to ptxas, which would otherwise recompute
  // them per chunk); the stage offset is folded into LDS immediates below.
  u32 ua[kUnits];
#pragma unroll
  for (u32 u = 0; u < kUnits; ++u)
    asm volatile("mov.b32 %0, %1;" : "=r"(ua[u]) : "r"(row0 + (swz_unit<BOX>(u, t) << 4)));
  const int W = nout(proto);
  const u64 nfull = len >> 5;
  const u32 r = (u32)(len & 31);  // 0 or 16
  // Each message tile starts at stage 0 and the chunk loop is unrolled over
  // the STAGES ring slots, so in each copy the stage -- its barriers and LDS
  // offsets -- is a compile-time constant; `used` bit s is the parity of
  // stage s's uses (a tile whose chunk count is not a multiple of STAGES
  // leaves the last slots of its final round unused).  Per chunk: one
  // wait, one compare, the arrive and a bit flip; the message epilogue is a
  // single copy outside the unrolled body (I-cache: the Sip bodies are big).
  const u32 nfull4 = (u32)(nfull / kPkts);  // chunks that hold kPkts whole packets
  u32 bars;  // shared address of full_bar[0]; empty_bar[s] = bars + 8 * (STAGES + s)
  asm volatile("mov.b32 %0, %1;" : "=r"(bars) : "r"(smem_u32(full_bar)));
  u32 used = 0;
  for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const u64 row_idx = tile * ROWS + t;
    H h;
    init_state(h, proto, sa);
    bool fast = true;
    if constexpr (STREAM) {
      if (row_idx < n) {
        h = rec[row_idx].h;
        fast = rec[row_idx].tlen == 0;
      }
    }
    u64 tl[4] = {0, 0, 0, 0};
    for (u32 cb = 0; cb < nchunks; cb += STAGES) {
#pragma unroll
      for (u32 ss = 0; ss < (u32)STAGES; ++ss) {
        const u32 c = cb + ss;
        if (c < nchunks) {
          mbar_wait_addr(bars + 8 * ss, (used >> ss) & 1);
          used ^= 1u << ss;
          if (c < nfull4) {
#pragma unroll
            for (u32 k = 0; k < kPkts; ++k) {
              const uint4 a = lds128(ua[2 * k] + ss * kStageBytes);
              const uint4 b = lds128(ua[2 * k + 1] + ss * kStageBytes);
              const u64 p[4] = {pack(a.x, a.y), pack(a.z, a.w), pack(b.x, b.y), pack(b.z, b.w)};
              if (!STREAM || fast) h.absorb32(p);
            }
          } else {
            // Last chunk of a message whose length is not a multiple of
            // BOX: 0..kPkts-1 whole packets, then the 16-byte tail if r != 0.
            const u32 kvalid = (u32)(nfull - (u64)kPkts * c);
            const u32 rowa = row0 + ss * kStageBytes;
            for (u32 k = 0; k < kvalid; ++k) {
              const uint4 a = lds128(rowa + (swz_unit<BOX>(2 * k, t) << 4));
              const uint4 b = lds128(rowa + (swz_unit<BOX>(2 * k + 1, t) << 4));
              const u64 p[4] = {pack(a.x, a.y), pack(a.z, a.w), pack(b.x, b.y), pack(b.z, b.w)};
              if (!STREAM || fast) h.absorb32(p);
            }
            if (r) {
              const uint4 a = lds128(rowa + (swz_unit<BOX>(2 * kvalid, t) << 4));
              tl[0] = pack(a.x, a.y);
              tl[1] = pack(a.z, a.w);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_addr(bars + 8 * (STAGES + ss));
        }
      }
    }
    if constexpr (STREAM) {
      if (row_idx < n) {
        if (fast) {
          rec[row_idx].h = h;
          rec[row_idx].total += len;
        } else {
          StreamRec<H> rr = rec[row_idx];
          stream_append<false>(rr, chunks + row_idx * len, len);
          rec[row_idx] = rr;
        }
      }
    } else {
      if (row_idx < n) h.finish(tl, r, len, out + row_idx * W);
    }
  }
}

// --------------------------------------------------------------------------
// Long-message kernel: the HighwayHash state of each message is split over a
// thread pair (lh::HighwayHalf), so a batch of few long messages fills twice
// as many warps (cfg4: 16,384 x 1 MiB = 1,024 warps instead of 512).
// One warp per CTA = 16 messages.  Requirements: len % 128 == 0, 16-B
// aligned base.  The byte matrix is viewed as a 3-D tensor
// {128 B, n rows, len/128 chunks}; one TMA box = 16 rows x CH chunks
// (16 x 512 B = 8 KiB for CH = 4), laid out [chunk][row][128 B] with the
// 128-byte swizzle, into a STAGES-deep ring refilled by lane 0 as soon as
// the warp has consumed a stage.  Half 0 of row r reads unit 2k of packet
// k, half 1 unit 2k+1; the lane -> row map keeps each quarter-warp's
// units in distinct banks.
// --------------------------------------------------------------------------
constexpr int kSplitRows = 16;

template <int STAGES, int CH>
constexpr size_t split_smem_bytes() {
  return 1024 + (size_t)STAGES * kSplitRows * CH * kBoxBytes + STAGES * 8;
}

// STREAM: the streaming append of whole-block chunks (as k_tma_fixed's):
// each half starts from its lanes of the message's StreamRec state and
// writes them back; a row with a pending tail skips the staged data and its
// half 0 runs the generic append from global memory.
template <int STAGES, int CH, int MINB, bool STREAM = false>
__global__ void __launch_bounds__(32, MINB)
    k_tma_split(const __grid_constant__ CUtensorMap tmap, const Highway proto, u64 n, u64 len,
                u64* __restrict__ out, StreamRec<Highway>* __restrict__ rec = nullptr,
                const uint8_t* __restrict__ chunks = nullptr) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr u32 kChunk = kSplitRows * kBoxBytes;  // 2 KiB: one 128-B chunk of 16 rows
  constexpr u32 kStage = CH * kChunk;
  uint64_t* bar = (uint64_t*)(smem + STAGES * kStage);
  // Lane -> row: each quarter-warp (8 lanes) takes rows whose swizzle
  // patterns r & 7 differ in bits 1-2 (rows 0,2,4,6 / 1,3,5,7 / 8,10,.. /
  // 9,11,..), so the 8 LDS.128 units it reads per packet are distinct banks.
  const u32 lane = threadIdx.x & 31, half = lane & 1;
  const u32 row = ((lane >> 1) & 3) * 2 + ((lane >> 3) & 1) + (lane >> 4) * 8, sw = row & 7;

  const u64 ntiles = (n + kSplitRows - 1) / kSplitRows;
  const u32 nch = (u32)(len / kBoxBytes);
  const u32 nst = (nch + CH - 1) / CH;  // stages per tile
  const u64 g = blockIdx.x, G = gridDim.x;
  const u64 my_tiles = g < ntiles ? (ntiles - g + G - 1) / G : 0;
  const u64 total = my_tiles * nst;

  __shared__ __align__(16) ProtoSmem sp;
  const u32 sa = stage_proto(proto, sp);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmap);
  }
  __syncwarp();
  u64 it_tile = g;
  u32 it_st = 0;
  auto issue_next = [&](u32 s) {
    mbar_arrive_expect_tx(&bar[s], kStage);
    tma_load_3d(smem + s * kStage, &tmap, 0, (int32_t)(it_tile * kSplitRows),
                (int32_t)(it_st * CH), &bar[s]);
    if (++it_st == nst) {
      it_st = 0;
      it_tile += G;
    }
  };
  if (lane == 0)
    for (u32 s = 0; s < (u32)STAGES && s < total; ++s) issue_next(s);

  u32 ua[4];
#pragma unroll
  for (u32 k = 0; k < 4; ++k)
    asm volatile("mov.b32 %0, %1;"
                 : "=r"(ua[k])
                 : "r"(smem_u32(smem) + row * kBoxBytes + (((2 * k + half) ^ sw) << 4)));

  const int W = proto.width / 64;
  HighwayHalf h;
  bool fast = true;
  // Row state at the start of a tile: the prototype, or (STREAM) the record.
  auto start_row = [&](u64 tl) {
    const u64 m = tl * kSplitRows + row;
    if constexpr (STREAM) {
      fast = true;
      if (m < n) {
        h.init(rec[m].h, half);
        fast = rec[m].tlen == 0;
      } else {
        h.load_state(sa, proto, half);
      }
    } else {
      h.load_state(sa, proto, half);
    }
  };
  u64 tile = g;
  start_row(tile);
  u32 st = 0, s = 0, ph = 0;
  for (u64 i = 0; i < total; ++i) {
    mbar_wait(&bar[s], ph);
    const u32 nvalid = (nch - st * CH) < (u32)CH ? (nch - st * CH) : (u32)CH;
    if (nvalid == (u32)CH) {
#pragma unroll
      for (u32 ss = 0; ss < (u32)STAGES; ++ss) {
        if (s == ss) {
#pragma unroll
          for (u32 c = 0; c < (u32)CH; ++c)
#pragma unroll
            for (u32 k = 0; k < 4; ++k) {
              const uint4 a = lds128(ua[k] + ss * kStage + c * kChunk);
              if (!STREAM || fast) h.update(pack(a.x, a.y), pack(a.z, a.w));
            }
        }
      }
    } else {
      for (u32 c = 0; c < nvalid; ++c)
#pragma unroll
        for (u32 k = 0; k < 4; ++k) {
          const uint4 a = lds128(ua[k] + s * kStage + c * kChunk);
          if (!STREAM || fast) h.update(pack(a.x, a.y), pack(a.z, a.w));
        }
    }
    __syncwarp();
    if (lane == 0 && i + STAGES < total) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_next(s);
    }
    if (++s == (u32)STAGES) {
      s = 0;
      ph ^= 1;
    }
    if (++st == nst) {
      const u64 m = tile * kSplitRows + row;
      if constexpr (STREAM) {
        if (m < n) {
          if (fast) {
            h.save(rec[m].h);
            if (half == 0) rec[m].total += len;
          } else if (half == 0) {
            StreamRec<Highway> rr = rec[m];
            stream_append<false>(rr, chunks + m * len, len);
            rec[m] = rr;
          }
        }
      } else {
        h.finalize_rounds();  // whole warp: shuffles between the halves
        if (m < n) h.store(out + m * W);
      }
      st = 0;
      tile += G;
      start_row(tile);
    }
  }
}

// --------------------------------------------------------------------------
// Host helpers
// --------------------------------------------------------------------------

// Status of the launch just issued.  The library links the CUDA runtime
// statically, so the "last error" cudaGetLastError reads and clears is this
// library's own (per host thread): it cannot consume a launch error that
// belongs to the caller's runtime (PyTorch's, say).  A sticky context error
// (an earlier kernel's illegal address) is not cleared by it and keeps
// failing every CUDA call of every runtime in the process, this one's too.
int cuda_err(cudaError_t e) { return e == cudaSuccess ? LH_OK : LH_ECUDA; }

// The device checks run on every call; the SM count and the compute
// capability are cached per device ordinal (idempotent writes, so racing
// first calls from several host threads agree).
int check_device(int* sms) {
  static int cache[128];  // 0 = not yet queried, -1 = unusable, else the SM count
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return LH_ENODEV;
  int v = (dev >= 0 && dev < 128) ? __atomic_load_n(&cache[dev], __ATOMIC_RELAXED) : 0;
  if (v == 0) {
    int major = 0, minor = 0, count = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return LH_ENODEV;
    // The library carries sm_100a SASS only (no PTX): anything but CC 10.0
    // could not run it, so report LH_ENODEV instead of failing each launch.
    v = (major != 10 || minor != 0 || count < 1) ? -1 : count;
    if (dev >= 0 && dev < 128) __atomic_store_n(&cache[dev], v, __ATOMIC_RELAXED);
  }
  if (v < 0) return LH_ENODEV;
  if (sms) *sms = v;
  return LH_OK;
}

// cudaFuncSetAttribute (dynamic shared memory) + the occupancy query, once
// per (kernel, device): both are host round trips that small launch-bound
// batches would otherwise pay on every call.
int prepare_kernel(const void* kern, int threads, size_t smem, int* per_sm) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return LH_ENODEV;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find({kern, dev});
    if (it != cache.end()) {
      *per_sm = it->second;
      return LH_OK;
    }
  }
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return LH_ECUDA;
  int v = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, threads, smem) != cudaSuccess ||
      v < 1)
    return LH_ECUDA;
  std::lock_guard<std::mutex> g(mu);
  cache[{kern, dev}] = v;
  *per_sm = v;
  return LH_OK;
}

unsigned grid_for(u64 n, int threads, int sms) {
  const u64 blocks = (n + threads - 1) / threads;
  const u64 cap = (u64)sms * 64;  // grid-stride beyond 64 waves' worth
  return (unsigned)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

// Process-wide settings are function-local statics initialised once by a
// lambda (thread-safe under C++11): host threads driving several devices
// (multi.py) may make their first calls concurrently.
u32 tma_l2_prefetch() {
  static const u32 pf = [] {
    const char* s = getenv("LH_TMA_PF");
    const int v = s ? atoi(s) : 0;
    return (u32)(v < 0 ? 0 : v);
  }();
  return pf;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000)p;
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}

template <class H>
int launch_direct(const H& proto, const uint8_t* buf, const u64* offsets, const u32* lengths,
                  u64 fixed_len, u64 n, u64* out, cudaStream_t st) {
  int sms = 0;
  int rc = check_device(&sms);
  if (rc) return rc;
  if (n == 0) return LH_OK;
  if (offsets || fixed_len >= 64)
    k_direct<H, true><<<grid_for(n, 256, sms), 256, 0, st>>>(proto, buf, offsets, lengths,
                                                             fixed_len, n, out);
  else
    k_direct<H, false><<<grid_for(n, 256, sms), 256, 0, st>>>(proto, buf, offsets, lengths,
                                                              fixed_len, n, out);
  return cuda_err(cudaGetLastError());
}

// Register-ring reader for ragged batches of medium/long messages
// (LH_KERNEL_DIRECT on the ragged entry points).
#ifndef LH_RING_DEPTH
#define LH_RING_DEPTH 2
#endif
constexpr int kRingDepth = LH_RING_DEPTH;
#ifndef LH_ALLOW_DEPTH1  // A/B builds only (tools/ring_depth1.sh)
static_assert(kRingDepth >= 2 && LH_FALLBACK_DEPTH >= 2,
              "ring depth 1 is not used (DESIGN.md §10)");
#endif

template <class H>
int launch_ring(const H& proto, const uint8_t* buf, const u64* offsets, const u32* lengths,
                u64 fixed_len, u64 n, u64* out, cudaStream_t st, const uint4* order = nullptr) {
  int sms = 0;
  int rc = check_device(&sms);
  if (rc) return rc;
  if (n == 0) return LH_OK;
  // 16-byte word loads for every hash (scripts/ring_word_ab.py): 4- and
  // 8-byte per-lane loads of messages a power-of-two apart (256 B, 4 KiB
  // records) ran 2-3.5x slower; 16-byte loads cost 1-6% on random lengths.
  // Ring depth: 2 for HighwayHash (equal or better than 4 everywhere), 4 for
  // Sip (short keys need it: cfg3-shaped SipHash-2-4 2.85 ms vs 3.09).
  const unsigned grid = grid_for(n, 128, sms);
  if constexpr (std::is_same<H, Highway>::value)
    k_ragged_ring<H, kRingDepth, 16><<<grid, 128, 0, st>>>(proto, buf, offsets, lengths,
                                                             fixed_len, n, out, order);
  else
    k_ragged_ring<H, 4, 16><<<grid, 128, 0, st>>>(proto, buf, offsets, lengths, fixed_len, n,
                                                    out, order);
  return cuda_err(cudaGetLastError());
}

// Warp-staged short-key kernel (HighwayHash only), ragged or fixed layout.
int launch_staged(const Highway& proto, const uint8_t* buf, const u64* offsets,
                  const u32* lengths, u64 fixed_len, u64 n, u64* out, cudaStream_t st) {
  int sms = 0;
  int rc = check_device(&sms);
  if (rc) return rc;
  if (n == 0) return LH_OK;
  // 2 warps per block of 4 messages per lane (cfg3: MPL 1 / 4 warps 1.900 ms,
  // MPL 2 1.859, MPL 4 1.805, MPL 4 / 2 warps 1.784, MPL 8 2.17).
  constexpr int kWarps = 2;
  const u64 warps = (n + 32 * LH_SHORT_MPL - 1) / (32 * LH_SHORT_MPL);
  const u64 cap = (u64)sms * 8 * (64 / kWarps);
  const u64 blocks = (warps + kWarps - 1) / kWarps;
  k_ragged_short<kWarps><<<(unsigned)(blocks < cap ? blocks : cap), kWarps * 32, 0, st>>>(
      proto, buf, offsets, lengths, fixed_len, n, out);
  return cuda_err(cudaGetLastError());
}

#ifndef LH_ANY_MPL
#define LH_ANY_MPL 4
#endif
// Warp-staged short keys for the Sip family (one digest word per message).
template <class H>
int launch_staged_any(const H& proto, const uint8_t* buf, const u64* offsets, const u32* lengths,
                      u64 fixed_len, u64 n, u64* out, cudaStream_t st) {
  int sms = 0;
  int rc = check_device(&sms);
  if (rc) return rc;
  if (n == 0) return LH_OK;
  constexpr int kWarps = 2, kMpl = LH_ANY_MPL;
  const u64 warps = (n + 32 * kMpl - 1) / (32 * kMpl);
  const u64 cap = (u64)sms * 256;
  const u64 blocks = (warps + kWarps - 1) / kWarps;
  const unsigned grid = (unsigned)(blocks < cap ? blocks : cap);
  if (offsets && IsSipHash<H>::value)  // ragged SipHash: length-sorted rounds
    k_staged_any<H, kWarps, kMpl, true><<<grid, kWarps * 32, 0, st>>>(proto, buf, offsets,
                                                                        lengths, fixed_len, n,
                                                                        out);
  else
    k_staged_any<H, kWarps, kMpl><<<grid, kWarps * 32, 0, st>>>(proto, buf, offsets, lengths,
                                                                fixed_len, n, out);
  return cuda_err(cudaGetLastError());
}

template <class H, int ROWS, int STAGES, int MINB, bool STREAM = false, int BOX = kBoxBytes>
int launch_tma_cfg(const H& proto, const uint8_t* msgs, u64 n, u64 len, u64* out,
                   cudaStream_t st, int sms, StreamRec<H>* rec = nullptr) {
  auto enc = get_encode();
  if (!enc) return LH_ECUDA;
  constexpr size_t smem = tma_smem_bytes<ROWS, STAGES, BOX>();
  auto kern = k_tma_fixed<H, ROWS, STAGES, MINB, STREAM, BOX>;
  int per_sm = 0;
  const int prc = prepare_kernel((const void*)kern, ROWS + 32, smem, &per_sm);
  if (prc) return prc;
  // Rows are split into segments of < 2^31 (TMA coordinates are int32).
  const u64 kSeg = 1ull << 30;
  const int W = nout(proto);
  for (u64 base = 0; base < n; base += kSeg) {
    const u64 nn = n - base < kSeg ? n - base : kSeg;
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)len, (cuuint64_t)nn};
    cuuint64_t strides[1] = {(cuuint64_t)len};
    cuuint32_t box[2] = {(cuuint32_t)BOX, (cuuint32_t)tma_box_rows(ROWS)};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)(msgs + base * len), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      BOX == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return LH_ECUDA;
    const u64 tiles = (nn + ROWS - 1) / ROWS;
    const u64 cap = (u64)sms * per_sm;
    const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
    kern<<<grid, ROWS + 32, smem, st>>>(map, proto, nn, len, STREAM ? out : out + base * W,
                                        tma_l2_prefetch(), STREAM ? rec + base : nullptr,
                                        msgs + base * len);
    int rc = cuda_err(cudaGetLastError());
    if (rc) return rc;
  }
  return LH_OK;
}

template <bool STREAM = false>
int launch_split(const Highway& proto, const uint8_t* msgs, u64 n, u64 len, u64* out,
                 cudaStream_t st, StreamRec<Highway>* rec = nullptr) {
  constexpr int STAGES = 3, CH = 4, MINB = 8;
  int sms = 0;
  int rc = check_device(&sms);
  if (rc) return rc;
  if (n == 0) return LH_OK;
  auto enc = get_encode();
  if (!enc) return LH_ECUDA;
  constexpr size_t smem = split_smem_bytes<STAGES, CH>();
  auto kern = k_tma_split<STAGES, CH, MINB, STREAM>;
  int per_sm = 0;
  rc = prepare_kernel((const void*)kern, 32, smem, &per_sm);
  if (rc) return rc;
  const u64 kSeg = 1ull << 30;
  const int W = proto.width / 64;
  for (u64 base = 0; base < n; base += kSeg) {
    const u64 nn = n - base < kSeg ? n - base : kSeg;
    CUtensorMap map;
    cuuint64_t dims[3] = {(cuuint64_t)kBoxBytes, (cuuint64_t)nn, (cuuint64_t)(len / kBoxBytes)};
    cuuint64_t strides[2] = {(cuuint64_t)len, (cuuint64_t)kBoxBytes};
    cuuint32_t box[3] = {(cuuint32_t)kBoxBytes, (cuuint32_t)kSplitRows, (cuuint32_t)CH};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)(msgs + base * len), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return LH_ECUDA;
    const u64 tiles = (nn + kSplitRows - 1) / kSplitRows;
    const u64 cap = (u64)sms * per_sm;
    const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
    kern<<<grid, 32, smem, st>>>(map, proto, nn, len, STREAM ? out : out + base * W,
                                 STREAM ? rec + base : nullptr, msgs + base * len);
    rc = cuda_err(cudaGetLastError());
    if (rc) return rc;
  }
  return LH_OK;
}

bool split_ok(const uint8_t* msgs, u64 n, u64 len) {
  return n > 0 && len >= 128 && len % 128 == 0 && ((uintptr_t)msgs % 16) == 0 &&
         len / 128 < (1ull << 31);
}

// Tuning knobs (read once): LH_TMA_CFG=128x4|256x3|512x3|128x3 tile shape,
// LH_TMA_PF=<boxes> L2 prefetch distance.  Defaults: automatic.
int tma_cfg_override() {
  static const int cfg = [] {
    const char* s = getenv("LH_TMA_CFG");
    if (!s) return 0;
    if (!strcmp(s, "128x4")) return 1;
    if (!strcmp(s, "256x3")) return 2;
    if (!strcmp(s, "512x3")) return 3;
    if (!strcmp(s, "128x3")) return 4;
    if (!strcmp(s, "384x4")) return 5;
    if (!strcmp(s, "320x5")) return 6;
    if (!strcmp(s, "448x3")) return 7;
    if (!strcmp(s, "512x6b64")) return 8;
    if (!strcmp(s, "256x6b64")) return 9;
    if (!strcmp(s, "512x5b64")) return 10;
    if (!strcmp(s, "512x3b64m2")) return 11;
    if (!strcmp(s, "480x3b64m2")) return 12;
    if (!strcmp(s, "512x4b64")) return 13;
    return 0;
  }();
  return cfg;
}

template <class H>
int launch_tma(const H& proto, const uint8_t* msgs, u64 n, u64 len, u64* out, cudaStream_t st) {
  int sms = 0;
  int rc = check_device(&sms);
  if (rc) return rc;
  if (n == 0) return LH_OK;
  switch (tma_cfg_override()) {
    case 1: return launch_tma_cfg<H, 128, 4, 3>(proto, msgs, n, len, out, st, sms);
    case 2: return launch_tma_cfg<H, 256, 3, 2>(proto, msgs, n, len, out, st, sms);
    case 3: return launch_tma_cfg<H, 512, 3, 1>(proto, msgs, n, len, out, st, sms);
    case 5: return launch_tma_cfg<H, 384, 4, 1>(proto, msgs, n, len, out, st, sms);
    case 6: return launch_tma_cfg<H, 320, 5, 1>(proto, msgs, n, len, out, st, sms);
    case 7: return launch_tma_cfg<H, 448, 3, 1>(proto, msgs, n, len, out, st, sms);
    case 4: return launch_tma_cfg<H, 128, 3, 4>(proto, msgs, n, len, out, st, sms);
    case 8: return launch_tma_cfg<H, 512, 6, 1, false, 64>(proto, msgs, n, len, out, st, sms);
    case 9: return launch_tma_cfg<H, 256, 6, 2, false, 64>(proto, msgs, n, len, out, st, sms);
    case 10: return launch_tma_cfg<H, 512, 5, 1, false, 64>(proto, msgs, n, len, out, st, sms);
    case 11: return launch_tma_cfg<H, 512, 3, 2, false, 64>(proto, msgs, n, len, out, st, sms);
    case 12: return launch_tma_cfg<H, 480, 3, 2, false, 64>(proto, msgs, n, len, out, st, sms);
    case 13: return launch_tma_cfg<H, 512, 4, 1, false, 64>(proto, msgs, n, len, out, st, sms);
    default: break;
  }
  // One 512-row CTA per SM (16 consumer warps sharing a 3 x 64 KiB ring)
  // measured fastest for large batches (profiles/README.md); smaller batches
  // use smaller tiles so every SM gets several, and few-but-long messages
  // use 32-row tiles to spread over as many SMs as possible.
  if (n >= (u64)sms * 512 * 8) return launch_tma_cfg<H, 512, 3, 1>(proto, msgs, n, len, out, st, sms);
  if (n >= (u64)sms * 128 * 3 * 4)
    return launch_tma_cfg<H, 128, 4, 3>(proto, msgs, n, len, out, st, sms);
  return launch_tma_cfg<H, 32, 8, 4>(proto, msgs, n, len, out, st, sms);
}

bool tma_ok(const uint8_t* msgs, u64 n, u64 len) {
  return len >= 32 && (len % 16) == 0 && ((uintptr_t)msgs % 16) == 0 && len < (1ull << 31) &&
         n > 0;
}

template <class H>
int dispatch_split(const H&, const uint8_t*, u64, u64, u64*, cudaStream_t) {
  return LH_EINVAL;  // only HighwayHash has a split-state kernel
}
template <>
int dispatch_split<Highway>(const Highway& proto, const uint8_t* msgs, u64 n, u64 len, u64* out,
                            cudaStream_t st) {
  if (!split_ok(msgs, n, len)) return LH_EINVAL;
  return launch_split(proto, msgs, n, len, out, st);
}

template <class H>
bool prefer_split(const H&, const uint8_t*, u64, u64) {
  return false;
}
template <>
bool prefer_split<Highway>(const Highway&, const uint8_t* msgs, u64 n, u64 len) {
  int sms = 148;
  check_device(&sms);
  // Few long messages: one thread per message would leave SMs idle; and
  // small-to-medium batches are latency-bound, where halving each thread's
  // Update chain wins (profiles/README.md: 131,072 x 1 KiB 29 us vs 52 us).
  return split_ok(msgs, n, len) &&
         ((len >= 4096 && n < (u64)sms * 256) || (len >= 512 && n < (u64)sms * 1024));
}

template <class H>
int dispatch_staged(const H& proto, const uint8_t* msgs, u64 n, u64 len, u64* out,
                    cudaStream_t st) {
  return launch_staged_any(proto, msgs, nullptr, nullptr, len, n, out, st);
}
template <>
int dispatch_staged<Highway>(const Highway& proto, const uint8_t* msgs, u64 n, u64 len, u64* out,
                             cudaStream_t st) {
  return launch_staged(proto, msgs, nullptr, nullptr, len, n, out, st);
}

// Fixed-length batches the TMA kernel does not take: rows whose length is
// not a multiple of 16 (so rows start at every alignment), or fewer than
// 1,024 rows (latency-bound).  Measured (scripts/untiled_ab.py, DESIGN.md
// §9): unaligned rows go to the register ring (HighwayHash 1.2-1.8x, Sip
// 1.4-2.2x the direct reader, whose alignment branches diverge); HighwayHash
// rows of <= 64 bytes to the warp-staged kernel; 16-byte-multiple rows of a
// small batch keep the direct reader (16-byte loads, next-packet prefetch).
template <class H>
int dispatch_untiled(const H& proto, const uint8_t* msgs, u64 n, u64 len, u64* out,
                     cudaStream_t st) {
  if (len > 32 && len % 16) return launch_ring(proto, msgs, nullptr, nullptr, len, n, out, st);
  return launch_direct(proto, msgs, nullptr, nullptr, len, n, out, st);
}
template <>
int dispatch_untiled<Highway>(const Highway& proto, const uint8_t* msgs, u64 n, u64 len, u64* out,
                              cudaStream_t st) {
  if (len <= 64) return launch_staged(proto, msgs, nullptr, nullptr, len, n, out, st);
  if (len % 16) return launch_ring(proto, msgs, nullptr, nullptr, len, n, out, st);
  return launch_direct(proto, msgs, nullptr, nullptr, len, n, out, st);
}

// SipHash (not SipTree) rows of 64..127 bytes (shorter ones go to the
// warp-staged kernel first, see SipFamily below): the register-ring
// kernel beats the TMA ring by 8-25% (scripts/untiled_ab.py-style sweep,
// SipHash-1-3 at 64 B 0.414 vs 0.522 ms per GiB); from 128 B,
// and for SipTree at every length, the TMA kernel is faster.
template <class H>
struct ShortRowsToRing {
  static constexpr bool value = false;
};
template <int C, int D>
struct ShortRowsToRing<Sip<C, D>> {
  static constexpr bool value = true;
};

// Sip-family rows of 12..63 bytes: the warp-staged kernel (4 keys per lane)
// beats the direct reader, the ring and, for SipHash, the TMA kernel by
// 5-17%; SipTree rows TMA can take stay on TMA (48 B: 0.79 vs 0.83 ms/GiB).
template <class H>
struct SipFamily {
  static constexpr int value = 0;
};
template <int C, int D>
struct SipFamily<Sip<C, D>> {
  static constexpr int value = 1;
};
template <int C, int D>
struct SipFamily<SipTree<C, D>> {
  static constexpr int value = 2;
};

template <class H>
int dispatch_fixed(const H& proto, const uint8_t* msgs, u64 n, u64 len, u64* out,
                   cudaStream_t st, int kernel) {
  if (kernel == LH_KERNEL_SPLIT) return n ? dispatch_split(proto, msgs, n, len, out, st) : LH_OK;
  if (kernel == LH_KERNEL_AUTO && prefer_split(proto, msgs, n, len))
    return dispatch_split(proto, msgs, n, len, out, st);
  if (kernel == LH_KERNEL_TMA) {
    if (n && !tma_ok(msgs, n, len)) return LH_EINVAL;
    return launch_tma(proto, msgs, n, len, out, st);
  }
  if (kernel == LH_KERNEL_RING) return launch_ring(proto, msgs, nullptr, nullptr, len, n, out, st);
  if (kernel == LH_KERNEL_STAGED) return dispatch_staged(proto, msgs, n, len, out, st);
  if (kernel == LH_KERNEL_AUTO && SipFamily<H>::value && len >= 12 && len <= 63 && n >= 1024 &&
      !(SipFamily<H>::value == 2 && tma_ok(msgs, n, len)))
    return launch_staged_any(proto, msgs, nullptr, nullptr, len, n, out, st);
  if (kernel == LH_KERNEL_AUTO && ShortRowsToRing<H>::value && len >= 32 && len < 128 &&
      n >= 1024)
    return launch_ring(proto, msgs, nullptr, nullptr, len, n, out, st);
  if (kernel == LH_KERNEL_AUTO && tma_ok(msgs, n, len) && n >= 1024)
    return launch_tma(proto, msgs, n, len, out, st);
  if (kernel == LH_KERNEL_AUTO) return dispatch_untiled(proto, msgs, n, len, out, st);
  return launch_direct(proto, msgs, nullptr, nullptr, len, n, out, st);
}

bool valid_width(int w) { return w == 64 || w == 128 || w == 256; }

template <class H>
int sip_dispatch_ragged(const H& h, const uint8_t* buf, const u64* off, const u32* lens, u64 n,
                        u64* out, cudaStream_t st, bool staged = false,
                        const uint4* order = nullptr) {
  if (order) return launch_ring(h, buf, off, lens, 0, n, out, st, order);
  if (staged) return launch_staged_any(h, buf, off, lens, 0, n, out, st);
  // The register-ring reader is the Sip ragged kernel at every length: its
  // alignment-branch-free word reads beat the prefetching direct reader even
  // on short keys (cfg3-shaped SipHash-2-4: 2.86 vs 3.91 ms).
  return launch_ring(h, buf, off, lens, 0, n, out, st);
}

template <class H>
int launch_tma_stream(StreamRec<H>* rec, const uint8_t* chunks, u64 n, u64 len,
                      cudaStream_t st) {
  int sms = 0;
  int rc = check_device(&sms);
  if (rc) return rc;
  H proto;
  memset(&proto, 0, sizeof proto);  // unused: every row starts from its record
  if (n >= (u64)sms * 512 * 8)
    return launch_tma_cfg<H, 512, 3, 1, true>(proto, chunks, n, len, nullptr, st, sms, rec);
  return launch_tma_cfg<H, 128, 4, 3, true>(proto, chunks, n, len, nullptr, st, sms, rec);
}


}  // namespace
