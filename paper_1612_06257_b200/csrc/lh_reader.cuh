// lh_reader.cuh — direct global-memory message reader (any alignment).
//
// Only 8-byte-aligned words that contain at least one message byte are
// read, so no access leaves the message's own aligned words (safe at the end
// of an allocation).  Blocks are 32-byte packets as 4 little-endian u64.
#pragma once
#include <stdint.h>

#include "lh_device.cuh"

namespace lh {

__device__ __forceinline__ u64 ldg64(const u64* p) { return __ldg((const unsigned long long*)p); }

// Bytes of the 16-byte window a|b starting at byte sh/8 (sh in 8..56).
__device__ __forceinline__ u64 funnel(u64 a, u64 b, u32 sh) {
  return (a >> sh) | (b << (64 - sh));
}

// Zero every byte at index >= r of the 32-byte value t.
__device__ __forceinline__ void mask_tail(u64 (&t)[4], u32 r) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int keep = (int)r - 8 * k;
    const u64 m = keep >= 8 ? ~0ull : (keep <= 0 ? 0ull : ((1ull << (8 * keep)) - 1));
    t[k] &= m;
  }
}

// Absorb nb full 32-byte blocks starting at p.
template <class H>
__device__ __forceinline__ void absorb_blocks(H& h, const uint8_t* p, u64 nb) {
  if (!nb) return;
  const uintptr_t a = (uintptr_t)p;
  const u32 sh = (u32)(a & 7) * 8;
  const u64* w = (const u64*)(a & ~(uintptr_t)7);
  if (sh == 0) {
    if ((a & 15) == 0) {
      const ulonglong2* w2 = (const ulonglong2*)w;
      for (u64 b = 0; b < nb; ++b) {
        const ulonglong2 x = __ldg(w2 + 2 * b);
        const ulonglong2 y = __ldg(w2 + 2 * b + 1);
        const u64 pk[4] = {x.x, x.y, y.x, y.y};
        h.absorb32(pk);
      }
    } else {
      for (u64 b = 0; b < nb; ++b) {
        const u64 pk[4] = {ldg64(w + 4 * b), ldg64(w + 4 * b + 1), ldg64(w + 4 * b + 2),
                           ldg64(w + 4 * b + 3)};
        h.absorb32(pk);
      }
    }
  } else {
    u64 cur = ldg64(w);
    for (u64 b = 0; b < nb; ++b) {
      const u64* q = w + 4 * b;
      const u64 n0 = ldg64(q + 1), n1 = ldg64(q + 2), n2 = ldg64(q + 3), n3 = ldg64(q + 4);
      const u64 pk[4] = {funnel(cur, n0, sh), funnel(n0, n1, sh), funnel(n1, n2, sh),
                         funnel(n2, n3, sh)};
      cur = n3;
      h.absorb32(pk);
    }
  }
}

// The r (0..31) bytes at p as 4 LE words, zero beyond r.
__device__ __forceinline__ void load_tail(const uint8_t* p, u32 r, u64 (&t)[4]) {
  t[0] = t[1] = t[2] = t[3] = 0;
  if (!r) return;
  const uintptr_t a = (uintptr_t)p;
  const u32 sh = (u32)(a & 7) * 8;
  const u64* w = (const u64*)(a & ~(uintptr_t)7);
  const u32 nw = (u32)(((a + r - 1) >> 3) - (a >> 3)) + 1;  // 1..5 covering words
  u64 W[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) W[k] = ((u32)k < nw) ? ldg64(w + k) : 0;
  if (sh == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = W[k];
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = funnel(W[k], W[k + 1], sh);
  }
  mask_tail(t, r);
}

// --------------------------------------------------------------------------
// Register-ring reader: absorb every whole 32-byte block of a message and
// leave its r = len % 32 tail bytes (zero beyond r) in t.  Used by the
// ragged/fixed ring kernel (lh_engine.cu) and the streaming append.  One
// thread per message keeps D packets in flight in a register ring, and the
// reader is branch-free in the byte alignment, so lanes whose messages
// differ in alignment do not diverge.  Loads are 16-byte words from the
// aligned-down address; a packet's output words are funnel_r(U[m + o],
// U[m + o + 1], s) over the 12 32-bit words of three consecutive loads, with
// o = (addr >> 2) & 3 picked by two SEL levels and s = 8 * (addr & 3) (a
// zero shift is the identity).  Loads are clamped to the last word that
// holds a message byte (never past the message); a clamped word only feeds
// a zero shift or masked tail bytes.
// (4- and 8-byte word forms were measured: 2-3.5x slower on messages a
// power of two apart.)
// --------------------------------------------------------------------------
template <int D, class H>
__device__ __forceinline__ void absorb_ring128(H& h, const uint8_t* msg, u64 len, u64 (&t)[4]) {
  const uintptr_t a = (uintptr_t)msg;
  const uint4* w = (const uint4*)(a & ~(uintptr_t)15);
  const u32 o = (u32)(a >> 2) & 3u, s = (u32)(a & 3) * 8;
  const u64 nb = len >> 5;
  const u32 r = (u32)(len & 31);
  const u64 lastw = len ? ((a + len - 1) >> 4) - (a >> 4) : 0;  // last 16-B word with a message byte
  auto ld = [&](u64 k) { return __ldg(w + (k < lastw ? k : lastw)); };
  // Full packet pk covers 16-byte words 2pk .. 2pk+2; words up to 2pk+1
  // always hold message bytes, only 2pk+2 is clamped.
  auto ld_packet = [&](uint4 (&x)[2], u64 pk) {
    const uint4* p = w + 2 * pk;
    x[0] = __ldg(p + 1);
    x[1] = __ldg(2 * pk + 2 < lastw ? p + 2 : w + lastw);
  };
  auto packet = [&](const uint4& f, const uint4 (&x)[2], u64 (&p)[4]) {
    const u32 U[12] = {f.x, f.y, f.z, f.w, x[0].x, x[0].y, x[0].z, x[0].w,
                       x[1].x, x[1].y, x[1].z, x[1].w};
    u32 A[11], V[9];
#pragma unroll
    for (int j = 0; j < 11; ++j) A[j] = (o & 1u) ? U[j + 1] : U[j];
#pragma unroll
    for (int j = 0; j < 9; ++j) V[j] = (o & 2u) ? A[j + 2] : A[j];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      p[j] = pack(__funnelshift_r(V[2 * j], V[2 * j + 1], s),
                  __funnelshift_r(V[2 * j + 1], V[2 * j + 2], s));
  };
  uint4 ring[D][2];
  uint4 first = len ? __ldg(w) : make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int k = 0; k < D; ++k)
    if ((u64)k < nb) ld_packet(ring[k], (u64)k);
  u64 b = 0;
  for (; b + D <= nb; b += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      u64 p[4];
      packet(first, ring[k], p);
      first = ring[k][1];
      if (b + k + D < nb) ld_packet(ring[k], b + k + D);
      h.absorb32(p);
    }
  }
#pragma unroll
  for (int k = 0; k < D - 1; ++k) {
    if (b + k < nb) {
      u64 p[4];
      packet(first, ring[k], p);
      first = ring[k][1];
      h.absorb32(p);
    }
  }
  t[0] = t[1] = t[2] = t[3] = 0;
  if (r) {
    uint4 x[2];
    const u64 base = 2 * nb;
    x[0] = ld(base + 1);
    x[1] = ld(base + 2);
    packet(first, x, t);
    mask_tail(t, r);
  }
}

}  // namespace lh
