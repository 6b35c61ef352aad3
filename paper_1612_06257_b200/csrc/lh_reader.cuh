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
// Register-ring readers: absorb every whole 32-byte block of a message and
// leave its r = len % 32 tail bytes (zero beyond r) in t.  Used by the
// ragged/fixed ring kernel (lh_engine.cu) and the streaming append.
// Ragged medium/long messages when the batch is too small to hide load
// latency with warps (cfg2: 65,536 messages of 0..1023 bytes, ~14 warps per
// SM, the longest chain 32 packets).  One thread per message reads 32-bit
// words and keeps D packets in flight in a register ring (D loads deep
// instead of one).  The reader is branch-free in the alignment: word m of
// the message is funnel_r(v[m], v[m+1], s) with s = 8 * (addr & 3) over the
// 4-byte-aligned word stream starting at addr & ~3 (a zero shift is the
// identity), so lanes whose messages differ in alignment do not diverge.
// Word loads are clamped to the last word that holds a message byte (never
// past the message); a clamped word only feeds a zero shift or masked tail
// bytes.
// --------------------------------------------------------------------------
template <int D, class H>
__device__ __forceinline__ void absorb_ring(H& h, const uint8_t* msg, u64 len, u64 (&t)[4]) {
  const uintptr_t a = (uintptr_t)msg;
  const u32* w = (const u32*)(a & ~(uintptr_t)3);
  const u32 s = (u32)(a & 3) * 8;
  const u64 nb = len >> 5;
  const u32 r = (u32)(len & 31);
  const u64 lastw = len ? ((a + len - 1) >> 2) - (a >> 2) : 0;  // last word with a message byte
  auto ld = [&](u64 k) { return __ldg(w + (k < lastw ? k : lastw)); };
  // Words 8*pk+1 .. 8*pk+8 of full packet pk: words up to 8*pk+7 always hold
  // message bytes (immediate-offset loads), only word 8*pk+8 is clamped.
  auto ld_packet = [&](u32 (&x)[8], u64 pk) {
    const u32* p = w + 8 * pk;
#pragma unroll
    for (int j = 0; j < 7; ++j) x[j] = __ldg(p + j + 1);
    x[7] = __ldg(8 * pk + 8 < lastw ? p + 8 : w + lastw);
  };
  // ring[k][j] = word 8*(b+k) + j + 1 of the stream; `first` = word 8*b.
  u32 ring[D][8];
  u32 first = len ? __ldg(w) : 0u;
#pragma unroll
  for (int k = 0; k < D; ++k)
    if ((u64)k < nb) ld_packet(ring[k], (u64)k);
  auto packet = [&](const u32 (&x)[8], u32& f, u64 (&p)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const u32 lo = __funnelshift_r(j ? x[2 * j - 1] : f, x[2 * j], s);
      const u32 hi = __funnelshift_r(x[2 * j], x[2 * j + 1], s);
      p[j] = pack(lo, hi);
    }
    f = x[7];
  };
  u64 b = 0;
  for (; b + D <= nb; b += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      u64 p[4];
      packet(ring[k], first, p);
      if (b + k + D < nb) ld_packet(ring[k], b + k + D);
      h.absorb32(p);
    }
  }
#pragma unroll
  for (int k = 0; k < D - 1; ++k) {
    if (b + k < nb) {
      u64 p[4];
      packet(ring[k], first, p);
      h.absorb32(p);
    }
  }
  t[0] = t[1] = t[2] = t[3] = 0;
  if (r) {
    // Tail words 8*nb .. 8*nb+8 (clamped), then zero bytes >= r.
    u32 x[8];
    const u64 base = 8 * nb;
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = ld(base + j + 1);
    packet(x, first, t);
    mask_tail(t, r);
  }
}

// The same reader over 8-byte words (5 loads per packet instead of 9): the
// byte shift sh = 8 * (addr & 7) is split into a 32-bit word select (sh &
// 32, per-thread SEL) and a funnel shift by sh & 31, still branch-free.
template <int D, class H>
__device__ __forceinline__ void absorb_ring64(H& h, const uint8_t* msg, u64 len, u64 (&t)[4]) {
  const uintptr_t a = (uintptr_t)msg;
  const u64* w = (const u64*)(a & ~(uintptr_t)7);
  const u32 sh = (u32)(a & 7) * 8;
  const bool big = (sh & 32u) != 0;
  const u32 s5 = sh & 31u;
  const u64 nb = len >> 5;
  const u32 r = (u32)(len & 31);
  const u64 lastw = len ? ((a + len - 1) >> 3) - (a >> 3) : 0;  // last word with a message byte
  auto ld = [&](u64 k) { return ldg64(w + (k < lastw ? k : lastw)); };
  // Words 4*pk+1 .. 4*pk+4 of full packet pk; only word 4*pk+4 can lie past
  // the message (aligned start), so only it is clamped.
  auto ld_packet = [&](u64 (&x)[4], u64 pk) {
    const u64* p = w + 4 * pk;
#pragma unroll
    for (int j = 0; j < 3; ++j) x[j] = ldg64(p + j + 1);
    x[3] = ldg64(4 * pk + 4 < lastw ? p + 4 : w + lastw);
  };
  // Bytes [sh/8, sh/8 + 8) of hi_w:lo_w.
  auto fun = [&](u64 lo_w, u64 hi_w) {
    const u32 x0 = big ? hi32(lo_w) : lo32(lo_w);
    const u32 x1 = big ? lo32(hi_w) : hi32(lo_w);
    const u32 x2 = big ? hi32(hi_w) : lo32(hi_w);
    return pack(__funnelshift_r(x0, x1, s5), __funnelshift_r(x1, x2, s5));
  };
  u64 ring[D][4];
  u64 first = len ? ldg64(w) : 0ull;
#pragma unroll
  for (int k = 0; k < D; ++k)
    if ((u64)k < nb) ld_packet(ring[k], (u64)k);
  auto packet = [&](const u64 (&x)[4], u64& f, u64 (&p)[4]) {
    p[0] = fun(f, x[0]);
    p[1] = fun(x[0], x[1]);
    p[2] = fun(x[1], x[2]);
    p[3] = fun(x[2], x[3]);
    f = x[3];
  };
  u64 b = 0;
  for (; b + D <= nb; b += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      u64 p[4];
      packet(ring[k], first, p);
      if (b + k + D < nb) ld_packet(ring[k], b + k + D);
      h.absorb32(p);
    }
  }
#pragma unroll
  for (int k = 0; k < D - 1; ++k) {
    if (b + k < nb) {
      u64 p[4];
      packet(ring[k], first, p);
      h.absorb32(p);
    }
  }
  t[0] = t[1] = t[2] = t[3] = 0;
  if (r) {
    u64 x[4];
    const u64 base = 4 * nb;
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = ld(base + j + 1);
    packet(x, first, t);
    mask_tail(t, r);
  }
}

// The same reader over 16-byte words (2 loads per packet instead of 5 or
// 9: per-lane loads of different messages are separate L1 sector requests,
// which bound the small, latency-exposed ragged batches).  The 12 32-bit
// words of three consecutive 16-byte loads feed the output words m =
// funnel_r(U[m + o], U[m + o + 1], s) with o = (addr >> 2) & 3 selected by
// two SEL levels and s = 8 * (addr & 3).
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

// 8-byte words for HighwayHash (cfg2 26.6 -> 22.5 us; 4 GiB of 512..1536-B
// messages 1.72 -> 1.33 ms); 4-byte words for the Sip family, whose extra
// ALU work makes the 64-bit form's selects cost more than the loads it saves.
template <class H>
struct RingWide {
  static constexpr bool value = false;
};
template <>
struct RingWide<Highway> {
  static constexpr bool value = true;
};

}  // namespace lh
