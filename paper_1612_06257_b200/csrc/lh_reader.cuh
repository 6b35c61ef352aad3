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

}  // namespace lh
