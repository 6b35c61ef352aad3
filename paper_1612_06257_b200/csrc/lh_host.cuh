// lh_host.cuh — host-side construction of the hasher prototypes that the
// kernels copy by value (key expansion happens once per batch, here).
#pragma once
#include <string.h>

#include "lh_device.cuh"

namespace lh {
// --------------------------------------------------------------------------
// Host-side hasher prototypes (the kernels copy them by value).
// --------------------------------------------------------------------------

// S/highway.py:20-31
static const u64 kInit0[4] = {0xDBE6D5D5FE4CCE2FULL, 0xA4093822299F31D0ULL, 0x13198A2E03707344ULL,
                       0x243F6A8885A308D3ULL};
static const u64 kInit1[4] = {0x3BD39E10CB0EF593ULL, 0xC0ACF169B5F18A8CULL, 0xBE5466CF34E90C6CULL,
                       0x452821E638D01377ULL};

static inline u64 h_rot32(u64 x) { return (x >> 32) | (x << 32); }

// Key expansion, S/highway.py:122-127 (one key per batch: done once here).
static inline Highway make_highway(const u64 key[4], int width, int rounds) {
  Highway h;
  memset(&h, 0, sizeof h);
  for (int i = 0; i < 4; ++i) {
    h.v0[i] = key[i] ^ kInit0[i];
    h.v1[i] = h_rot32(key[i]) ^ kInit1[i];
    h.m0[i] = kInit0[i];
    h.m1[i] = kInit1[i];
  }
  h.rounds = rounds;
  h.width = width;
  h.one = 1;
  return h;
}

template <int C, int D>
inline void h_sip_init(SipCore<C, D>& s, const SipKey& k) {
  s.v0 = 0x736F6D6570736575ull ^ k.k0;
  s.v1 = 0x646F72616E646F6Dull ^ k.k1;
  s.v2 = 0x6C7967656E657261ull ^ k.k0;
  s.v3 = 0x7465646279746573ull ^ k.k1;
}

template <int C, int D>
inline Sip<C, D> make_sip(const u64 key[2], int c, int d) {
  Sip<C, D> h;
  memset(&h, 0, sizeof h);
  h_sip_init(h.s, SipKey{key[0], key[1]});
  h.c = c;
  h.d = d;
  h.k = SipMul{1u, 1u << 13, 1u << 17, 1u << 16};
  return h;
}

template <int C, int D>
inline SipTree<C, D> make_siptree(const u64 key[2], int c, int d) {
  SipTree<C, D> h;
  memset(&h, 0, sizeof h);
  const SipKey k{key[0], key[1]};
  h.key = k;
  h_sip_init(h.l0, k);
  h_sip_init(h.l1, k);
  h_sip_init(h.l2, k);
  h_sip_init(h.l3, k);
  h.c = c;
  h.d = d;
  h.k = SipMul{1u, 1u << 13, 1u << 17, 1u << 16};
  return h;
}

}  // namespace lh
