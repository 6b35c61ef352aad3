// lh_device.cuh — per-message hash state machines for the sm_100a engine.
//
// Everything here is integer work on registers: one message's whole state
// lives in one thread.  The three "hashers" share one interface so the
// message readers (TMA-staged shared memory, or direct global loads) can
// feed any of them:
//
//   h.absorb32(p)            — one 32-byte block as 4 little-endian u64 words
//   h.finish(t, r, len, out) — tail t (r = len % 32 bytes, zero beyond r)
//
// Semantics follow the reference package `lanehash` (S = pkg/src/lanehash):
//   HighwayHash  S/highway.py:122-254   SipHash  S/sip.py:73-108
//   SipTreeHash  S/sip.py:111-128
#pragma once
#include <stdint.h>

namespace lh {

typedef uint64_t u64;
typedef uint32_t u32;

__device__ __forceinline__ u32 lo32(u64 x) { return (u32)x; }
__device__ __forceinline__ u32 hi32(u64 x) { return (u32)(x >> 32); }
__device__ __forceinline__ u64 pack(u32 lo, u32 hi) {
  return ((u64)hi << 32) | (u64)lo;
}
// Swapping the 32-bit halves is a register rename, not an instruction.
__device__ __forceinline__ u64 rot32(u64 x) { return pack(hi32(x), lo32(x)); }

// mul32 (S/highway.py:80-82): low32(a) * high32(b), full 64-bit product.
// One IMAD.WIDE.U32.
// Written as PTX mul.wide.u32: the C++ form (u64)x * (u64)y made ptxas add a
// zero high cross-term (an extra VIADD per multiply).
__device__ __forceinline__ u64 mul_lo_hi(u64 a, u64 b) {
  u64 r;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(lo32(a)), "r"(hi32(b)));
  return r;
}

// 64-bit add split across the two integer pipes: low word IADD3 (ALU pipe,
// carry out), high word IMAD.X hi*one + hi + carry (FMA pipe).  `one` is a
// runtime 1 supplied by the host so ptxas cannot fold the IMAD back into an
// ALU IADD3.X.  HighwayHash is ALU-pipe bound (PRMT, LOP3, IADD3 all issue
// there); this moves the high halves of all 20 64-bit adds per Update to the FMA
// pipe, except the 3-input v1 += p + m0 (one IADD3 + one IADD3.X per lane)
// (ALU: 20 PRMT + 16 LOP3 + 20 IADD3 = 56; FMA: 8 IMAD.WIDE + 12 IMAD.X).
__device__ __forceinline__ u64 add64_mixed(u64 a, u64 b, u32 one) {
  u32 lo, hi;
  asm("add.cc.u32 %0, %2, %3;\n\t"
      "madc.lo.u32 %1, %4, %6, %5;"
      : "=r"(lo), "=r"(hi)
      : "r"(lo32(a)), "r"(lo32(b)), "r"(hi32(a)), "r"(hi32(b)), "r"(one));
  return pack(lo, hi);
}

// Zipper merge of one lane pair (S/highway.py:35-38, 73-77).  Output byte i
// of the 16-byte pair comes from input byte ZIP[i] = 3 C 2 5 E 1 F 0 B 4 A D
// 9 6 8 7.  With input words W0..W3 (bytes 0-3, 4-7, 8-11, 12-15):
//   R0 = [b3 b12 b2 b5]   R1 = [b14 b1 b15 b0]
//   R2 = [b11 b4 b10 b13] R3 = [b9 b6 b8 b7]
// R0 and R2 each draw on three input words; both take their W1/W3 bytes from
// one shared intermediate u = [b5 b12 b4 b13], so the pair costs 5 PRMT.
__device__ __forceinline__ void zipper(u64 lo, u64 hi, u64& zlo, u64& zhi) {
  const u32 w0 = lo32(lo), w1 = hi32(lo), w2 = lo32(hi), w3 = hi32(hi);
  const u32 u = __byte_perm(w1, w3, 0x5041);
  const u32 r0 = __byte_perm(w0, u, 0x4253);
  const u32 r1 = __byte_perm(w3, w0, 0x4352);
  const u32 r2 = __byte_perm(w2, u, 0x7263);
  const u32 r3 = __byte_perm(w2, w1, 0x7061);
  zlo = pack(r0, r1);
  zhi = pack(r2, r3);
}

// The whole per-message HighwayHash state (S/highway.py:43-44, 122-150) plus
// the finalization parameters.  The key-only initial state is expanded on
// the host (lh_host.cuh: make_highway) and passed by value as a kernel
// parameter (the "prototype"); each message starts from a copy of it.
struct Highway {
  u64 v0[4], v1[4], m0[4], m1[4];
  int rounds;
  int width;  // 64, 128 or 256
  u32 one;    // = 1, opaque to the compiler (see add64_mixed)

  // S/highway.py:130-150 — per-lane order of steps 1-5, then the two
  // zipper-merge adds.
  __device__ __forceinline__ void update(u64 p0, u64 p1, u64 p2, u64 p3) {
    const u64 p[4] = {p0, p1, p2, p3};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v1[i] += p[i] + m0[i];  // 3-input IADD3 + IADD3.X: 2 instructions, no FMA-pipe help needed
      m0[i] ^= mul_lo_hi(v1[i], v0[i]);
      v0[i] = add64_mixed(v0[i], m1[i], one);
      m1[i] ^= mul_lo_hi(v0[i], v1[i]);
    }
    u64 z0, z1, z2, z3;
    zipper(v1[0], v1[1], z0, z1);
    zipper(v1[2], v1[3], z2, z3);
    v0[0] = add64_mixed(v0[0], z0, one);
    v0[1] = add64_mixed(v0[1], z1, one);
    v0[2] = add64_mixed(v0[2], z2, one);
    v0[3] = add64_mixed(v0[3], z3, one);
    zipper(v0[0], v0[1], z0, z1);
    zipper(v0[2], v0[3], z2, z3);
    v1[0] = add64_mixed(v1[0], z0, one);
    v1[1] = add64_mixed(v1[1], z1, one);
    v1[2] = add64_mixed(v1[2], z2, one);
    v1[3] = add64_mixed(v1[3], z3, one);
  }

  __device__ __forceinline__ void absorb32(const u64 (&p)[4]) {
    update(p[0], p[1], p[2], p[3]);
  }

  // The 16 state words from a copy of the prototype in shared memory (at
  // shared address `sa`, 16-byte aligned, v0 v1 m0 m1 order) with 8
  // LDS.128; the scalars from `proto`.  Kernels that start a new message
  // every few hundred instructions use it instead of `h = proto`, which
  // ptxas lowers to 16 LDCU.64 + 32 IMAD.U32 moves per message (the
  // parameter lives in the constant bank).  The loads are volatile so they
  // are not hoisted into 32 live registers.
  __device__ __forceinline__ void load_state(u32 sa, const Highway& proto) {
    u64* w[16] = {&v0[0], &v0[1], &v0[2], &v0[3], &v1[0], &v1[1], &v1[2], &v1[3],
                  &m0[0], &m0[1], &m0[2], &m0[3], &m1[0], &m1[1], &m1[2], &m1[3]};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      u32 a, b, c, d;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                   : "r"(sa + 16 * k));
      *w[2 * k] = pack(a, b);
      *w[2 * k + 1] = pack(c, d);
    }
    rounds = proto.rounds;
    width = proto.width;
    one = proto.one;
  }

  // S/highway.py:153-173: the exact inverse of update for the same packet
  // (self-test only; never on a hashing path).
  __device__ __forceinline__ void update_inverse(const u64 (&p)[4]) {
    u64 z0, z1, z2, z3;
    zipper(v0[0], v0[1], z0, z1);
    zipper(v0[2], v0[3], z2, z3);
    v1[0] -= z0;
    v1[1] -= z1;
    v1[2] -= z2;
    v1[3] -= z3;
    zipper(v1[0], v1[1], z0, z1);
    zipper(v1[2], v1[3], z2, z3);
    v0[0] -= z0;
    v0[1] -= z1;
    v0[2] -= z2;
    v0[3] -= z3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      m1[i] ^= mul_lo_hi(v0[i], v1[i]);
      v0[i] -= m1[i];
      m0[i] ^= mul_lo_hi(v1[i], v0[i]);
      v1[i] -= p[i] + m0[i];
    }
  }

  // S/highway.py:182-220.  t holds the r tail bytes (zero beyond r).
  __device__ __forceinline__ void remainder(const u64 (&t)[4], u32 r) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v0[i] = pack(lo32(v0[i]) + r, hi32(v0[i]) + r);
      v1[i] = pack(__funnelshift_l(lo32(v1[i]), lo32(v1[i]), r),
                   __funnelshift_l(hi32(v1[i]), hi32(v1[i]), r));
    }
    // Packet: tail[0 : 4*floor(r/4)], zeros, then the r%4 leftover bytes
    // little-endian in packet bytes 28..31.
    const u32 whole = r & ~3u;
    u64 p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int keep = (int)whole - 8 * k;  // bytes of word k to keep
      const u64 mask = keep >= 8 ? ~0ull : (keep <= 0 ? 0ull : ((1ull << (8 * keep)) - 1));
      p[k] = t[k] & mask;
    }
    // whole is a multiple of 4: the leftover word starts on a 32-bit half.
    // Select word whole/8 with two-level selects (keeps t in registers).
    const u64 s01 = (whole & 8) ? t[1] : t[0];
    const u64 s23 = (whole & 8) ? t[3] : t[2];
    const u64 src = (whole & 16) ? s23 : s01;
    u32 left = (whole & 4) ? hi32(src) : lo32(src);
    const u32 nleft = r & 3u;
    left &= nleft ? ((1u << (8 * nleft)) - 1u) : 0u;
    p[3] |= (u64)left << 32;
    update(p[0], p[1], p[2], p[3]);
  }

  // S/highway.py:176-179, 223-234.
  __device__ __forceinline__ void finalize_rounds() {
    for (int i = 0; i < rounds; ++i)
      update(rot32(v0[2]), rot32(v0[3]), rot32(v0[0]), rot32(v0[1]));
  }

  __device__ __forceinline__ void permute_update() {
    update(rot32(v0[2]), rot32(v0[3]), rot32(v0[0]), rot32(v0[1]));
  }

  // finalize_rounds + the first W lane sums, with the last two rounds peeled
  // out of the loop so the compiler drops the state the digest never reads.
  // W = 1 (HighwayHash-64): out[0] reads lane 0 only, so the last round
  // needs lanes 0-1 (v1[0] takes the zipper of v0[0], v0[1]) and skips the
  // second zipper's high word; the round before needs only v0 of lanes 2-3
  // (the last round's packet is rot32 of v0[2], v0[3]), so their multiplies
  // and the (2,3) v0 zipper go.  W = 2 drops lanes 2-3 of the last round.
  // About 70 of ~312 finalization instructions for W = 1.
  template <int W>
  __device__ __forceinline__ void finalize_out(u64* out) {
    int k = rounds;
    for (; k > 2; --k) permute_update();
    if (k == 2) permute_update();
    if (k >= 1) permute_update();
    out[0] = v0[0] + v1[0] + m0[0] + m1[0];
    if (W >= 2) out[1] = v0[1] + v1[1] + m0[1] + m1[1];
    if (W == 4) {
      out[2] = v0[2] + v1[2] + m0[2] + m1[2];
      out[3] = v0[3] + v1[3] + m0[3] + m1[3];
    }
  }

  // Width dispatch (uniform across a launch: one branch is hot).
  __device__ __forceinline__ void finalize_out(u64* out) {
    if (width == 64)
      finalize_out<1>(out);
    else if (width == 128)
      finalize_out<2>(out);
    else
      finalize_out<4>(out);
  }

  // Writes width/64 lane sums; lane 0 is HighwayHash-64.
  __device__ __forceinline__ void finish(const u64 (&t)[4], u32 r, u64 /*len*/,
                                         u64* out) {
    if (r) remainder(t, r);
    finalize_out(out);
  }
};

// HighwayHash with the 1024-bit state split over a thread pair (long
// messages, few of them).  Half h = 0 holds lanes {0,1}, h = 1 lanes {2,3}.
// Update never mixes the halves (per-lane steps 1-5, zipper pairs (0,1) and
// (2,3), S/highway.py:137-149), so it runs thread-locally on half the work;
// only PermuteAndUpdate (S/highway.py:176-179) crosses halves: half 0's new
// packet words are rot32 of half 1's v0 and vice versa — one 64-bit
// __shfl_xor pair per word per round.  Partner = lane ^ 1.
struct HighwayHalf {
  u64 v0[2], v1[2], m0[2], m1[2];
  int rounds;
  int width;
  u32 one;
  u32 half;

  __device__ __forceinline__ void init(const Highway& full, u32 h) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      v0[i] = h ? full.v0[2 + i] : full.v0[i];
      v1[i] = h ? full.v1[2 + i] : full.v1[i];
      m0[i] = h ? full.m0[2 + i] : full.m0[i];
      m1[i] = h ? full.m1[2 + i] : full.m1[i];
    }
    rounds = full.rounds;
    width = full.width;
    one = full.one;
    half = h;
  }

  // This half's lanes from the shared-memory prototype (Highway::load_state
  // layout: v0[4] v1[4] m0[4] m1[4]), 4 volatile LDS.128.
  __device__ __forceinline__ void load_state(u32 sa, const Highway& full, u32 h) {
    u64* w[8] = {&v0[0], &v0[1], &v1[0], &v1[1], &m0[0], &m0[1], &m1[0], &m1[1]};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u32 a, b, c, d;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                   : "r"(sa + 32 * k + 16 * h));
      *w[2 * k] = pack(a, b);
      *w[2 * k + 1] = pack(c, d);
    }
    rounds = full.rounds;
    width = full.width;
    one = full.one;
    half = h;
  }

  // LH_SPLIT_PLAIN_ADD (A/B): plain 64-bit adds in the split kernel, which is
  // bound by the latency of the Update chain, not by ALU slots.
  __device__ __forceinline__ u64 add_(u64 a, u64 b) const {
#ifdef LH_SPLIT_PLAIN_ADD
    return a + b;
#else
    return add64_mixed(a, b, one);
#endif
  }

  __device__ __forceinline__ void update(u64 pa, u64 pb) {
    const u64 p[2] = {pa, pb};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      v1[i] += p[i] + m0[i];  // 3-input IADD3 + IADD3.X: 2 instructions, no FMA-pipe help needed
      m0[i] ^= mul_lo_hi(v1[i], v0[i]);
      v0[i] = add_(v0[i], m1[i]);
      m1[i] ^= mul_lo_hi(v0[i], v1[i]);
    }
    u64 z0, z1;
    zipper(v1[0], v1[1], z0, z1);
    v0[0] = add_(v0[0], z0);
    v0[1] = add_(v0[1], z1);
    zipper(v0[0], v0[1], z0, z1);
    v1[0] = add_(v1[0], z0);
    v1[1] = add_(v1[1], z1);
  }

  // t: the full 32-byte tail (both threads hold it), r = len % 32.
  __device__ __forceinline__ void remainder(const u64 (&t)[4], u32 r) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      v0[i] = pack(lo32(v0[i]) + r, hi32(v0[i]) + r);
      v1[i] = pack(__funnelshift_l(lo32(v1[i]), lo32(v1[i]), r),
                   __funnelshift_l(hi32(v1[i]), hi32(v1[i]), r));
    }
    const u32 whole = r & ~3u;
    u64 p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int keep = (int)whole - 8 * k;
      const u64 mask = keep >= 8 ? ~0ull : (keep <= 0 ? 0ull : ((1ull << (8 * keep)) - 1));
      p[k] = t[k] & mask;
    }
    const u64 s01 = (whole & 8) ? t[1] : t[0];
    const u64 s23 = (whole & 8) ? t[3] : t[2];
    const u64 src = (whole & 16) ? s23 : s01;
    u32 left = (whole & 4) ? hi32(src) : lo32(src);
    const u32 nleft = r & 3u;
    left &= nleft ? ((1u << (8 * nleft)) - 1u) : 0u;
    p[3] |= (u64)left << 32;
    update(half ? p[2] : p[0], half ? p[3] : p[1]);
  }

  __device__ __forceinline__ static u64 shfl_xor1(u64 x) {
    return pack(__shfl_xor_sync(0xffffffffu, lo32(x), 1), __shfl_xor_sync(0xffffffffu, hi32(x), 1));
  }

  // All 32 lanes of the warp must call this together (shuffles).
  __device__ __forceinline__ void finalize_rounds() {
    for (int i = 0; i < rounds; ++i) {
      const u64 o0 = shfl_xor1(v0[0]), o1 = shfl_xor1(v0[1]);
      update(rot32(o0), rot32(o1));
    }
  }

  // Writes this half's two lanes back into a full state (streaming).
  __device__ __forceinline__ void save(Highway& full) const {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      full.v0[2 * half + i] = v0[i];
      full.v1[2 * half + i] = v1[i];
      full.m0[2 * half + i] = m0[i];
      full.m1[2 * half + i] = m1[i];
    }
  }

  // Writes this half's lanes of the width/64 lane sums (lane 0 first).
  __device__ __forceinline__ void store(u64* out) const {
    const u64 s0 = v0[0] + v1[0] + m0[0] + m1[0];
    const u64 s1 = v0[1] + v1[1] + m0[1] + m1[1];
    if (half == 0) {
      out[0] = s0;
      if (width >= 128) out[1] = s1;
    } else if (width == 256) {
      out[2] = s0;
      out[3] = s1;
    }
  }
};

// ---------------- SipHash-c-d (S/sip.py:73-108) ----------------

__device__ __forceinline__ u64 rotl64(u64 x, int b) {
  return (x << b) | (x >> (64 - b));
}

__device__ __forceinline__ u64 mulwide(u32 a, u32 b) {
  u64 r;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
  return r;
}

// Runtime constants that move part of SipRound to the FMA pipe: `one` for
// add64_mixed, and (LH_SIP_WIDE_ROT builds only) 2^13 / 2^17 / 2^16 so those
// rotates become IMAD.WIDE.U32 products (x * 2^k = x << k in the low word,
// x >> (32-k) in the high word) merged by a 3-input LOP3 with the following
// XOR.  Set by the host; opaque to ptxas, which would otherwise
// strength-reduce them.
struct SipMul {
  u32 one, m13, m17, m16;
};

// rotl64(x, k) ^ v with the shifts done as two 32x32->64 multiplies by 2^k:
// 2 IMAD.WIDE (FMA pipe) + 2 LOP3.
__device__ __forceinline__ u64 rotl_xor_wide(u64 x, u32 pow2k, u64 v) {
  const u64 a = mulwide(lo32(x), pow2k), b = mulwide(hi32(x), pow2k);
  const u32 lo = (lo32(a) | hi32(b)) ^ lo32(v);
  const u32 hi = (lo32(b) | hi32(a)) ^ hi32(v);
  return pack(lo, hi);
}

// rotl64(x, k) ^ v for 0 < k < 32 as two funnel shifts: 2 SHF + 2 LOP3 (ALU).
template <int K>
__device__ __forceinline__ u64 rotl_xor_shf(u64 x, u64 v) {
  const u32 hi = __funnelshift_l(lo32(x), hi32(x), K);
  const u32 lo = __funnelshift_l(hi32(x), lo32(x), K);
  return pack(lo ^ lo32(v), hi ^ hi32(v));
}

// rotl64(x, 16) ^ v as two byte permutes: 2 PRMT + 2 LOP3 (ALU).
__device__ __forceinline__ u64 rotl16_xor_prmt(u64 x, u64 v) {
  const u32 lo = __byte_perm(hi32(x), lo32(x), 0x5432);
  const u32 hi = __byte_perm(hi32(x), lo32(x), 0x1076);
  return pack(lo ^ lo32(v), hi ^ hi32(v));
}

// S/sip.py:73-86.  The four 64-bit adds are IADD3 (ALU) + IMAD.X (FMA, free
// beside an ALU instruction); every rotate runs on the ALU pipe: by 13, 17
// and 21 as two funnel shifts, by 16 as two PRMT, by 32 as a register rename:
// 20 ALU slots per round.  tools/issuemix.cu showed why the
// former IMAD.WIDE rotates (LH_SIP_WIDE_ROT, the A/B knob: by 13 and 17
// always, by 16 on every other round) only looked cheaper: an IMAD.WIDE holds
// the ALU issue slot for 2 clocks besides its 4 FMA clocks, so a WIDE pair
// costs the ALU pipe what two SHF cost and the FMA pipe 8 clocks on top.
// All-ALU: SipHash-2-4 / -1-3 / SipTree-2-4 / -1-3 over 2^24 x 1 KiB
// 5.48 / 3.00 / 6.08 / 3.39 -> 5.16 / 2.83 / 5.83 / 3.26 ms.
template <bool W16>
__device__ __forceinline__ void sip_round(u64& v0, u64& v1, u64& v2, u64& v3, const SipMul& k) {
#ifdef LH_SIP_WIDE_ROT
  v0 = add64_mixed(v0, v1, k.one);
  v1 = rotl_xor_wide(v1, k.m13, v0);
  v0 = rot32(v0);
  v2 = add64_mixed(v2, v3, k.one);
  v3 = W16 ? rotl_xor_wide(v3, k.m16, v2) : rotl16_xor_prmt(v3, v2);
  v0 = add64_mixed(v0, v3, k.one);
  v3 = rotl_xor_shf<21>(v3, v0);
  v2 = add64_mixed(v2, v1, k.one);
  v1 = rotl_xor_wide(v1, k.m17, v2);
  v2 = rot32(v2);
#else
  v0 = add64_mixed(v0, v1, k.one);
  v1 = rotl_xor_shf<13>(v1, v0);
  v0 = rot32(v0);
  v2 = add64_mixed(v2, v3, k.one);
  v3 = rotl16_xor_prmt(v3, v2);
  v0 = add64_mixed(v0, v3, k.one);
  v3 = rotl_xor_shf<21>(v3, v0);
  v2 = add64_mixed(v2, v1, k.one);
  v1 = rotl_xor_shf<17>(v1, v2);
  v2 = rot32(v2);
#endif
}

__device__ __forceinline__ void sip_round(u64& v0, u64& v1, u64& v2, u64& v3, const SipMul& k) {
  sip_round<false>(v0, v1, v2, v3, k);
}

// n SipRounds (n compile-time when N > 0); the two forms differ only in
// LH_SIP_WIDE_ROT builds.
template <int N>
__device__ __forceinline__ void sip_rounds(u64& v0, u64& v1, u64& v2, u64& v3, const SipMul& k,
                                           int n) {
  if (N > 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i & 1)
        sip_round<true>(v0, v1, v2, v3, k);
      else
        sip_round<false>(v0, v1, v2, v3, k);
    }
  } else {
    int i = 0;
    for (; i + 1 < n; i += 2) {
      sip_round<false>(v0, v1, v2, v3, k);
      sip_round<true>(v0, v1, v2, v3, k);
    }
    if (i < n) sip_round<false>(v0, v1, v2, v3, k);
  }
}

struct SipKey {
  u64 k0, k1;
};

// Round counts: compile-time when C,D > 0, else the runtime c,d fields.
template <int C, int D>
struct SipCore {
  u64 v0, v1, v2, v3;
  __device__ __forceinline__ void init(const SipKey& k) {
    v0 = 0x736F6D6570736575ull ^ k.k0;
    v1 = 0x646F72616E646F6Dull ^ k.k1;
    v2 = 0x6C7967656E657261ull ^ k.k0;
    v3 = 0x7465646279746573ull ^ k.k1;
  }
  __device__ __forceinline__ void compress(u64 m, int c, const SipMul& k) {
    v3 ^= m;
    sip_rounds<C>(v0, v1, v2, v3, k, c);
    v0 ^= m;
  }
  __device__ __forceinline__ u64 final(u64 m_last, int c, int d, const SipMul& k) {
    compress(m_last, c, k);
    v2 ^= 0xFF;
    sip_rounds<D>(v0, v1, v2, v3, k, d);
    return v0 ^ v1 ^ v2 ^ v3;
  }
};

template <int C, int D>
struct Sip {
  SipCore<C, D> s;
  int c, d;
  SipMul k;
  __device__ __forceinline__ void init(const SipKey& k, int c_, int d_) {
    s.init(k);
    c = c_;
    d = d_;
  }
  __device__ __forceinline__ void absorb32(const u64 (&p)[4]) {
#pragma unroll
    for (int w = 0; w < 4; ++w) s.compress(p[w], c, k);
  }
  // Tail: r = len % 32 bytes in t (zero beyond r).  Whole words first, then
  // the final word = leftover bytes | (len & 0xFF) << 56 (S/sip.py:100-101).
  __device__ __forceinline__ void finish(const u64 (&t)[4], u32 r, u64 len, u64* out) {
    const u32 nw = r >> 3;
#pragma unroll
    for (int w = 0; w < 3; ++w)
      if ((u32)w < nw) s.compress(t[w], c, k);
    const u64 s01 = (nw & 1) ? t[1] : t[0];
    const u64 s23 = (nw & 1) ? t[3] : t[2];
    const u64 last = (nw & 2) ? s23 : s01;
    out[0] = s.final(last | ((len & 0xFF) << 56), c, d, k);
  }
};

// SipTreeHash (S/sip.py:111-128): the zero-padded message's 64-bit words are
// dealt round-robin to 4 independent SipHash chains (ILP 4 in one thread);
// each chain's own length is padded_len/4; the 4 digests are folded with one
// more SipHash over their 32-byte little-endian concatenation.
template <int C, int D>
struct SipTree {
  SipCore<C, D> l0, l1, l2, l3;
  SipKey key;
  int c, d;
  SipMul k;
  __device__ __forceinline__ void init(const SipKey& k, int c_, int d_) {
    key = k;
    l0.init(k);
    l1.init(k);
    l2.init(k);
    l3.init(k);
    c = c_;
    d = d_;
  }
  __device__ __forceinline__ void absorb32(const u64 (&p)[4]) {
    l0.compress(p[0], c, k);
    l1.compress(p[1], c, k);
    l2.compress(p[2], c, k);
    l3.compress(p[3], c, k);
  }
  __device__ __forceinline__ void finish(const u64 (&t)[4], u32 r, u64 len, u64* out) {
    if (r) absorb32(t);  // zero-padded final block
    const u64 lane_len = ((len + 31) & ~31ull) >> 2;
    const u64 m = (lane_len & 0xFF) << 56;
    const u64 h0 = l0.final(m, c, d, k);
    const u64 h1 = l1.final(m, c, d, k);
    const u64 h2 = l2.final(m, c, d, k);
    const u64 h3 = l3.final(m, c, d, k);
    SipCore<C, D> f;
    f.init(key);
    f.compress(h0, c, k);
    f.compress(h1, c, k);
    f.compress(h2, c, k);
    f.compress(h3, c, k);
    out[0] = f.final(32ull << 56, c, d, k);
  }
};

}  // namespace lh
