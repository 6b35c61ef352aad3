// lh_sip_variants.h — the Sip-family instantiations, one object file each
// (lh_sip_variant.cu compiled with -DLH_VAR_TAG=... by _build.py), called by
// the extern "C" boundary in lh_engine.cu.  Compile-time round counts for
// SipHash-2-4 and -1-3 (the reference's SIPHASH_24 / SIPHASH_13,
// S/sip.py:64-66), runtime counts for every other (c, d).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// X(tag, C, D, TREE)
#define LH_SIP_VARIANTS(X) \
  X(s24, 2, 4, 0)          \
  X(s13, 1, 3, 0)          \
  X(s00, 0, 0, 0)          \
  X(t24, 2, 4, 1)          \
  X(t13, 1, 3, 1)          \
  X(t00, 0, 0, 1)

namespace lh {
#define LH_SIP_DECLARE(tag, C, D, TREE)                                                        \
  int sip_fixed_##tag(const uint64_t key[2], int c, int d, const uint8_t* msgs, uint64_t n,   \
                      uint64_t len, uint64_t* out, cudaStream_t st, int kernel);              \
  int sip_ragged_##tag(const uint64_t key[2], int c, int d, const uint8_t* buf,               \
                       const uint64_t* off, const uint32_t* lens, uint64_t n, uint64_t* out,  \
                       cudaStream_t st, bool staged, const uint4* order);                     \
  int sip_stream_tma_##tag(void* rec, const uint8_t* chunks, uint64_t n, uint64_t len,        \
                           cudaStream_t st);
LH_SIP_VARIANTS(LH_SIP_DECLARE)
#undef LH_SIP_DECLARE
}  // namespace lh
