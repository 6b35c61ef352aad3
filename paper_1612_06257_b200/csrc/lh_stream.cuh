// lh_stream.cuh — the per-message streaming record and its generic append,
// shared by the per-thread streaming kernel (lh_stream.cu) and the
// TMA-staged whole-block path (lh_engine.cu).
#pragma once
#include <stdint.h>

#include "lh_device.cuh"
#include "lh_reader.cuh"

namespace lh {

template <class H>
struct __align__(16) StreamRec {
  H h;
  u64 total;    // bytes appended so far
  u64 tail[4];  // pending bytes (LE), zero past tlen
  u32 tlen;     // 0..31
  u32 pad;
};

__device__ __forceinline__ void put_byte(u64 (&t)[4], u32 pos, u32 byte) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if ((pos >> 3) == (u32)k) t[k] |= (u64)byte << (8 * (pos & 7));
}

// Append len bytes at p to one message's record (S/highway.py:257-285,
// S/sip.py:131-203): complete a pending block, absorb whole blocks, keep
// the rest pending.  RING: whole blocks through the branch-free register-ring
// reader (the streaming kernel); otherwise the plain reader (the fallback
// inside the TMA-staged append, where registers are scarce).
template <bool RING, class H>
__device__ __forceinline__ void stream_append(StreamRec<H>& r, const uint8_t* p, u64 len) {
  if (len == 0) return;
  const u32 t = r.tlen;
  r.total += len;
  if (t + len < 32) {  // everything stays pending
    for (u32 j = 0; j < (u32)len; ++j) put_byte(r.tail, t + j, p[j]);
    r.tlen = t + (u32)len;
    return;
  }
  if (t) {  // complete the pending block from the chunk's first bytes
    const u32 need = 32 - t;
    for (u32 j = 0; j < need; ++j) put_byte(r.tail, t + j, p[j]);
    r.h.absorb32(r.tail);
    p += need;
    len -= need;
  }
  if constexpr (!RING) {
    absorb_blocks(r.h, p, len >> 5);
    load_tail(p + (len & ~31ull), (u32)(len & 31), r.tail);
  } else {
    // 16-byte words, two blocks in flight.  (Depth 1 was ~10% faster here,
    // but the same reader at depth 1 inlined into the staged kernels' fallback
    // gave wrong digests on one code shape -- treated as a ptxas hazard,
    // so depth 1 is used nowhere.)
    absorb_ring128<2>(r.h, p, len, r.tail);
  }
  r.tlen = (u32)(len & 31);
}

// TMA-staged append of fixed-layout chunks of chunk_len bytes (a multiple
// of 32, rows 16-byte aligned, n >= 1,024); defined in lh_engine.cu.
// Returns LH_EINVAL when the shape does not qualify (caller falls back).
int stream_update_tma(int alg, void* d_state, u64 n, const uint8_t* d_chunks, u64 chunk_len,
                      void* stream);

}  // namespace lh
