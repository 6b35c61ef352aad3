// lh_stream.cu — batched incremental (streaming) hashing on the device.
//
// The batch analogue of the reference's streaming hashers:
//   HighwayHash  StreamingHasher   S/highway.py:257-285
//   SipHash      SipHasher         S/sip.py:131-169
//   SipTreeHash  SipTreeHasher     S/sip.py:172-203
// n messages advance together: every message keeps its hasher state, a
// <= 31-byte pending tail and its total length in one HBM record
// (StreamRec<H>); lh_stream_update appends one chunk per message (fixed
// layout or ragged), lh_stream_finish reads the records and writes digests.
// All three hashers absorb 32-byte blocks (HighwayHash packets; 4 SipHash
// words; one word per SipTree lane, S/sip.py:186-188), so only a block's
// worth of tail is ever buffered, and only the total length feeds
// finalization (S/highway.py:278-285: only len mod 32 matters; SipHash the
// length byte; SipTree the lane length).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lanehash_b200.h"
#include "lh_device.cuh"
#include "lh_host.cuh"
#include "lh_reader.cuh"
#include "lh_stream.cuh"

using namespace lh;

namespace {

template <class H>
__global__ void k_stream_init(StreamRec<H>* __restrict__ rec, const H proto, u64 n) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    StreamRec<H> r;
    r.h = proto;
    r.total = 0;
    r.tail[0] = r.tail[1] = r.tail[2] = r.tail[3] = 0;
    r.tlen = 0;
    r.pad = 0;
    rec[i] = r;
  }
}

template <class H>
__global__ void k_stream_update(StreamRec<H>* __restrict__ rec, u64 n,
                                const uint8_t* __restrict__ buf, const u64* __restrict__ offsets,
                                const u32* __restrict__ lengths, u64 chunk_len) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    const uint8_t* p;
    u64 len;
    if (offsets) {
      const u64 off = offsets[i];
      len = lengths ? (u64)lengths[i] : offsets[i + 1] - off;
      p = buf + off;
    } else {
      p = buf + i * chunk_len;
      len = chunk_len;
    }
    if (len == 0) continue;
    StreamRec<H> r = rec[i];
    stream_append<true>(r, p, len);
    rec[i] = r;
  }
}

// The absorbed state does not depend on the digest width (S/highway.py:
// 223-234 only reads it in finalize), so HighwayHash finishes at the width
// the caller asks for now.
__device__ __forceinline__ void set_lanes(Highway& h, int lanes) { h.width = 64 * lanes; }
template <class H>
__device__ __forceinline__ void set_lanes(H&, int) {}

template <class H>
__global__ void k_stream_finish(const StreamRec<H>* __restrict__ rec, u64 n,
                                u64* __restrict__ out, int lanes) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    StreamRec<H> r = rec[i];
    set_lanes(r.h, lanes);
    r.h.finish(r.tail, r.tlen, r.total, out + i * lanes);
  }
}

unsigned grid_for(u64 n) {
  const u64 b = (n + 255) / 256;
  return (unsigned)(b == 0 ? 1 : (b > 148 * 64 ? 148 * 64 : b));
}

int err() { return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA; }

}  // namespace

extern "C" {

size_t lh_stream_state_bytes(int alg) {
  switch (alg) {
    case LH_ALG_HIGHWAY: return sizeof(StreamRec<Highway>);
    case LH_ALG_SIPHASH: return sizeof(StreamRec<Sip<0, 0>>);
    case LH_ALG_SIPTREE: return sizeof(StreamRec<SipTree<0, 0>>);
    default: return 0;
  }
}

int lh_stream_init(int alg, void* d_state, uint64_t n, const uint64_t* key, int p1, int p2,
                   void* stream) {
  if (!key || (n && !d_state)) return LH_EINVAL;
  if ((uintptr_t)d_state % 16) return LH_EALIGN;
  cudaStream_t st = (cudaStream_t)stream;
  if (alg == LH_ALG_HIGHWAY) {
    if ((p1 != 64 && p1 != 128 && p1 != 256) || p2 < 0) return LH_EINVAL;
    if (!n) return LH_OK;
    k_stream_init<<<grid_for(n), 256, 0, st>>>((StreamRec<Highway>*)d_state,
                                               make_highway(key, p1, p2), n);
    return err();
  }
  if (p1 < 1 || p2 < 1) return LH_EINVAL;
  if (alg == LH_ALG_SIPHASH) {
    if (!n) return LH_OK;
    k_stream_init<<<grid_for(n), 256, 0, st>>>((StreamRec<Sip<0, 0>>*)d_state,
                                               make_sip<0, 0>(key, p1, p2), n);
    return err();
  }
  if (alg == LH_ALG_SIPTREE) {
    if (!n) return LH_OK;
    k_stream_init<<<grid_for(n), 256, 0, st>>>((StreamRec<SipTree<0, 0>>*)d_state,
                                               make_siptree<0, 0>(key, p1, p2), n);
    return err();
  }
  return LH_EINVAL;
}

int lh_stream_update(int alg, void* d_state, uint64_t n, const uint8_t* d_buf,
                     const uint64_t* d_offsets, const uint32_t* d_lengths, uint64_t chunk_len,
                     void* stream) {
  if (n && !d_state) return LH_EINVAL;
  if (n && !d_buf && (d_offsets || chunk_len)) return LH_EINVAL;
  if ((uintptr_t)d_state % 16 || (uintptr_t)d_offsets % 8 || (uintptr_t)d_lengths % 4)
    return LH_EALIGN;
  if (!n) return LH_OK;
  if (!d_offsets) {
    // Whole-block fixed-layout chunks: TMA-staged rows (rows with a pending
    // tail take the generic append inside that kernel).
    const int rc = stream_update_tma(alg, d_state, n, d_buf, chunk_len, stream);
    if (rc != LH_EINVAL) return rc;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned g = grid_for(n);
  switch (alg) {
    case LH_ALG_HIGHWAY:
      k_stream_update<<<g, 256, 0, st>>>((StreamRec<Highway>*)d_state, n, d_buf, d_offsets,
                                         d_lengths, chunk_len);
      return err();
    case LH_ALG_SIPHASH:
      k_stream_update<<<g, 256, 0, st>>>((StreamRec<Sip<0, 0>>*)d_state, n, d_buf, d_offsets,
                                         d_lengths, chunk_len);
      return err();
    case LH_ALG_SIPTREE:
      k_stream_update<<<g, 256, 0, st>>>((StreamRec<SipTree<0, 0>>*)d_state, n, d_buf,
                                         d_offsets, d_lengths, chunk_len);
      return err();
    default: return LH_EINVAL;
  }
}

int lh_stream_finish(int alg, const void* d_state, uint64_t n, uint64_t* d_out, int lanes,
                     void* stream) {
  if (n && (!d_state || !d_out)) return LH_EINVAL;
  if ((uintptr_t)d_state % 16 || (uintptr_t)d_out % 8) return LH_EALIGN;
  if (lanes != 1 && lanes != 2 && lanes != 4) return LH_EINVAL;
  if (!n) return LH_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned g = grid_for(n);
  switch (alg) {
    case LH_ALG_HIGHWAY:
      k_stream_finish<<<g, 256, 0, st>>>((const StreamRec<Highway>*)d_state, n, d_out, lanes);
      return err();
    case LH_ALG_SIPHASH:
      if (lanes != 1) return LH_EINVAL;
      k_stream_finish<<<g, 256, 0, st>>>((const StreamRec<Sip<0, 0>>*)d_state, n, d_out, 1);
      return err();
    case LH_ALG_SIPTREE:
      if (lanes != 1) return LH_EINVAL;
      k_stream_finish<<<g, 256, 0, st>>>((const StreamRec<SipTree<0, 0>>*)d_state, n, d_out, 1);
      return err();
    default: return LH_EINVAL;
  }
}

}  // extern "C"
