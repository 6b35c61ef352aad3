// lh_quality.cu — avalanche flip tallies on the device (quality harness).
//
// Computes S/_kernels.py:247-265 (avalanche_counts): for every message and
// every input bit b, diff = hash(msg ^ (1 << b)) ^ hash(msg), and
// counts[b][ob] += bit ob of diff.  This is what the reference's avalanche
// protocol (S/quality.py:105-194) and finalization-round experiment
// (S/quality.py:245-293) spend their time on: 8*size+1 hashes per message.
//
// Grid: blockIdx.x = a group of 256 messages (8 warps x 32), blockIdx.y = one
// input byte (its 8 bits).  A warp hashes its 32 messages once (base), then
// once per flipped bit; the 64 output-bit columns of the 32 diffs are
// counted with 64 warp ballots + popcounts and accumulated in shared memory,
// flushed to the global int64 tallies with one atomic per cell per block.
// Messages are at most 32 bytes (the reference's sizes are 3..32) and live
// in registers; d_msgs == NULL selects counter messages (message i = the
// little-endian bytes of i), the reference's exhaustive 3-byte enumeration
// (S/quality.py:261-265) without a 48 MiB input buffer.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lanehash_b200.h"
#include "lh_device.cuh"
#include "lh_host.cuh"

using namespace lh;

namespace {

constexpr int kQWarps = 8;

// Hash of a <= 32-byte message held as 4 LE words (zero past size).
template <class H>
__device__ __forceinline__ u64 hash_words(const H& proto, const u64 (&w)[4], u32 size) {
  H h = proto;
  u64 out[4];
  if (size == 32) {
    h.absorb32(w);
    const u64 z[4] = {0, 0, 0, 0};
    h.finish(z, 0, 32, out);
  } else {
    h.finish(w, size, size, out);
  }
  return out[0];
}

template <class H>
__global__ void __launch_bounds__(kQWarps * 32)
    k_avalanche(const H proto, const uint8_t* __restrict__ msgs, u64 iters, u32 size,
                unsigned long long* __restrict__ counts) {
  __shared__ u32 tally[8][64];
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (u32 c = threadIdx.x; c < 8 * 64; c += blockDim.x) (&tally[0][0])[c] = 0;
  __syncthreads();

  const u32 byte = blockIdx.y;  // input byte whose 8 bits this block flips
  const u64 m = ((u64)blockIdx.x * kQWarps + warp) * 32 + lane;
  const bool valid = m < iters;
  u64 w[4] = {0, 0, 0, 0};
  if (valid) {
    if (msgs) {
      const uint8_t* p = msgs + m * size;
      for (u32 j = 0; j < size; ++j) {
        const u64 b = p[j];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if ((j >> 3) == (u32)k) w[k] |= b << (8 * (j & 7));
      }
    } else {  // counter message: LE bytes of m, truncated to size
      w[0] = size >= 8 ? m : (m & ((1ull << (8 * size)) - 1));
    }
  }
  const u64 base = valid ? hash_words(proto, w, size) : 0;
  if (byte < size) {
    for (u32 bit = 0; bit < 8; ++bit) {
      const u32 b = 8 * byte + bit;
      u64 f[4] = {w[0], w[1], w[2], w[3]};
      const u64 mask = 1ull << (b & 63);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((b >> 6) == (u32)k) f[k] ^= mask;
      const u64 d = valid ? (hash_words(proto, f, size) ^ base) : 0;
      u32 c0 = 0, c1 = 0;
#pragma unroll
      for (int ob = 0; ob < 32; ++ob) {
        const u32 b0 = __popc(__ballot_sync(0xffffffffu, (u32)(d >> ob) & 1u));
        const u32 b1 = __popc(__ballot_sync(0xffffffffu, (u32)(d >> (ob + 32)) & 1u));
        if (lane == (u32)ob) {
          c0 = b0;
          c1 = b1;
        }
      }
      if (c0) atomicAdd(&tally[bit][lane], c0);
      if (c1) atomicAdd(&tally[bit][lane + 32], c1);
    }
  }
  __syncthreads();
  for (u32 c = threadIdx.x; c < 8 * 64; c += blockDim.x) {
    const u32 bit = c >> 6, ob = c & 63;
    const u32 v = tally[bit][ob];
    if (v && byte < size)
      atomicAdd(&counts[(u64)(8 * byte + bit) * 64 + ob], (unsigned long long)v);
  }
}

template <class H>
int launch(const H& proto, const uint8_t* msgs, u64 iters, u32 size, int64_t* counts,
           cudaStream_t st) {
  if (!iters) return LH_OK;
  const u64 groups = (iters + kQWarps * 32 - 1) / (kQWarps * 32);
  if (groups > 0x7fffffffull) return LH_ETOOBIG;
  dim3 grid((unsigned)groups, size);
  k_avalanche<H><<<grid, kQWarps * 32, 0, st>>>(proto, msgs, iters, size,
                                                (unsigned long long*)counts);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}

}  // namespace

extern "C" int lh_avalanche_counts(int alg, const uint64_t* key, const uint8_t* d_msgs,
                                   uint64_t iters, uint32_t size, int p1, int p2,
                                   int64_t* d_counts, void* stream) {
  if (!key || !d_counts || size < 1 || size > 32 || p1 < 0) return LH_EINVAL;
  if ((uintptr_t)d_counts % 8) return LH_EALIGN;
  cudaStream_t st = (cudaStream_t)stream;
  switch (alg) {
    case LH_ALG_HIGHWAY: return launch(make_highway(key, 64, p1), d_msgs, iters, size, d_counts, st);
    case LH_ALG_SIPHASH:
      if (p1 < 1 || p2 < 1) return LH_EINVAL;
      if (p1 == 2 && p2 == 4) return launch(make_sip<2, 4>(key, 2, 4), d_msgs, iters, size, d_counts, st);
      if (p1 == 1 && p2 == 3) return launch(make_sip<1, 3>(key, 1, 3), d_msgs, iters, size, d_counts, st);
      return launch(make_sip<0, 0>(key, p1, p2), d_msgs, iters, size, d_counts, st);
    case LH_ALG_SIPTREE:
      if (p1 < 1 || p2 < 1) return LH_EINVAL;
      if (p1 == 2 && p2 == 4)
        return launch(make_siptree<2, 4>(key, 2, 4), d_msgs, iters, size, d_counts, st);
      if (p1 == 1 && p2 == 3)
        return launch(make_siptree<1, 3>(key, 1, 3), d_msgs, iters, size, d_counts, st);
      return launch(make_siptree<0, 0>(key, p1, p2), d_msgs, iters, size, d_counts, st);
    default: return LH_EINVAL;
  }
}
