// lh_plan.cu — one pass over a ragged layout's metadata: per-chunk byte
// spans and a count of invalid messages (include/lanehash_b200.h:
// lh_ragged_plan).
//
// The host pipeline (engine._ragged_host_pipelined) streams a host ragged
// batch through the GPU in message-range chunks; each chunk needs the byte
// span [min start, max end) of its messages so only that span crosses PCIe.
// The same pass validates the layout before any hashing kernel reads it:
// a message is invalid if (offsets[n+1] form) offsets[i+1] < offsets[i], if
// start + length wraps, or if it ends past buf_len.  Grid: blockIdx.y = the
// chunk, blockIdx.x = a 4,096-message slice of it, so every block reduces
// into one chunk (warp shuffles, then one atomic per warp).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lanehash_b200.h"

namespace {

constexpr unsigned kPlanThreads = 256;
constexpr uint64_t kSlice = 4096;

__global__ void __launch_bounds__(kPlanThreads)
    k_ragged_plan(const uint64_t* __restrict__ off, const uint32_t* __restrict__ lens, uint64_t n,
                  uint64_t chunk_msgs, uint64_t buf_len, unsigned long long* __restrict__ lo,
                  unsigned long long* __restrict__ hi, unsigned long long* __restrict__ bad) {
  const uint64_t c = blockIdx.y;
  const uint64_t c0 = c * chunk_msgs;
  const uint64_t c1 = c0 + chunk_msgs < n ? c0 + chunk_msgs : n;
  const uint64_t s0 = c0 + (uint64_t)blockIdx.x * kSlice;
  const uint64_t s1 = s0 + kSlice < c1 ? s0 + kSlice : c1;
  unsigned long long mn = ~0ull, mx = 0;
  unsigned nbad = 0;
  for (uint64_t i = s0 + threadIdx.x; i < s1; i += kPlanThreads) {
    const uint64_t start = off[i];
    uint64_t end;
    bool ok;
    if (lens) {
      end = start + lens[i];
      ok = end >= start;  // no wrap
    } else {
      end = off[i + 1];
      ok = end >= start;  // non-decreasing offsets
    }
    ok = ok && end <= buf_len;
    nbad += !ok;
    mn = start < mn ? start : mn;
    mx = end > mx ? end : mx;
  }
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, s);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, mx, s);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  nbad = __reduce_add_sync(0xffffffffu, nbad);
  if ((threadIdx.x & 31) == 0) {
    if (mn != ~0ull) atomicMin(&lo[c], mn);
    if (mx) atomicMax(&hi[c], mx);
    if (nbad) atomicAdd(bad, (unsigned long long)nbad);
  }
}

}  // namespace

extern "C" int lh_ragged_plan(const uint64_t* d_offsets, const uint32_t* d_lengths, uint64_t n,
                              uint64_t chunk_msgs, uint64_t buf_len, uint64_t* d_lo,
                              uint64_t* d_hi, uint64_t* d_bad, void* stream) {
  if (!d_bad || (n && (!d_offsets || !d_lo || !d_hi || chunk_msgs == 0))) return LH_EINVAL;
  if ((uintptr_t)d_offsets % 8 || (uintptr_t)d_lengths % 4 || (uintptr_t)d_lo % 8 ||
      (uintptr_t)d_hi % 8 || (uintptr_t)d_bad % 8)
    return LH_EALIGN;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t nchunks = n ? (n + chunk_msgs - 1) / chunk_msgs : 0;
  if (nchunks > 65535) return LH_ETOOBIG;
  if (cudaMemsetAsync(d_bad, 0, 8, st) != cudaSuccess) return LH_ECUDA;
  if (!n) return LH_OK;
  if (cudaMemsetAsync(d_lo, 0xFF, 8 * nchunks, st) != cudaSuccess ||
      cudaMemsetAsync(d_hi, 0, 8 * nchunks, st) != cudaSuccess)
    return LH_ECUDA;
  const uint64_t per = chunk_msgs < n ? chunk_msgs : n;
  const uint64_t slices = (per + kSlice - 1) / kSlice;
  if (slices > 0x7fffffffull) return LH_ETOOBIG;
  k_ragged_plan<<<dim3((unsigned)slices, (unsigned)nchunks), kPlanThreads, 0, st>>>(
      d_offsets, d_lengths, n, chunk_msgs, buf_len, (unsigned long long*)d_lo,
      (unsigned long long*)d_hi, (unsigned long long*)d_bad);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}
