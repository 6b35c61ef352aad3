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
//
// lh_ragged_plan_stats adds the lane balance of the natural order: with
// work(i) = (len_i >> unit_shift) + fixed_units (packets or words, plus the
// per-message finalization), stats[0] = sum of work and stats[1] = sum over
// the groups of 32 consecutive messages of 32 * max work -- what a kernel
// with one message per lane spends.  stats[0] / stats[1] is the warp
// efficiency; the host orders the batch by length class (lh_ragged_order)
// when it is low.
//
// lh_ragged_order: a counting sort of the messages by length class into
// 16-byte schedule records {offset, length, index}, longest class first (classes: work units up to 127 exactly, then 8 steps
// per octave, so lanes of one class differ by < 12.5%).  Three launches:
// histogram, scan, scatter.  The order inside a class is arbitrary (atomic
// cursors); digests are written by message index, so results do not depend
// on it.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lanehash_b200.h"

namespace {

constexpr unsigned kPlanThreads = 256;
constexpr uint64_t kSlice = 4096;

__global__ void __launch_bounds__(kPlanThreads)
    k_ragged_plan(const uint64_t* __restrict__ off, const uint32_t* __restrict__ lens, uint64_t n,
                  uint64_t chunk_msgs, uint64_t buf_len, unsigned long long* __restrict__ lo,
                  unsigned long long* __restrict__ hi, unsigned long long* __restrict__ bad,
                  unsigned long long* __restrict__ stats, unsigned unit_shift,
                  unsigned fixed_units) {
  const uint64_t c = blockIdx.y;
  const uint64_t c0 = c * chunk_msgs;
  const uint64_t c1 = c0 + chunk_msgs < n ? c0 + chunk_msgs : n;
  const uint64_t s0 = c0 + (uint64_t)blockIdx.x * kSlice;
  const uint64_t s1 = s0 + kSlice < c1 ? s0 + kSlice : c1;
  unsigned long long mn = ~0ull, mx = 0;
  unsigned nbad = 0;
  unsigned long long wsum = 0, wmax32 = 0;  // stats (lane 0 accumulates wmax32)
  for (uint64_t i0 = s0; i0 < s1; i0 += kPlanThreads) {
    const uint64_t i = i0 + threadIdx.x;
    unsigned long long work = 0;
    if (i < s1) {
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
      work = ok ? ((end - start) >> unit_shift) + fixed_units : 0;
    }
    if (stats) {  // uniform branch; every lane of the warp reaches the reduction
      const unsigned w32 = work < 0xFFFFFFFFull ? (unsigned)work : 0xFFFFFFFFu;
      wsum += w32;
      wmax32 += 32ull * __reduce_max_sync(0xffffffffu, w32);
    }
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
  if (stats) {  // one pair of global atomics per block
    __shared__ unsigned long long acc[2];
    if (threadIdx.x == 0) acc[0] = acc[1] = 0;
    __syncthreads();
#pragma unroll
    for (int s = 16; s; s >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, s);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&acc[0], wsum);
      atomicAdd(&acc[1], wmax32);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(&stats[0], acc[0]);
      atomicAdd(&stats[1], acc[1]);
    }
  }
}

constexpr unsigned kClasses = 512;

// Length class of `units` work units: exact below 128, then 8 per octave.
__device__ __forceinline__ unsigned length_class(uint64_t units) {
  if (units < 128) return (unsigned)units;
  if (units > 0x7fffffffull) units = 0x7fffffffull;
  const unsigned u = (unsigned)units, e = 31 - __clz(u);  // e >= 7
  return 128 + (e - 7) * 8 + ((u >> (e - 3)) & 7);         // <= 128 + 23 * 8 + 7 = 319
}

__device__ __forceinline__ uint64_t msg_len(const uint64_t* off, const uint32_t* lens,
                                            uint64_t i) {
  return lens ? (uint64_t)lens[i] : off[i + 1] - off[i];
}

__global__ void __launch_bounds__(256)
    k_order_hist(const uint64_t* __restrict__ off, const uint32_t* __restrict__ lens, uint64_t n,
                 unsigned unit_shift, unsigned* __restrict__ hist) {
  __shared__ unsigned h[kClasses];
  for (unsigned c = threadIdx.x; c < kClasses; c += 256) h[c] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256)
    atomicAdd(&h[length_class(msg_len(off, lens, i) >> unit_shift)], 1u);
  __syncthreads();
  for (unsigned c = threadIdx.x; c < kClasses; c += 256)
    if (h[c]) atomicAdd(&hist[c], h[c]);
}

// cursor[c] = number of messages in classes above c (longest first): a
// block-wide suffix sum of the 512 counters.
__global__ void __launch_bounds__(kClasses)
    k_order_scan(const unsigned* __restrict__ hist, unsigned* __restrict__ cursor) {
  __shared__ unsigned wsum[kClasses / 32];
  const unsigned c = kClasses - 1 - threadIdx.x;  // thread 0 = the longest class
  const unsigned v = hist[c], lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const unsigned o = __shfl_up_sync(0xffffffffu, inc, s);
    if (lane >= (unsigned)s) inc += o;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  unsigned before = 0;
  for (unsigned k = 0; k < w; ++k) before += wsum[k];
  cursor[c] = before + inc - v;
}

constexpr int kOrderPer = 8;  // messages per thread: 2,048 per block

__global__ void __launch_bounds__(256)
    k_order_scatter(const uint64_t* __restrict__ off, const uint32_t* __restrict__ lens,
                    uint64_t n, unsigned unit_shift, unsigned* __restrict__ cursor,
                    uint4* __restrict__ sched) {
  __shared__ unsigned cnt[kClasses], base[kClasses];
  for (unsigned c = threadIdx.x; c < kClasses; c += 256) cnt[c] = 0;
  __syncthreads();
  const uint64_t b0 = (uint64_t)blockIdx.x * 256 * kOrderPer;
  unsigned cls[kOrderPer], rank[kOrderPer];
  uint64_t start[kOrderPer], len[kOrderPer];
#pragma unroll
  for (int k = 0; k < kOrderPer; ++k) {
    const uint64_t i = b0 + (uint64_t)k * 256 + threadIdx.x;
    cls[k] = kClasses;
    if (i < n) {
      start[k] = off[i];
      len[k] = lens ? (uint64_t)lens[i] : off[i + 1] - start[k];
      cls[k] = length_class(len[k] >> unit_shift);
      rank[k] = atomicAdd(&cnt[cls[k]], 1u);
    }
  }
  __syncthreads();
  for (unsigned c = threadIdx.x; c < kClasses; c += 256)
    if (cnt[c]) base[c] = atomicAdd(&cursor[c], cnt[c]);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kOrderPer; ++k)
    if (cls[k] < kClasses) {
      // {offset, length (saturated: 0xFFFFFFFF = read it from the layout), index}
      const uint32_t l32 = len[k] < 0xFFFFFFFFull ? (uint32_t)len[k] : 0xFFFFFFFFu;
      sched[base[cls[k]] + rank[k]] =
          make_uint4((uint32_t)start[k], (uint32_t)(start[k] >> 32), l32,
                     (uint32_t)(b0 + (uint64_t)k * 256 + threadIdx.x));
    }
}

}  // namespace

extern "C" int lh_ragged_plan_stats(const uint64_t* d_offsets, const uint32_t* d_lengths,
                                    uint64_t n, uint64_t chunk_msgs, uint64_t buf_len,
                                    uint64_t* d_lo, uint64_t* d_hi, uint64_t* d_bad,
                                    uint64_t* d_stats, unsigned unit_shift, unsigned fixed_units,
                                    void* stream) {
  if (!d_bad || (n && (!d_offsets || !d_lo || !d_hi || chunk_msgs == 0)) || unit_shift > 31)
    return LH_EINVAL;
  if ((uintptr_t)d_offsets % 8 || (uintptr_t)d_lengths % 4 || (uintptr_t)d_lo % 8 ||
      (uintptr_t)d_hi % 8 || (uintptr_t)d_bad % 8 || (uintptr_t)d_stats % 8)
    return LH_EALIGN;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t nchunks = n ? (n + chunk_msgs - 1) / chunk_msgs : 0;
  if (nchunks > 65535) return LH_ETOOBIG;
  if (cudaMemsetAsync(d_bad, 0, 8, st) != cudaSuccess) return LH_ECUDA;
  if (d_stats && cudaMemsetAsync(d_stats, 0, 16, st) != cudaSuccess) return LH_ECUDA;
  if (!n) return LH_OK;
  if (cudaMemsetAsync(d_lo, 0xFF, 8 * nchunks, st) != cudaSuccess ||
      cudaMemsetAsync(d_hi, 0, 8 * nchunks, st) != cudaSuccess)
    return LH_ECUDA;
  const uint64_t per = chunk_msgs < n ? chunk_msgs : n;
  const uint64_t slices = (per + kSlice - 1) / kSlice;
  if (slices > 0x7fffffffull) return LH_ETOOBIG;
  k_ragged_plan<<<dim3((unsigned)slices, (unsigned)nchunks), kPlanThreads, 0, st>>>(
      d_offsets, d_lengths, n, chunk_msgs, buf_len, (unsigned long long*)d_lo,
      (unsigned long long*)d_hi, (unsigned long long*)d_bad, (unsigned long long*)d_stats,
      unit_shift, fixed_units);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}

extern "C" int lh_ragged_plan(const uint64_t* d_offsets, const uint32_t* d_lengths, uint64_t n,
                              uint64_t chunk_msgs, uint64_t buf_len, uint64_t* d_lo,
                              uint64_t* d_hi, uint64_t* d_bad, void* stream) {
  return lh_ragged_plan_stats(d_offsets, d_lengths, n, chunk_msgs, buf_len, d_lo, d_hi, d_bad,
                              nullptr, 0, 0, stream);
}

extern "C" int lh_ragged_order(const uint64_t* d_offsets, const uint32_t* d_lengths, uint64_t n,
                               unsigned unit_shift, void* d_sched, uint32_t* d_scratch,
                               void* stream) {
  if ((n && (!d_offsets || !d_sched)) || !d_scratch || unit_shift > 31) return LH_EINVAL;
  if ((uintptr_t)d_offsets % 8 || (uintptr_t)d_lengths % 4 || (uintptr_t)d_sched % 16 ||
      (uintptr_t)d_scratch % 4)
    return LH_EALIGN;
  if (n > 0xFFFFFFFFull) return LH_ETOOBIG;
  if (!n) return LH_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned* hist = d_scratch;
  unsigned* cursor = d_scratch + kClasses;
  if (cudaMemsetAsync(hist, 0, sizeof(unsigned) * kClasses, st) != cudaSuccess) return LH_ECUDA;
  const uint64_t hb = (n + 2047) / 2048;
  k_order_hist<<<(unsigned)(hb < 1184 ? hb : 1184), 256, 0, st>>>(d_offsets, d_lengths, n,
                                                                   unit_shift, hist);
  k_order_scan<<<1, kClasses, 0, st>>>(hist, cursor);
  k_order_scatter<<<(unsigned)((n + 256 * kOrderPer - 1) / (256 * kOrderPer)), 256, 0, st>>>(
      d_offsets, d_lengths, n, unit_shift, cursor, (uint4*)d_sched);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}
