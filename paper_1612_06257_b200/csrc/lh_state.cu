// lh_state.cu — HighwayHash's state-level primitives on caller states, and
// a device self-test of the Update bijection (SURVEY.md §8a rows a2, a4, a5,
// a10 exposed one by one, as the reference module exposes them).
//
//   update           S/highway.py:130-150  (lh::Highway::update, the hot-path code)
//   update_inverse   S/highway.py:153-173  (lh::Highway::update_inverse)
//   update_remainder S/highway.py:182-199  (lh::Highway::remainder)
//   finalize         S/highway.py:223-234  (lh::Highway::finalize_rounds + lane sums)
//   sip_round        S/sip.py:73-86        (lh::sip_round, the SipHash kernels' round)
//
// The reference uses update_inverse only as a test oracle: the permutation
// check of T/test_update.py:56-67 and the acceptance gate
// T/test_acceptance.py:42-63 (100,000 round trips in < 5 s).  Here the same
// check runs on the device over any number of synthetic states, through the
// exact Update the hashing kernels inline.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lanehash_b200.h"
#include "lh_device.cuh"
#include "lh_mix.cuh"

using namespace lh;

namespace {

__device__ __forceinline__ void load_state(Highway& h, const u64* s) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h.v0[i] = s[i];
    h.v1[i] = s[4 + i];
    h.m0[i] = s[8 + i];
    h.m1[i] = s[12 + i];
  }
}

__device__ __forceinline__ void store_state(const Highway& h, u64* s) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s[i] = h.v0[i];
    s[4 + i] = h.v1[i];
    s[8 + i] = h.m0[i];
    s[12 + i] = h.m1[i];
  }
}

template <bool INV>
__global__ void k_update_states(u64* __restrict__ states, const u64* __restrict__ packets, u64 n,
                                u32 one) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    Highway h;
    h.one = one;
    load_state(h, states + 16 * i);
    const u64 p[4] = {packets[4 * i], packets[4 * i + 1], packets[4 * i + 2], packets[4 * i + 3]};
    if (INV)
      h.update_inverse(p);
    else
      h.update(p[0], p[1], p[2], p[3]);
    store_state(h, states + 16 * i);
  }
}

// S/highway.py:182-199 on caller states: tail i is tails[32i .. 32i+r_i)
// (bytes beyond r_i are ignored), r_i in 1..31; other r_i leave state i as is.
__global__ void k_remainder_states(u64* __restrict__ states, const uint8_t* __restrict__ tails,
                                   const u32* __restrict__ rs, u64 n, u32 one) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    const u32 r = rs[i];
    if (r == 0 || r >= 32) continue;
    Highway h;
    h.one = one;
    load_state(h, states + 16 * i);
    u64 t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u64 w = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) w |= (u64)tails[32 * i + 8 * k + b] << (8 * b);
      t[k] = w;
    }
    h.remainder(t, r);
    store_state(h, states + 16 * i);
  }
}

// S/highway.py:223-234 on caller states: `rounds` PermuteAndUpdates, then
// width/64 lane sums per state (lane 0 first).
__global__ void k_finalize_states(const u64* __restrict__ states, u64 n, int width, int rounds,
                                  u32 one, u64* __restrict__ out) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    Highway h;
    h.one = one;
    h.rounds = rounds;
    h.width = width;
    load_state(h, states + 16 * i);
    h.finalize_rounds();
    const int W = width / 64;
    for (int k = 0; k < W; ++k) {
      const u64 v0 = k == 0 ? h.v0[0] : k == 1 ? h.v0[1] : k == 2 ? h.v0[2] : h.v0[3];
      const u64 v1 = k == 0 ? h.v1[0] : k == 1 ? h.v1[1] : k == 2 ? h.v1[2] : h.v1[3];
      const u64 m0 = k == 0 ? h.m0[0] : k == 1 ? h.m0[1] : k == 2 ? h.m0[2] : h.m0[3];
      const u64 m1 = k == 0 ? h.m1[0] : k == 1 ? h.m1[1] : k == 2 ? h.m1[2] : h.m1[3];
      out[i * W + k] = v0 + v1 + m0 + m1;
    }
  }
}

// S/sip.py:73-86: `rounds` SipRounds on n caller states (4 lanes each).
__global__ void k_sip_round_states(u64* __restrict__ states, u64 n, int rounds, SipMul k) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    u64 v0 = states[4 * i], v1 = states[4 * i + 1], v2 = states[4 * i + 2],
        v3 = states[4 * i + 3];
    sip_rounds<0>(v0, v1, v2, v3, k, rounds);  // both round variants, alternating
    states[4 * i] = v0;
    states[4 * i + 1] = v1;
    states[4 * i + 2] = v2;
    states[4 * i + 3] = v3;
  }
}

// Case i = words 20i .. 20i+19 of the synthetic stream: 16 state lanes, then
// 4 packet lanes.  result[0] += failures, result[1] ^= fold of update(s).
__global__ void k_bijectivity(u64 key, u64 n, u32 one, unsigned long long* result) {
  u64 fails = 0, fold = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    u64 s[16], p[4];
#pragma unroll
    for (int j = 0; j < 16; ++j) s[j] = synth_word(key, 20 * i + j);
#pragma unroll
    for (int j = 0; j < 4; ++j) p[j] = synth_word(key, 20 * i + 16 + j);
    Highway h;
    h.one = one;
    load_state(h, s);
    h.update(p[0], p[1], p[2], p[3]);
#pragma unroll
    for (int j = 0; j < 4; ++j) fold ^= h.v0[j] ^ h.v1[j] ^ h.m0[j] ^ h.m1[j];
    h.update_inverse(p);
    u64 diff = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      diff |= (h.v0[j] ^ s[j]) | (h.v1[j] ^ s[4 + j]) | (h.m0[j] ^ s[8 + j]) | (h.m1[j] ^ s[12 + j]);
    fails += diff != 0;
  }
  // Warp-reduce, then one atomic per warp.
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fails += __shfl_xor_sync(0xffffffffu, fails, o);
    fold ^= __shfl_xor_sync(0xffffffffu, fold, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (fails) atomicAdd(&result[0], (unsigned long long)fails);
    atomicXor(&result[1], (unsigned long long)fold);
  }
}

unsigned grid_for(u64 items, int sms) {
  const u64 b = (items + 255) / 256;
  const u64 cap = (u64)sms * 8;
  return (unsigned)(b == 0 ? 1 : (b > cap ? cap : b));
}

int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

extern "C" {

int lh_highway_update_states(uint64_t* d_states, const uint64_t* d_packets, uint64_t n,
                             int inverse, void* stream) {
  if (n && (!d_states || !d_packets)) return LH_EINVAL;
  if (inverse != 0 && inverse != 1) return LH_EINVAL;
  if ((uintptr_t)d_states % 8 || (uintptr_t)d_packets % 8) return LH_EALIGN;
  if (!n) return LH_OK;
  const unsigned g = grid_for(n, sm_count());
  cudaStream_t st = (cudaStream_t)stream;
  if (inverse)
    k_update_states<true><<<g, 256, 0, st>>>(d_states, d_packets, n, 1u);
  else
    k_update_states<false><<<g, 256, 0, st>>>(d_states, d_packets, n, 1u);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}

int lh_highway_remainder_states(uint64_t* d_states, const uint8_t* d_tails,
                                const uint32_t* d_r, uint64_t n, void* stream) {
  if (n && (!d_states || !d_tails || !d_r)) return LH_EINVAL;
  if ((uintptr_t)d_states % 8 || (uintptr_t)d_r % 4) return LH_EALIGN;
  if (!n) return LH_OK;
  k_remainder_states<<<grid_for(n, sm_count()), 256, 0, (cudaStream_t)stream>>>(
      d_states, d_tails, d_r, n, 1u);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}

int lh_highway_finalize_states(const uint64_t* d_states, uint64_t n, int width, int rounds,
                               uint64_t* d_out, void* stream) {
  if (width != 64 && width != 128 && width != 256) return LH_EINVAL;
  if (rounds < 0) return LH_EINVAL;
  if (n && (!d_states || !d_out)) return LH_EINVAL;
  if ((uintptr_t)d_states % 8 || (uintptr_t)d_out % 8) return LH_EALIGN;
  if (!n) return LH_OK;
  k_finalize_states<<<grid_for(n, sm_count()), 256, 0, (cudaStream_t)stream>>>(
      d_states, n, width, rounds, 1u, d_out);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}

int lh_sip_round_states(uint64_t* d_states, uint64_t n, int rounds, void* stream) {
  if (rounds < 0 || (n && !d_states)) return LH_EINVAL;
  if ((uintptr_t)d_states % 8) return LH_EALIGN;
  if (!n || !rounds) return LH_OK;
  const SipMul k = {1u, 1u << 13, 1u << 17, 1u << 16};
  k_sip_round_states<<<grid_for(n, sm_count()), 256, 0, (cudaStream_t)stream>>>(d_states, n,
                                                                                rounds, k);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}

int lh_highway_bijectivity(uint64_t seed, uint64_t n, uint64_t* d_result, void* stream) {
  if (!d_result) return LH_EINVAL;
  if ((uintptr_t)d_result % 8) return LH_EALIGN;
  if (!n) return LH_OK;
  const unsigned g = grid_for(n, sm_count());
  k_bijectivity<<<g, 256, 0, (cudaStream_t)stream>>>(synth_key(seed, 0), n, 1u,
                                                      (unsigned long long*)d_result);
  return cudaGetLastError() == cudaSuccess ? LH_OK : LH_ECUDA;
}

}  // extern "C"
