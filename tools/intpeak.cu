// intpeak.cu — integer-pipe ceilings on this B200 (tuning/roofline tool).
//
//  1. alu:   independent LOP3/IADD3 chains (ALU pipe)       -> warp-instr/s
//  2. prmt:  independent PRMT chains (ALU pipe)              -> warp-instr/s
//  3. imadx: IMAD with carry chains (FMA pipe)               -> warp-instr/s
//  4. wide:  IMAD.WIDE.U32 chains (FMA-heavy)                -> warp-instr/s
//  5. update: the engine's HighwayHash Update (lh_device.cuh) on registers
//     only, 1 thread per message, no memory traffic         -> Updates/s
// The last number is the INT roof of the hash path: a launch of U Updates
// can not finish faster than U / (Updates/s).  Prints JSON.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/intpeak tools/intpeak.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_1612_06257_b200/csrc/lh_device.cuh"
#include "../paper_1612_06257_b200/csrc/lh_host.cuh"

using namespace lh;

__global__ void k_alu(u32* out, u32 seed, int iters) {
  u32 a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed ^ (threadIdx.x * 8 + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a[k] = (a[k] ^ (a[(k + 1) & 7] + 0x9E3779B9u)) + a[(k + 3) & 7];
    }
  }
  u32 s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= a[k];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_prmt(u32* out, u32 seed, int iters) {
  u32 a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed ^ (threadIdx.x * 8 + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __byte_perm(a[k], a[(k + 1) & 7], 0x5041);
  }
  u32 s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= a[k];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_wide(u64* out, u32 seed, int iters) {
  u64 a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 8 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = mul_lo_hi(a[k], a[(k + 5) & 7] | (1ull << 40));
  }
  u64 s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= a[k];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_imadx(u64* out, u32 seed, u32 one, int iters) {
  u64 a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 8 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = add64_mixed(a[k], a[(k + 3) & 7], one);
  }
  u64 s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= a[k];
  if (s == 0x12345678u) out[0] = s;
}

// Packets come from shared memory with the same LDS.128 pattern as the
// TMA kernel (2 per Update), so the SASS mix matches the real hot loop
// minus the HBM stream.
__global__ void __launch_bounds__(256) k_update(const Highway proto, u64* out, int iters) {
  __shared__ uint4 pk[8][256];
  for (int j = 0; j < 8; ++j)
    pk[j][threadIdx.x] = make_uint4(threadIdx.x * 16 + j, blockIdx.x, j * 77, ~threadIdx.x);
  __syncthreads();
  Highway h = proto;
  for (int i = 0; i < iters; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint4 a = pk[j][threadIdx.x], b = pk[(j + 3) & 7][threadIdx.x];
      h.update(pack(a.x, a.y), pack(a.z, a.w), pack(b.x, b.y), pack(b.z, b.w));
    }
  }
  u64 s = 0;  // every lane must reach the output or ptxas drops lanes 2,3
#pragma unroll
  for (int k = 0; k < 4; ++k) s ^= h.v0[k] + h.v1[k] + h.m0[k] + h.m1[k];
  if (s == 0x12345678ull) out[0] = s;
}

template <class F>
static float time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  u64* d;
  cudaMalloc(&d, 64);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  const double warps = (double)blocks * threads / 32;
  const double alu_instr = warps * iters * 8 * 2;  // LOP3 + IADD3 per chain step
  float ms = time_ms([&] { k_alu<<<blocks, threads>>>((u32*)d, 7, iters); });
  const double alu = alu_instr / (ms * 1e-3);
  ms = time_ms([&] { k_prmt<<<blocks, threads>>>((u32*)d, 7, iters); });
  const double prmt = warps * iters * 8 / (ms * 1e-3);
  ms = time_ms([&] { k_wide<<<blocks, threads>>>(d, 7, iters); });
  const double wide = warps * iters * 8 / (ms * 1e-3);
  ms = time_ms([&] { k_imadx<<<blocks, threads>>>(d, 7, 1, iters); });
  const double addm = warps * iters * 8 / (ms * 1e-3);  // IADD3 + IMAD.X pairs
  const u64 key[4] = {1, 2, 3, 4};
  const Highway proto = make_highway(key, 64, 4);
  int ublocks = sms * 2;  // 16 warps per SM, as the bench kernel
  const int uiters = 8192;
  ms = time_ms([&] { k_update<<<ublocks, 256>>>(proto, d, uiters); });
  const double updates = (double)ublocks * 256 * uiters / (ms * 1e-3);
  printf("{\"sms\": %d, \"clock_khz_attr\": %d,\n", sms, clk_khz);
  printf(" \"alu_warp_instr_per_s\": %.4e, \"alu_lane_ops_per_s\": %.4e,\n", alu, alu * 32);
  printf(" \"prmt_warp_instr_per_s\": %.4e,\n", prmt);
  printf(" \"imad_wide_warp_instr_per_s\": %.4e,\n", wide);
  printf(" \"add64_mixed_pairs_warp_per_s\": %.4e,\n", addm);
  printf(" \"highway_updates_per_s\": %.4e,\n", updates);
  printf(" \"canonical_ops_per_update\": 80, \"ops_per_s\": %.4e,\n", updates * 80);
  printf(" \"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
