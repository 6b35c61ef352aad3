// latency.cu — dependent-issue latency (clocks per instruction in a single
// dependent chain, one warp per SM sub-partition) of the instruction
// sequences on the HighwayHash Update's critical chain.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/latency tools/latency.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include "../paper_1612_06257_b200/csrc/lh_device.cuh"
using namespace lh;

enum { L_IADD3, L_LOP3, L_PRMT, L_SHF, L_IMAD, L_WIDE, L_ADD64M, L_ADD64, L_ADD64_3IN, L_ZIP_ADD, L_N };
static const char* kName[L_N] = {"iadd3", "lop3", "prmt", "shf", "imad", "imad_wide", "add64_iadd3_imadx",
                                 "add64_iadd3_iadd3x", "add64_3input", "zipper_plus_add64"};
static const int kSteps[L_N] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1};

template <int M>
__global__ void k_lat(u64* out, u64 seed, u32 one, int iters) {
  u64 x = seed * (threadIdx.x + 1), y = seed ^ 0x9E3779B97F4A7C15ull, z = seed + 77;
  u32 a = (u32)x, b = (u32)y | 1u;
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (M == L_IADD3) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b));
      if (M == L_LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6A;" : "+r"(a) : "r"(b), "r"(one));
      if (M == L_PRMT) asm volatile("prmt.b32 %0, %0, %1, 0x5041;" : "+r"(a) : "r"(b));
      if (M == L_SHF) asm volatile("shf.l.wrap.b32 %0, %0, %0, 13;" : "+r"(a));
      if (M == L_IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(one));
      if (M == L_WIDE) { x = mul_lo_hi(x, y) ^ 0; x = pack(lo32(x), hi32(x) | 1u); }
      if (M == L_ADD64M) x = add64_mixed(x, y, one);
      if (M == L_ADD64) {
        u32 lo, hi;
        asm volatile("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;" : "=r"(lo), "=r"(hi)
                     : "r"(lo32(x)), "r"(lo32(y)), "r"(hi32(x)), "r"(hi32(y)));
        x = pack(lo, hi);
      }
      if (M == L_ADD64_3IN) x = x + y + z;
      if (M == L_ZIP_ADD) {  // zipper of (x, y) then a 64-bit add into x: one chain link of the Update
        u64 z0, z1;
        zipper(x, y, z0, z1);
        x = add64_mixed(x, z0, one);
        y = add64_mixed(y, z1, one);
      }
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (u64)(t1 - t0);
  if ((x ^ y ^ a) == 0x1234567ull) out[0] = x;
}

template <int M>
static void run(u64* d, int sms) {
  const int iters = 4096;
  u64 h = 0;
  double best = 1e30;
  for (int r = 0; r < 3; ++r) {
    k_lat<M><<<sms, 128>>>(d, 0x1234567ull + r, 1, iters);  // 4 warps per SM: one per sub-partition
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    best = (double)h < best ? (double)h : best;
  }
  printf("%s\"%s\": %.2f", M ? ", " : "", kName[M], best / (iters * 16.0 * kSteps[M]));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  u64* d;
  cudaMalloc(&d, 8 * sms);
  printf("{\"unit\": \"clocks per dependent step, one warp per sub-partition\", ");
  run<L_IADD3>(d, sms); run<L_LOP3>(d, sms); run<L_PRMT>(d, sms); run<L_SHF>(d, sms); run<L_IMAD>(d, sms);
  run<L_WIDE>(d, sms); run<L_ADD64M>(d, sms); run<L_ADD64>(d, sms); run<L_ADD64_3IN>(d, sms); run<L_ZIP_ADD>(d, sms);
  printf(", \"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
