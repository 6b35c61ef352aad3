// Read-bandwidth ceilings on this B200 (tuning tool, not product):
//   1. LDG.128 grid-stride streaming read (XOR-reduce)
//   2. TMA 2-D box ring, CTA-wide (ROWS x 128 B boxes), null consumer
//   3. same with per-warp rings (32 x 128 B boxes)
//   4. D2D cudaMemcpy (read+write)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/membench tools/membench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../paper_1612_06257_b200/csrc/lh_tma.cuh"
using namespace lh;

__global__ void k_ldg(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldg(p + i), b = __ldg(p + i + stride), c = __ldg(p + i + 2 * stride), d = __ldg(p + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n16; i += stride) acc ^= __ldg(p + i).x;
  if (acc == 0x12345678) out[0] = acc;
}

template <int ROWS, int STAGES>
__global__ void __launch_bounds__(ROWS + 32) k_tma_cta(const __grid_constant__ CUtensorMap tmap, uint64_t n, uint64_t len, unsigned* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  constexpr uint32_t SB = ROWS * 128;
  uint64_t* full = (uint64_t*)(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], ROWS / 32); } fence_mbar_init(); }
  __syncthreads();
  uint64_t ntiles = (n + ROWS - 1) / ROWS; uint32_t nch = (len + 127) / 128;
  if (warp == ROWS / 32) {
    if (lane == 0) { uint32_t it = 0;
      for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) for (uint32_t c = 0; c < nch; ++c, ++it) {
        uint32_t s = it % STAGES, ph = (it / STAGES) & 1; mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], SB); tma_load_2d(smem + s * SB, &tmap, c * 128, t * ROWS, &full[s]); } }
    return;
  }
  uint32_t acc = 0, it = 0; uint32_t base = smem_u32(smem) + threadIdx.x * 128;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) for (uint32_t c = 0; c < nch; ++c, ++it) {
    uint32_t s = it % STAGES, ph = (it / STAGES) & 1; mbar_wait(&full[s], ph);
    uint4 a = lds128(base + s * SB); acc ^= a.x;
    __syncwarp(); if (lane == 0) mbar_arrive(&empty[s]); }
  if (acc == 0x12345678) out[0] = acc;
}

template <int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32) k_tma_warp(const __grid_constant__ CUtensorMap tmap, uint64_t n, uint64_t len, unsigned* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * STAGES * 4096;
  uint64_t* bar = (uint64_t*)(smem + WARPS * STAGES * 4096) + warp * STAGES;
  uint64_t ntiles = (n + 31) / 32; uint32_t nch = (len + 127) / 128;
  uint64_t g = (uint64_t)blockIdx.x * WARPS + warp, G = (uint64_t)gridDim.x * WARPS;
  uint64_t mine = g < ntiles ? (ntiles - g + G - 1) / G : 0, total = mine * nch;
  if (lane == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1); fence_mbar_init(); }
  __syncwarp();
  uint64_t itile = g; uint32_t ich = 0;
  auto issue = [&](uint32_t s) { mbar_arrive_expect_tx(&bar[s], 4096); tma_load_2d(ring + s * 4096, &tmap, ich * 128, itile * 32, &bar[s]); if (++ich == nch) { ich = 0; itile += G; } };
  if (lane == 0) for (uint32_t s = 0; s < STAGES && s < total; ++s) issue(s);
  uint32_t acc = 0, s = 0, ph = 0; uint32_t base = smem_u32(ring) + lane * 128;
  for (uint64_t i = 0; i < total; ++i) {
    mbar_wait(&bar[s], ph); uint4 a = lds128(base + s * 4096); acc ^= a.x; __syncwarp();
    if (lane == 0 && i + STAGES < total) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(s); }
    if (++s == STAGES) { s = 0; ph ^= 1; } }
  if (acc == 0x12345678) out[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static CUtensorMap make_map(void* p, uint64_t n, uint64_t len, uint32_t rows) {
  CUtensorMap m; cuuint64_t dims[2] = {len, n}; cuuint64_t str[1] = {len}; cuuint32_t box[2] = {128, rows}; cuuint32_t es[2] = {1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) printf("encode failed\n");
  return m;
}

template <class F> static float timeit(F f, int reps = 10) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for (int i = 0; i < reps; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}

int main() {
  void* pfn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &pfn, cudaEnableDefault, &q); enc = (PFN_cuTensorMapEncodeTiled_v12000)pfn;
  const uint64_t L = 1024, N = 1ull << 24; const size_t bytes = N * L;
  uint8_t* d; cudaMalloc(&d, bytes); cudaMemset(d, 1, bytes); unsigned* o; cudaMalloc(&o, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char* name, float ms) { printf("%-28s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6); };
  for (int bpsm : {2, 4, 8}) for (int thr : {256, 512}) {
    char nm[64]; snprintf(nm, 64, "ldg128 %dx%d", bpsm, thr);
    rep(nm, timeit([&] { k_ldg<<<sms * bpsm, thr>>>((const uint4*)d, bytes / 16, o); }));
  }
  {
    CUtensorMap m = make_map(d, N, L, 256);
    size_t sm = 1024 + 3 * 256 * 128 + 64; cudaFuncSetAttribute(k_tma_cta<256, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    rep("tma cta 256x3 (2/SM)", timeit([&] { k_tma_cta<256, 3><<<sms * 2, 288, sm>>>(m, N, L, o); }));
  }
  {
    CUtensorMap m = make_map(d, N, L, 128);
    size_t sm = 1024 + 4 * 128 * 128 + 64; cudaFuncSetAttribute(k_tma_cta<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    rep("tma cta 128x4 (3/SM)", timeit([&] { k_tma_cta<128, 4><<<sms * 3, 160, sm>>>(m, N, L, o); }));
  }
  {
    CUtensorMap m = make_map(d, N, L, 32);
    size_t sm = 1024 + 8 * 3 * 4096 + 8 * 3 * 8; cudaFuncSetAttribute(k_tma_warp<8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    rep("tma warp 8x3 (2/SM)", timeit([&] { k_tma_warp<8, 3><<<sms * 2, 256, sm>>>(m, N, L, o); }));
    size_t sm2 = 1024 + 4 * 6 * 4096 + 4 * 6 * 8; cudaFuncSetAttribute(k_tma_warp<4, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    rep("tma warp 4x6 (2/SM)", timeit([&] { k_tma_warp<4, 6><<<sms * 2, 128, sm2>>>(m, N, L, o); }));
  }
  uint8_t* d2; if (cudaMalloc(&d2, bytes / 2) == cudaSuccess) {
    float ms = timeit([&] { cudaMemcpyAsync(d2, d, bytes / 2, cudaMemcpyDeviceToDevice); });
    printf("%-28s %8.3f ms  %8.1f GB/s (read+write)\n", "memcpy d2d 8 GiB", ms, bytes / ms / 1e6);
  }
  cudaError_t e = cudaDeviceSynchronize(); printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
