/* C caller of the engine's ABI (include/lanehash_b200.h) with the CUDA
 * runtime only: hashes the reference's frozen ramp vectors
 * (T/test_highway.py:32-50) and the published SipHash-2-4 vectors
 * (T/test_sip.py:19-36, first 8) and prints PASS/FAIL per check.
 * Build: see __graft_entry__.build() (gcc + -lcudart). */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "lanehash_b200.h"

static const struct { unsigned len; uint64_t digest; } kFrozen64[] = {
    {0, 0x907A56DE22C26E53ull},  {1, 0x7EAB43AAC7CDDD78ull},  {3, 0x9705CD8B7EEFA20Bull},
    {4, 0xF205A46893007EDAull},  {31, 0x8053546F9076FC43ull}, {32, 0xA0C964D9ECD580FCull},
    {33, 0x1BF7E3CB13A96183ull}, {63, 0xF9742F53750C795Bull}, {64, 0x75542C5D4CD2A6FFull},
    {1024, 0x7787F312AF72EDD3ull}};
static const uint64_t kSip24[8] = {0x726fdb47dd0e0e31ull, 0x74f839c593dc67fdull,
                                   0x0d6c8009d9a94f5aull, 0x85676696d7fb7e2dull,
                                   0xcf2794e0277187b7ull, 0x18765564cd99a68dull,
                                   0xcbc9466e58fee3ceull, 0xab0200f58b01d137ull};

int main(void) {
  uint8_t msg[1024];
  for (int i = 0; i < 1024; ++i) msg[i] = (uint8_t)i;
  uint64_t key4[4], key2[2];
  memcpy(key4, msg, 32); /* ramp key, little-endian lanes */
  memcpy(key2, msg, 16);
  uint8_t* d_msg;
  uint64_t* d_out;
  if (cudaMalloc((void**)&d_msg, 1024) != cudaSuccess || cudaMalloc((void**)&d_out, 64) != cudaSuccess) {
    printf("FAIL cudaMalloc\n");
    return 2;
  }
  cudaMemcpy(d_msg, msg, 1024, cudaMemcpyHostToDevice);
  int fails = 0;
  printf("%s\n", lh_version());
  for (unsigned k = 0; k < sizeof kFrozen64 / sizeof kFrozen64[0]; ++k) {
    uint64_t got = 0;
    int rc = lh_highway_fixed(d_msg, 1, kFrozen64[k].len, key4, 64, 4, d_out, NULL);
    cudaMemcpy(&got, d_out, 8, cudaMemcpyDeviceToHost);
    const int ok = rc == LH_OK && got == kFrozen64[k].digest;
    fails += !ok;
    printf("%s highway64 len=%u rc=%d got=%016llx\n", ok ? "PASS" : "FAIL", kFrozen64[k].len, rc,
           (unsigned long long)got);
  }
  for (unsigned len = 0; len < 8; ++len) {
    uint64_t got = 0;
    int rc = lh_siphash_fixed(d_msg, 1, len, key2, 2, 4, 0, d_out, NULL);
    cudaMemcpy(&got, d_out, 8, cudaMemcpyDeviceToHost);
    const int ok = rc == LH_OK && got == kSip24[len];
    fails += !ok;
    printf("%s siphash24 len=%u rc=%d\n", ok ? "PASS" : "FAIL", len, rc);
  }
  /* argument validation maps to LH_EINVAL like the reference's ValueError */
  const int bad = lh_highway_fixed(d_msg, 1, 8, key4, 96, 4, d_out, NULL);
  fails += bad != LH_EINVAL;
  printf("%s width=96 -> %s\n", bad == LH_EINVAL ? "PASS" : "FAIL", lh_strerror(bad));
  cudaFree(d_msg);
  cudaFree(d_out);
  printf("%d failures\n", fails);
  return fails ? 1 : 0;
}
