// intpeak.cu — per-class integer throughput on this B200 (roofline tool).
//
// SURVEY.md §8(d) defines the integer roof of each hash as its canonical
// 32-bit op mix divided by the measured rates of the SASS classes that mix
// uses.  This program measures those rates: one kernel per class, each
// thread running 8 independent dependence chains of a single instruction
// (so the pipe, not latency, is the limit), 64 warps per SM on every SM.
//
//   iadd3   IADD3 a = a + b + c                 (ALU pipe)
//   lop3    LOP3  a = a ^ b ^ c                 (ALU)
//   prmt    PRMT  byte permute                  (ALU)
//   shf     SHF.L.W funnel rotate               (ALU)
//   imad    IMAD  a = a * b + c  (32-bit)        (FMA)
//   wide    IMAD.WIDE.U32 32x32->64             (FMA, 64-bit result)
//   add64   IADD3 + IADD3.X  (64-bit add, both halves on ALU)
//   add64m  IADD3 + IMAD.X   (64-bit add, high half on FMA: the engine's form)
// and 1:1 interleaved pairs, which show which classes share a pipe and the
// dual-issue (instructions per clock) ceiling:
//   prmt+lop3, prmt+imad, lop3+wide, shf+imad, iadd3+imad
// plus the engine's full HighwayHash Update and SipRound on registers (the
// achievable rates of the real instruction mixes).
//
// Output: one JSON object (warp-instructions per second per class, at the
// SM clock sampled during the run).  The SASS of each kernel's loop is
// checked by tools/intpeak_sass.py (one instruction per op).  The roofs per
// hash are computed from this table by paper_1612_06257_b200/introof.py.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//            -o tools/intpeak tools/intpeak.cu   (run via tools/intpeak.py)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_1612_06257_b200/csrc/lh_device.cuh"
#include "../paper_1612_06257_b200/csrc/lh_host.cuh"

using namespace lh;

enum Op { IADD3, LOP3, PRMT, SHF, IMAD, WIDE, ADD64, ADD64M, NOPS };
static const char* kOpName[NOPS] = {"iadd3", "lop3", "prmt", "shf", "imad", "wide", "add64",
                                    "add64m"};
// SASS instructions one op issues (add64 / add64m are pairs).
static const int kOpInstr[NOPS] = {1, 1, 1, 1, 1, 1, 2, 2};

template <int OP>
__device__ __forceinline__ void op32(u32& a, u32 b, u32 c) {
  if (OP == IADD3) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a) : "r"(b), "r"(c));
  if (OP == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a) : "r"(b), "r"(c));
  if (OP == PRMT) asm volatile("prmt.b32 %0, %0, %1, 0x5041;" : "+r"(a) : "r"(b));
  if (OP == SHF) asm volatile("shf.l.wrap.b32 %0, %0, %1, 13;" : "+r"(a) : "r"(b));
  if (OP == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
}

// Single class: 8 chains x UNROLL steps per loop trip.
template <int OP>
__global__ void __launch_bounds__(256) k_class(u32* out, u32 seed, u32 one, int iters) {
  constexpr int UNROLL = 16;
  if (OP == WIDE || OP == ADD64 || OP == ADD64M) {
    u64 a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = (u64)seed * (threadIdx.x + 8 * k + 1) + blockIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < UNROLL; ++j)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const u64 b = a[(k + 1) & 7];
          if (OP == WIDE) a[k] = mul_lo_hi(a[k], b);
          if (OP == ADD64M) a[k] = add64_mixed(a[k], b, one);
          if (OP == ADD64) {
            u32 lo, hi;
            asm volatile("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
                         : "=r"(lo), "=r"(hi)
                         : "r"(lo32(a[k])), "r"(lo32(b)), "r"(hi32(a[k])), "r"(hi32(b)));
            a[k] = pack(lo, hi);
          }
        }
    }
    u64 s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k];
    if (s == 0x1234567ull) out[0] = (u32)s;
  } else {
    u32 a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed * (threadIdx.x + 8 * k + 1) + blockIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < UNROLL; ++j)
#pragma unroll
        for (int k = 0; k < 8; ++k) op32<OP>(a[k], a[(k + 1) & 7], a[(k + 3) & 7]);
    }
    u32 s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k];
    if (s == 0x1234567u) out[0] = s;
  }
}

// 1:1 pairs: chains 0-3 run class A, chains 4-7 class B.  Every chain
// depends only on itself and on loop-invariant registers (f[], a runtime
// PRMT selector), rotated per step so ptxas cannot fold two steps into one:
// the pair rate then measures dual issue, not latency.
template <int OP>
__device__ __forceinline__ void op_feed(u32& a, u32 f0, u32 f1, u32 sel) {
  if (OP == IADD3) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a) : "r"(f0), "r"(f1));
  if (OP == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6A;" : "+r"(a) : "r"(f0), "r"(f1));
  if (OP == PRMT) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(a) : "r"(f0), "r"(sel));
  if (OP == SHF) asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a) : "r"(f0), "r"(sel));
  if (OP == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(f0), "r"(f1));
}

template <int A, int B>
__global__ void __launch_bounds__(256) k_pair(u32* out, u32 seed, u32 one, int iters) {
  constexpr int UNROLL = 16;
  u32 a[8], f[4];
  u64 w[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed * (threadIdx.x + 8 * k + 1) + blockIdx.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[k] = seed * (0x9E3779B9u + 77 * k) + one + blockIdx.x;
    w[k] = (u64)a[k] * 0x9E3779B97F4A7C15ull;
  }
  const u32 sel = (seed & 0x3333u) | 0x4100u, wm = f[3] | 1u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
#pragma unroll
      for (int k = 0; k < 4; ++k) op_feed<A>(a[k], f[(j + k) & 3], f[(j + k + 1) & 3], sel);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (B == WIDE)
          w[k] = mulwide(lo32(w[k]) ^ hi32(w[k]), wm);
        else
          op_feed<B>(a[4 + k], f[(j + k + 2) & 3], f[(j + k + 3) & 3], sel);
      }
    }
  }
  u32 s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= a[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) s ^= lo32(w[k]) ^ hi32(w[k]);
  if (s == 0x1234567u) out[0] = s;
}

// The engine's HighwayHash Update on registers: 8 packets per trip from
// shared memory (2 LDS.128 each, as the TMA kernel reads them).
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

// The engine's SipRound on registers, 2 independent states per thread.
__global__ void __launch_bounds__(256) k_sipround(const SipMul km, u64* out, int iters) {
  u64 v[2][4];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int k = 0; k < 4; ++k) v[s][k] = (u64)(threadIdx.x + 1) * (k + 3 + s) + blockIdx.x;
  for (int i = 0; i < iters; i += 8) {
#pragma unroll
    for (int s = 0; s < 2; ++s) sip_rounds<8>(v[s][0], v[s][1], v[s][2], v[s][3], km, 8);
  }
  u64 x = 0;
#pragma unroll
  for (int s = 0; s < 2; ++s) x ^= v[s][0] ^ v[s][1] ^ v[s][2] ^ v[s][3];
  if (x == 0x12345678ull) out[0] = x;
}

// SipRound instruction-selection variants (A/B for csrc/lh_device.cuh):
//  0 the engine's sip_rounds (W16 alternating)     1 rot16 by PRMT every round
//  2 rot16 by IMAD.WIDE every round                3 as 0 with plain 64-bit adds
//  4 no IMAD.WIDE (rot13/17 by SHF), mixed adds    5 as 4 with plain adds
template <int V>
__device__ __forceinline__ void sip_round_v(u64& v0, u64& v1, u64& v2, u64& v3, const SipMul& k,
                                            int r) {
  auto add = [&](u64 a, u64 b) { return (V == 3 || V == 5) ? a + b : add64_mixed(a, b, k.one); };
  const bool w16 = V == 2 || ((V == 0 || V == 3) && (r & 1));
  v0 = add(v0, v1);
  v1 = V >= 4 ? rotl_xor_shf<13>(v1, v0) : rotl_xor_wide(v1, k.m13, v0);
  v0 = rot32(v0);
  v2 = add(v2, v3);
  v3 = w16 ? rotl_xor_wide(v3, k.m16, v2) : rotl16_xor_prmt(v3, v2);
  v0 = add(v0, v3);
  v3 = rotl_xor_shf<21>(v3, v0);
  v2 = add(v2, v1);
  v1 = V >= 4 ? rotl_xor_shf<17>(v1, v2) : rotl_xor_wide(v1, k.m17, v2);
  v2 = rot32(v2);
}

template <int V, int S>
__global__ void __launch_bounds__(256) k_sipvar(const SipMul km, u64* out, int iters) {
  u64 v[S][4];
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int k = 0; k < 4; ++k) v[s][k] = (u64)(threadIdx.x + 1) * (k + 3 + s) + blockIdx.x;
  for (int i = 0; i < iters; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int s = 0; s < S; ++s) sip_round_v<V>(v[s][0], v[s][1], v[s][2], v[s][3], km, j);
  }
  u64 x = 0;
#pragma unroll
  for (int s = 0; s < S; ++s) x ^= v[s][0] ^ v[s][1] ^ v[s][2] ^ v[s][3];
  if (x == 0x12345678ull) out[0] = x;
}

template <class F>
static float time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

static unsigned sm_clock_mhz() {
  int v = 0;
  // cudaDevAttrClockRate is the max clock; the live one comes from NVML in
  // the driver script (scripts/intpeak.sh) -- here report the attribute.
  cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, 0);
  return (unsigned)(v / 1000);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  u32* d = nullptr;
  cudaMalloc(&d, 64);
  const int blocks = sms * 8, threads = 256;  // 64 warps per SM
  const double warps = (double)blocks * threads / 32;
  const int iters = 512;                        // x 16 x 8 ops per thread
  const double ops_per_warp = (double)iters * 16 * 8;
  printf("{\"sms\": %d, \"clock_attr_mhz\": %u, \"warps_per_sm\": %d,\n", sms, sm_clock_mhz(),
         blocks * threads / 32 / sms);
  printf(" \"classes\": {");
#define RUN_CLASS(OPV)                                                                         \
  {                                                                                            \
    const float ms = time_ms([&] { k_class<OPV><<<blocks, threads>>>(d, 7, 1, iters); });       \
    const double r = warps * ops_per_warp * kOpInstr[OPV] / (ms * 1e-3);                      \
    printf("%s\"%s\": {\"warp_instr_per_s\": %.5e, \"sass_per_op\": %d, \"ms\": %.4f}",        \
           OPV ? ", " : "", kOpName[OPV], r, kOpInstr[OPV], ms);                               \
  }
  RUN_CLASS(IADD3) RUN_CLASS(LOP3) RUN_CLASS(PRMT) RUN_CLASS(SHF) RUN_CLASS(IMAD)
  RUN_CLASS(WIDE) RUN_CLASS(ADD64) RUN_CLASS(ADD64M)
  printf("},\n \"pairs\": {");
#define RUN_PAIR(A, B, NAME, FIRST)                                                            \
  {                                                                                            \
    const float ms = time_ms([&] { k_pair<A, B><<<blocks, threads>>>(d, 7, 1, iters); });      \
    const double r = warps * ops_per_warp / (ms * 1e-3);                                      \
    printf("%s\"%s\": {\"warp_instr_per_s\": %.5e, \"ms\": %.4f}", FIRST ? "" : ", ", NAME, r,  \
           ms);                                                                                \
  }
  RUN_PAIR(PRMT, LOP3, "prmt+lop3", 1) RUN_PAIR(PRMT, IMAD, "prmt+imad", 0)
  RUN_PAIR(LOP3, IMAD, "lop3+imad", 0) RUN_PAIR(SHF, IMAD, "shf+imad", 0)
  RUN_PAIR(IADD3, IMAD, "iadd3+imad", 0) RUN_PAIR(SHF, LOP3, "shf+lop3", 0)
  RUN_PAIR(PRMT, PRMT, "prmt+prmt", 0) RUN_PAIR(IMAD, IMAD, "imad+imad", 0)
  printf("},\n");
  const u64 key[4] = {1, 2, 3, 4};
  const Highway proto = make_highway(key, 64, 4);
  const int ublocks = sms * 2, uiters = 8192;  // 16 warps per SM, as the bench kernel
  float ms = time_ms([&] { k_update<<<ublocks, 256>>>(proto, (u64*)d, uiters); });
  const double updates = (double)ublocks * 256 * uiters / (ms * 1e-3);
  // The same Update at low occupancy (long-message shards leave 1-2 warps per
  // sub-partition): clocks per warp-Update at 4, 8, 16 and 32 warps per SM.
  {
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    printf(" \"update_clk_per_warp_by_warps_per_sm\": {");
    const int shapes[4][2] = {{1, 128}, {1, 256}, {2, 256}, {4, 256}};
    for (int k = 0; k < 4; ++k) {
      const int nb = sms * shapes[k][0], th = shapes[k][1];
      const float m = time_ms([&] { k_update<<<nb, th>>>(proto, (u64*)d, uiters); });
      const int wps = shapes[k][0] * th / 32;  // warps per SM
      // each sub-partition runs wps/4 warps; a warp-Update then takes:
      const double clk = m * 1e-3 * khz * 1e3 / uiters;
      printf("%s\"%d\": %.1f", k ? ", " : "", wps, clk);
    }
    printf("},\n");
  }
  const SipMul km{1u, 1u << 13, 1u << 17, 1u << 16};
  const int sblocks = sms * 8, siters = 4096;
  ms = time_ms([&] { k_sipround<<<sblocks, 256>>>(km, (u64*)d, siters); });
  const double sips = (double)sblocks * 256 * siters * 2 / (ms * 1e-3);
  printf(" \"highway_update_per_s\": %.5e, \"sipround_per_s\": %.5e,\n", updates, sips);
  printf(" \"sipround_variants_clk_per_warp_round\": {");
#define RUN_SV(V, S, FIRST)                                                                     \
  {                                                                                            \
    const float m = time_ms([&] { k_sipvar<V, S><<<sblocks, 256>>>(km, (u64*)d, siters); });   \
    const double r = (double)sblocks * 256 * siters * S / (m * 1e-3);                        \
    printf("%s\"v%d_s%d\": %.4e", FIRST ? "" : ", ", V, S, r);                                  \
  }
  RUN_SV(0, 1, 1) RUN_SV(0, 2, 0) RUN_SV(1, 1, 0) RUN_SV(1, 2, 0) RUN_SV(2, 1, 0) RUN_SV(2, 2, 0)
  RUN_SV(3, 1, 0) RUN_SV(3, 2, 0) RUN_SV(4, 1, 0) RUN_SV(4, 2, 0) RUN_SV(5, 1, 0) RUN_SV(5, 2, 0)
  printf("},\n");
  printf(" \"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
