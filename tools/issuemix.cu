// issuemix.cu — how many warp-instructions per clock one SM sub-partition
// issues when ALU-pipe and FMA-pipe integer instructions are mixed, as a
// function of the number of *register* source operands of each instruction
// and of the ALU:FMA ratio.  (tools/intpeak.cu found single classes at 0.5
// per SMSP per clock, but 1:1 ALU+IMAD mixes at only 0.63-0.72 instead of
// 1.0, while IADD3 + IMAD.X pairs reach 0.95; the engine's real mixes sit at
// 0.56-0.6.  This tool separates the candidate causes: register-file read
// bandwidth (operands per clock) vs. a pairing rule between the pipes.)
//
// Every kernel: 64 warps per SM in one wave; each thread runs NA independent
// chains of ALU form AF and NB independent chains of FMA form BF, RA and RB
// ops per chain per step; rates = instructions / (CUDA-event time x the SM
// clock attribute; the runs draw ~250 W, far from any throttle).  The
// in-kernel clock64() maxima are printed too, but they run short for kernels
// whose 8 blocks per SM are not all co-resident (> 32 registers).
//
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/issuemix tools/issuemix.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

typedef uint32_t u32;
typedef uint64_t u64;

// ALU forms
enum { A_LOP3_3R, A_LOP3_2R, A_LOP3_2R_U, A_SHF_1R, A_SHF_3R, A_PRMT_2R, A_IADD3_3R, A_PRMT_1R, A_NONE };
// FMA forms
enum { B_IMAD_3R, B_IMAD_2R_IMM, B_IMAD_2R_RZ, B_IMAD_2R_U, B_WIDE_2R, B_WIDE_1R_U, B_NONE, B_HI_2R, B_HI_3R, B_LOHI_2R, B_HI_2R_U };

template <int F>
__device__ __forceinline__ void opA(u32& a, u32 f0, u32 f1, u32 uni) {
  if (F == A_LOP3_3R) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6A;" : "+r"(a) : "r"(f0), "r"(f1));
  if (F == A_LOP3_2R) asm volatile("xor.b32 %0, %0, %1;" : "+r"(a) : "r"(f0));
  if (F == A_LOP3_2R_U) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6A;" : "+r"(a) : "r"(f0), "r"(uni));
  if (F == A_SHF_1R) asm volatile("shf.l.wrap.b32 %0, %0, %0, 13;" : "+r"(a));
  if (F == A_SHF_3R) asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a) : "r"(f0), "r"(f1));
  if (F == A_PRMT_2R) asm volatile("prmt.b32 %0, %0, %1, 0x5041;" : "+r"(a) : "r"(f0));
  if (F == A_IADD3_3R)
    asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a) : "r"(f0), "r"(f1));
  if (F == A_PRMT_1R) asm volatile("prmt.b32 %0, %0, %0, 0x2103;" : "+r"(a));
}

template <int F>
__device__ __forceinline__ void opB(u32& a, u32& hi, u32 f0, u32 f1, u32 uni) {
  if (F == B_IMAD_3R) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(f0), "r"(f1));
  if (F == B_IMAD_2R_IMM) asm volatile("mad.lo.u32 %0, %0, 0x9E3779B1, %1;" : "+r"(a) : "r"(f1));
  if (F == B_IMAD_2R_RZ) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(a) : "r"(f0));
  if (F == B_IMAD_2R_U) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(uni), "r"(f1));
  if (F == B_HI_2R) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a) : "r"(f0));
  if (F == B_HI_2R_U) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a) : "r"(uni));
  if (F == B_HI_3R) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(f0), "r"(f1));
  if (F == B_LOHI_2R) {  // the 64-bit product as IMAD + IMAD.HI (two 32-bit results), xor-fed like the WIDE forms
    const u32 x = a ^ hi;
    asm volatile("mul.lo.u32 %0, %2, %3;\n\tmul.hi.u32 %1, %2, %3;" : "=r"(a), "=r"(hi) : "r"(x), "r"(f0));
  }
  if (F == B_WIDE_2R) {
    u64 w;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(a ^ hi), "r"(f0));
    a = (u32)w;
    hi = (u32)(w >> 32);
  }
  if (F == B_WIDE_1R_U) {
    u64 w;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(a ^ hi), "r"(uni));
    a = (u32)w;
    hi = (u32)(w >> 32);
  }
}

template <int AF, int BF, int RA, int RB, int NA, int NB>
__global__ void __launch_bounds__(256) k_mix(u32* out, u64* cyc, u32 seed, u32 uni, int iters) {
  constexpr int UNROLL = 8;
  u32 a[NA > 0 ? NA : 1], b[NB > 0 ? NB : 1], bh[NB > 0 ? NB : 1], f[4];
#pragma unroll
  for (int k = 0; k < NA; ++k) a[k] = seed * (threadIdx.x + 8 * k + 1) + blockIdx.x;
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    b[k] = seed * (threadIdx.x + 8 * k + 77) + blockIdx.x;
    bh[k] = b[k] * 3;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) f[k] = (seed * (0x9E3779B9u + 77 * k) + blockIdx.x) | 1u;
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      // interleave: round-robin one A op and one B op while any remain
#pragma unroll
      for (int r = 0; r < (RA > RB ? RA : RB); ++r) {
#pragma unroll
        for (int k = 0; k < (NA > NB ? NA : NB); ++k) {
          if (r < RA && k < NA) opA<AF>(a[k], f[(j + k) & 3], f[(j + k + 1) & 3], uni);
          if (r < RB && k < NB) opB<BF>(b[k], bh[k], f[(j + k + 2) & 3], f[(j + k + 3) & 3], uni);
        }
      }
    }
  }
  const long long t1 = clock64();
  u32 s = 0;
#pragma unroll
  for (int k = 0; k < NA; ++k) s ^= a[k];
#pragma unroll
  for (int k = 0; k < NB; ++k) s ^= b[k] ^ bh[k];
  if (s == 0x1234567u) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (u64)(t1 - t0);
}

static int g_sms;
static u32* g_out;
static u64* g_cyc;
static bool g_first = true;

template <int AF, int BF, int RA, int RB, int NA, int NB>
static void run(const char* name, int warps_per_sm = 64) {
  const int blocks_per_sm = warps_per_sm / 8;
  const int blocks = g_sms * blocks_per_sm, iters = 2048;
  u64* h = (u64*)malloc(sizeof(u64) * blocks);
  double best = 1e30, best_ms = 1e30, mn_c = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_mix<AF, BF, RA, RB, NA, NB><<<blocks, 256>>>(g_out, g_cyc, 7, 0x9E3779B1u, iters);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best_ms = ms < best_ms ? ms : best_ms;
    cudaMemcpy(h, g_cyc, sizeof(u64) * blocks, cudaMemcpyDeviceToHost);
    double mx = 0, mn = 1e30;
    for (int i = 0; i < blocks; ++i) {
      mx = h[i] > mx ? (double)h[i] : mx;
      mn = h[i] < mn ? (double)h[i] : mn;
    }
    if (mx < best) {
      best = mx;
      mn_c = mn;
    }
  }
  free(h);
  // the WIDE forms carry one LOP3 per op (the xor that feeds the multiply)
  const int xa = (BF == B_WIDE_2R || BF == B_WIDE_1R_U || BF == B_LOHI_2R) ? RB * NB : 0;
  const int xb = BF == B_LOHI_2R ? RB * NB : 0;  // two FMA instructions per op
  const double per_warp = (double)iters * 8 * (RA * NA + RB * NB + xa + xb);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double clk = best_ms * 1e-3 * khz * 1e3;  // SM clocks of the launch
  const double ipc_smsp = per_warp * warps_per_sm / 4.0 / clk;
  const double alu = (double)iters * 8 * (RA * NA + xa) * warps_per_sm / 4.0 / clk;
  const double fma = (double)iters * 8 * (RB * NB + xb) * warps_per_sm / 4.0 / clk;
  printf("%s\n  \"%s\": {\"ipc_smsp\": %.3f, \"alu_per_clk\": %.3f, \"fma_per_clk\": %.3f, \"warps_per_sm\": %d, \"cyc_max\": %.0f, \"cyc_min\": %.0f, \"event_us\": %.1f}",
         g_first ? "" : ",", name, ipc_smsp, alu, fma, warps_per_sm, best, mn_c, best_ms * 1e3);
  g_first = false;
}

int main() {
  cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&g_out, 64);
  cudaMalloc(&g_cyc, sizeof(u64) * g_sms * 8);
  printf("{");
  // single classes (0.5 per SMSP per clock each)
  run<A_LOP3_3R, B_NONE, 1, 0, 8, 0>("lop3_3r");
  run<A_PRMT_1R, B_NONE, 1, 0, 8, 0>("prmt_1r");
  run<A_SHF_1R, B_NONE, 1, 0, 8, 0>("shf_1r");
  run<A_NONE, B_IMAD_3R, 0, 1, 0, 8>("imad_3r");
  run<A_NONE, B_IMAD_2R_U, 0, 1, 0, 8>("imad_2r_u");
  run<A_NONE, B_WIDE_2R, 0, 1, 0, 8>("xor+wide_2r");
  run<A_NONE, B_WIDE_1R_U, 0, 1, 0, 8>("xor+wide_1r_u");
  // 1:1, register-operand-count sweep
  run<A_LOP3_3R, B_IMAD_3R, 1, 1, 4, 4>("lop3_3r+imad_3r");
  run<A_LOP3_2R, B_IMAD_3R, 1, 1, 4, 4>("lop3_2r+imad_3r");
  run<A_LOP3_2R_U, B_IMAD_3R, 1, 1, 4, 4>("lop3_2r_u+imad_3r");
  run<A_SHF_1R, B_IMAD_3R, 1, 1, 4, 4>("shf_1r+imad_3r");
  run<A_PRMT_1R, B_IMAD_3R, 1, 1, 4, 4>("prmt_1r+imad_3r");
  run<A_LOP3_3R, B_IMAD_2R_IMM, 1, 1, 4, 4>("lop3_3r+imad_2r_imm");
  run<A_LOP3_3R, B_IMAD_2R_RZ, 1, 1, 4, 4>("lop3_3r+imad_2r_rz");
  run<A_LOP3_3R, B_IMAD_2R_U, 1, 1, 4, 4>("lop3_3r+imad_2r_u");
  run<A_LOP3_2R, B_IMAD_2R_IMM, 1, 1, 4, 4>("lop3_2r+imad_2r_imm");
  run<A_LOP3_2R, B_IMAD_2R_RZ, 1, 1, 4, 4>("lop3_2r+imad_2r_rz");
  run<A_LOP3_2R_U, B_IMAD_2R_U, 1, 1, 4, 4>("lop3_2r_u+imad_2r_u");
  run<A_SHF_1R, B_IMAD_2R_RZ, 1, 1, 4, 4>("shf_1r+imad_2r_rz");
  run<A_PRMT_1R, B_IMAD_2R_U, 1, 1, 4, 4>("prmt_1r+imad_2r_u");
  run<A_SHF_1R, B_IMAD_2R_U, 1, 1, 4, 4>("shf_1r+imad_2r_u");
  run<A_SHF_3R, B_IMAD_3R, 1, 1, 4, 4>("shf_3r+imad_3r");
  run<A_PRMT_2R, B_IMAD_2R_RZ, 1, 1, 4, 4>("prmt_2r+imad_2r_rz");
  run<A_IADD3_3R, B_IMAD_3R, 1, 1, 4, 4>("iadd3_3r+imad_3r");
  // ratio sweep
  run<A_LOP3_3R, B_IMAD_3R, 2, 1, 4, 4>("2lop3_3r+1imad_3r");
  run<A_LOP3_3R, B_IMAD_3R, 3, 1, 4, 4>("3lop3_3r+1imad_3r");
  run<A_LOP3_3R, B_IMAD_3R, 1, 2, 4, 4>("1lop3_3r+2imad_3r");
  run<A_LOP3_2R, B_IMAD_2R_RZ, 2, 1, 4, 4>("2lop3_2r+1imad_2r_rz");
  run<A_SHF_1R, B_IMAD_2R_U, 2, 1, 4, 4>("2shf_1r+1imad_2r_u");
  run<A_SHF_1R, B_IMAD_2R_U, 3, 1, 4, 4>("3shf_1r+1imad_2r_u");
  // IMAD.WIDE mixes (64-bit result; each WIDE op carries one LOP3)
  run<A_LOP3_3R, B_WIDE_2R, 1, 1, 4, 4>("lop3_3r+xorwide_2r");
  run<A_LOP3_3R, B_WIDE_2R, 2, 1, 4, 4>("2lop3_3r+1xorwide_2r");
  run<A_SHF_1R, B_WIDE_1R_U, 1, 1, 4, 4>("shf_1r+xorwide_1r_u");
  run<A_SHF_1R, B_WIDE_1R_U, 2, 1, 4, 4>("2shf_1r+1xorwide_1r_u");
  run<A_SHF_1R, B_WIDE_1R_U, 3, 1, 4, 4>("3shf_1r+1xorwide_1r_u");
  // IMAD.HI (32-bit result): does it pair with the ALU pipe where IMAD.WIDE does not?
  run<A_NONE, B_HI_2R, 0, 1, 0, 8>("hi_2r");
  run<A_NONE, B_HI_3R, 0, 1, 0, 8>("hi_3r");
  run<A_NONE, B_LOHI_2R, 0, 1, 0, 8>("xor+lohi_2r");
  run<A_SHF_1R, B_HI_2R_U, 1, 1, 4, 4>("shf_1r+hi_2r_u");
  run<A_SHF_1R, B_HI_2R_U, 2, 1, 4, 4>("2shf_1r+1hi_2r_u");
  run<A_SHF_1R, B_HI_2R_U, 3, 1, 4, 4>("3shf_1r+1hi_2r_u");
  run<A_LOP3_3R, B_HI_3R, 1, 1, 4, 4>("lop3_3r+hi_3r");
  run<A_LOP3_3R, B_HI_3R, 2, 1, 4, 4>("2lop3_3r+1hi_3r");
  run<A_SHF_1R, B_LOHI_2R, 1, 1, 4, 4>("shf_1r+xorlohi_2r");
  run<A_SHF_1R, B_LOHI_2R, 2, 1, 4, 4>("2shf_1r+1xorlohi_2r");
  run<A_SHF_1R, B_LOHI_2R, 3, 1, 4, 4>("3shf_1r+1xorlohi_2r");
  run<A_SHF_1R, B_WIDE_2R, 2, 1, 4, 4>("2shf_1r+1xorwide_2r");
  run<A_SHF_1R, B_WIDE_2R, 3, 1, 4, 4>("3shf_1r+1xorwide_2r");
  // more chains / fewer warps
  run<A_LOP3_3R, B_IMAD_3R, 1, 1, 8, 8>("lop3_3r+imad_3r_16chains");
  run<A_LOP3_3R, B_IMAD_3R, 1, 1, 4, 4>("lop3_3r+imad_3r_w32", 32);
  run<A_LOP3_3R, B_IMAD_3R, 1, 1, 4, 4>("lop3_3r+imad_3r_w16", 16);
  run<A_LOP3_3R, B_IMAD_3R, 1, 1, 4, 4>("lop3_3r+imad_3r_w8", 8);
  run<A_SHF_1R, B_IMAD_2R_U, 1, 1, 4, 4>("shf_1r+imad_2r_u_w16", 16);
  printf("\n, \"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
