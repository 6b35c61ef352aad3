// lh_engine.cu — HighwayHash launches, PRF, and the extern "C" boundary
// (include/lanehash_b200.h).  Kernels: lh_kernels.cuh; the Sip family's
// instantiations: lh_sip_variant.cu (one object per variant).
#include "lh_kernels.cuh"
#include "lh_sip_variants.h"

#define LH_VERSION_STR "paper_1612_06257_b200 0.3.0 (sm_100a)"

namespace {

// --------------------------------------------------------------------------
// PRF: hash64(key, le64(ctr)).  With r = 8 the remainder packet is
// (ctr, 0, 0, 0) (S/highway.py:206-220) and the length injection is
// key-only, so `proto` arrives already tweaked; per counter: 1 + rounds
// updates.
// --------------------------------------------------------------------------
// The first Update absorbs the packet (ctr, 0, 0, 0): lanes 1-3 see a
// constant packet word, so their per-lane steps 1-5 (S/highway.py:137-141)
// and the whole zipper pair (2,3) are the same for every counter and are
// precomputed on the host (prf_proto); only lane 0's steps and the pair
// (0,1) zippers run per counter (~26 of ~78 instructions).
struct PrfProto {
  Highway h;      // lanes 1..3 after steps 1-5; lanes 2,3 fully updated;
                  // lane 0: m0/m1 pre-update, v0 = v0_pre + m1_pre (step 4)
  u64 v1_0_base;  // v1[0] + m0[0] before the update (steps 1-2 minus ctr)
  u32 v0_0_hi;    // hi32 of lane-0 v0 before step 4 (used by step 3)
};

__global__ void __launch_bounds__(256) k_prf(const PrfProto proto, u64 start, u64 n,
                                             u64* __restrict__ out) {
  __shared__ __align__(16) u64 s_state[16];  // proto.h's state (see Highway::load_state)
  if (threadIdx.x < 16) {
    const u64* src = threadIdx.x < 4 ? proto.h.v0 : threadIdx.x < 8 ? proto.h.v1
                     : threadIdx.x < 12 ? proto.h.m0 : proto.h.m1;
    s_state[threadIdx.x] = src[threadIdx.x & 3];
  }
  __syncthreads();
  const u32 s_state_a = smem_u32(s_state);
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    Highway h;
    h.load_state(s_state_a, proto.h);
    const u64 v1_0 = proto.v1_0_base + (start + i);         // steps 1-2
    h.m0[0] ^= (u64)lo32(v1_0) * (u64)proto.v0_0_hi;        // step 3
    h.m1[0] ^= mul_lo_hi(h.v0[0], v1_0);                    // step 5 (v0 post step 4)
    h.v1[0] = v1_0;
    u64 z0, z1;
    zipper(h.v1[0], h.v1[1], z0, z1);
    h.v0[0] = add64_mixed(h.v0[0], z0, h.one);
    h.v0[1] = add64_mixed(h.v0[1], z1, h.one);
    zipper(h.v0[0], h.v0[1], z0, z1);
    h.v1[0] = add64_mixed(h.v1[0], z0, h.one);
    h.v1[1] = add64_mixed(h.v1[1], z1, h.one);
    h.finalize_out<1>(out + i);
  }
}

}  // namespace


// Host precompute for k_prf (see PrfProto).  Mirrors S/highway.py:130-150
// and 182-199 on the host for the counter-independent parts.
static u64 h_mul32(u64 a, u64 b) { return (u64)(uint32_t)a * (u64)(uint32_t)(b >> 32); }
static void h_zipper(u64 lo, u64 hi, u64& zlo, u64& zhi) {
  static const int kZip[16] = {3, 12, 2, 5, 14, 1, 15, 0, 11, 4, 10, 13, 9, 6, 8, 7};
  uint8_t in[16], o[16];
  for (int b = 0; b < 8; ++b) {
    in[b] = (uint8_t)(lo >> (8 * b));
    in[8 + b] = (uint8_t)(hi >> (8 * b));
  }
  for (int b = 0; b < 16; ++b) o[b] = in[kZip[b]];
  zlo = zhi = 0;
  for (int b = 7; b >= 0; --b) {
    zlo = (zlo << 8) | o[b];
    zhi = (zhi << 8) | o[8 + b];
  }
}

static PrfProto prf_proto(const u64 key[4], int rounds) {
  Highway h = make_highway(key, 64, rounds);
  for (int i = 0; i < 4; ++i) {  // length injection for r = 8 (S/highway.py:188-197)
    const uint32_t lo = (uint32_t)h.v0[i] + 8u, hi = (uint32_t)(h.v0[i] >> 32) + 8u;
    h.v0[i] = ((u64)hi << 32) | lo;
    const uint32_t l1 = (uint32_t)h.v1[i], h1 = (uint32_t)(h.v1[i] >> 32);
    const uint32_t rl = (l1 << 8) | (l1 >> 24), rh = (h1 << 8) | (h1 >> 24);
    h.v1[i] = ((u64)rh << 32) | rl;
  }
  PrfProto p;
  memset(&p, 0, sizeof p);
  p.v1_0_base = h.v1[0] + h.m0[0];
  p.v0_0_hi = (uint32_t)(h.v0[0] >> 32);
  for (int i = 1; i < 4; ++i) {  // steps 1-5 with packet word 0
    h.v1[i] += h.m0[i];
    h.m0[i] ^= h_mul32(h.v1[i], h.v0[i]);
    h.v0[i] += h.m1[i];
    h.m1[i] ^= h_mul32(h.v0[i], h.v1[i]);
  }
  h.v0[0] += h.m1[0];  // lane 0 step 4 is counter-independent
  u64 z2, z3;
  h_zipper(h.v1[2], h.v1[3], z2, z3);
  h.v0[2] += z2;
  h.v0[3] += z3;
  h_zipper(h.v0[2], h.v0[3], z2, z3);
  h.v1[2] += z2;
  h.v1[3] += z3;
  p.h = h;
  return p;
}


namespace lh {
int stream_update_tma(int alg, void* d_state, u64 n, const uint8_t* d_chunks, u64 chunk_len,
                      void* stream) {
  if (n < 1024 || chunk_len % 32 || !tma_ok(d_chunks, n, chunk_len)) return LH_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  switch (alg) {
    case LH_ALG_HIGHWAY: {
      Highway proto;
      memset(&proto, 0, sizeof proto);
      if (prefer_split(proto, d_chunks, n, chunk_len))  // few long chunks: 2 threads per row
        return launch_split<true>(proto, d_chunks, n, chunk_len, nullptr, st,
                                  (StreamRec<Highway>*)d_state);
      return launch_tma_stream((StreamRec<Highway>*)d_state, d_chunks, n, chunk_len, st);
    }
    case LH_ALG_SIPHASH:
      return sip_stream_tma_s00(d_state, d_chunks, n, chunk_len, st);
    case LH_ALG_SIPTREE:
      return sip_stream_tma_t00(d_state, d_chunks, n, chunk_len, st);
    default:
      return LH_EINVAL;
  }
}
}  // namespace lh

// ==========================================================================
// extern "C" boundary
// ==========================================================================
extern "C" {

const char* lh_version(void) { return LH_VERSION_STR; }

const char* lh_strerror(int code) {
  switch (code) {
    case LH_OK: return "ok";
    case LH_EINVAL: return "invalid argument";
    case LH_EALIGN: return "misaligned pointer";
    case LH_ECUDA: return "CUDA runtime error";
    case LH_ENODEV: return "no sm_100 CUDA device";
    case LH_ETOOBIG: return "size out of supported range";
    default: return "unknown error";
  }
}

int lh_highway_fixed_kernel(const uint8_t* d_msgs, uint64_t n, uint64_t len,
                            const uint64_t key[4], int width, int rounds, uint64_t* d_out,
                            void* stream, int kernel) {
  if (!key || !valid_width(width) || rounds < 0 || (n && !d_out) || (n && len && !d_msgs))
    return LH_EINVAL;
  if ((uintptr_t)d_out % 8) return LH_EALIGN;
  if (kernel < 0 || kernel > LH_KERNEL_RING) return LH_EINVAL;
  if (len && n > UINT64_MAX / len) return LH_ETOOBIG;
  const Highway h = make_highway(key, width, rounds);
  return dispatch_fixed(h, d_msgs, n, len, d_out, (cudaStream_t)stream, kernel);
}

int lh_highway_fixed(const uint8_t* d_msgs, uint64_t n, uint64_t len, const uint64_t key[4],
                     int width, int rounds, uint64_t* d_out, void* stream) {
  return lh_highway_fixed_kernel(d_msgs, n, len, key, width, rounds, d_out, stream,
                                 LH_KERNEL_AUTO);
}

int lh_highway_ragged_kernel(const uint8_t* d_buf, const uint64_t* d_offsets,
                             const uint32_t* d_lengths, uint64_t n, const uint64_t key[4],
                             int width, int rounds, uint64_t* d_out, void* stream, int kernel) {
  if (!key || !valid_width(width) || rounds < 0 || (n && (!d_out || !d_offsets || !d_buf)))
    return LH_EINVAL;
  if ((uintptr_t)d_out % 8 || (uintptr_t)d_offsets % 8 || (uintptr_t)d_lengths % 4)
    return LH_EALIGN;
  if (kernel != LH_KERNEL_AUTO && kernel != LH_KERNEL_DIRECT && kernel != LH_KERNEL_STAGED &&
      kernel != LH_KERNEL_RING)
    return LH_EINVAL;
  const Highway h = make_highway(key, width, rounds);
  if (kernel == LH_KERNEL_DIRECT || kernel == LH_KERNEL_RING)
    return launch_ring(h, d_buf, d_offsets, d_lengths, 0, n, d_out, (cudaStream_t)stream);
  return launch_staged(h, d_buf, d_offsets, d_lengths, 0, n, d_out, (cudaStream_t)stream);
}

int lh_highway_ragged(const uint8_t* d_buf, const uint64_t* d_offsets, const uint32_t* d_lengths,
                      uint64_t n, const uint64_t key[4], int width, int rounds, uint64_t* d_out,
                      void* stream) {
  return lh_highway_ragged_kernel(d_buf, d_offsets, d_lengths, n, key, width, rounds, d_out,
                                  stream, LH_KERNEL_AUTO);
}

// Variant choice: compile-time rounds for 2-4 and 1-3, runtime otherwise.
static int sip_fixed_impl(const uint8_t* d_msgs, u64 n, u64 len, const u64 key[2], int c, int d,
                          int tree, u64* d_out, cudaStream_t st, int kernel) {
  const bool r24 = c == 2 && d == 4, r13 = c == 1 && d == 3;
  if (tree) {
    if (r24) return sip_fixed_t24(key, c, d, d_msgs, n, len, d_out, st, kernel);
    if (r13) return sip_fixed_t13(key, c, d, d_msgs, n, len, d_out, st, kernel);
    return sip_fixed_t00(key, c, d, d_msgs, n, len, d_out, st, kernel);
  }
  if (r24) return sip_fixed_s24(key, c, d, d_msgs, n, len, d_out, st, kernel);
  if (r13) return sip_fixed_s13(key, c, d, d_msgs, n, len, d_out, st, kernel);
  return sip_fixed_s00(key, c, d, d_msgs, n, len, d_out, st, kernel);
}

int lh_siphash_fixed_kernel(const uint8_t* d_msgs, uint64_t n, uint64_t len,
                            const uint64_t key[2], int c, int d, int tree, uint64_t* d_out,
                            void* stream, int kernel) {
  if (!key || c < 1 || d < 1 || (n && !d_out) || (n && len && !d_msgs)) return LH_EINVAL;
  if ((uintptr_t)d_out % 8) return LH_EALIGN;
  if (kernel < 0 || kernel > LH_KERNEL_RING || kernel == LH_KERNEL_SPLIT) return LH_EINVAL;
  if (len && n > UINT64_MAX / len) return LH_ETOOBIG;
  return sip_fixed_impl(d_msgs, n, len, key, c, d, tree, d_out, (cudaStream_t)stream, kernel);
}

int lh_siphash_fixed(const uint8_t* d_msgs, uint64_t n, uint64_t len, const uint64_t key[2],
                     int c, int d, int tree, uint64_t* d_out, void* stream) {
  return lh_siphash_fixed_kernel(d_msgs, n, len, key, c, d, tree, d_out, stream,
                                 LH_KERNEL_AUTO);
}

static int sip_ragged_impl(const uint8_t* d_buf, const uint64_t* d_offsets,
                           const uint32_t* d_lengths, uint64_t n, const uint64_t key[2], int c,
                           int d, int tree, uint64_t* d_out, cudaStream_t st, bool staged,
                           const uint4* order) {
  const bool r24 = c == 2 && d == 4, r13 = c == 1 && d == 3;
  if (tree) {
    if (r24)
      return sip_ragged_t24(key, c, d, d_buf, d_offsets, d_lengths, n, d_out, st, staged, order);
    if (r13)
      return sip_ragged_t13(key, c, d, d_buf, d_offsets, d_lengths, n, d_out, st, staged, order);
    return sip_ragged_t00(key, c, d, d_buf, d_offsets, d_lengths, n, d_out, st, staged, order);
  }
  if (r24)
    return sip_ragged_s24(key, c, d, d_buf, d_offsets, d_lengths, n, d_out, st, staged, order);
  if (r13)
    return sip_ragged_s13(key, c, d, d_buf, d_offsets, d_lengths, n, d_out, st, staged, order);
  return sip_ragged_s00(key, c, d, d_buf, d_offsets, d_lengths, n, d_out, st, staged, order);
}

int lh_siphash_ragged_kernel(const uint8_t* d_buf, const uint64_t* d_offsets,
                             const uint32_t* d_lengths, uint64_t n, const uint64_t key[2], int c,
                             int d, int tree, uint64_t* d_out, void* stream, int kernel) {
  if (!key || c < 1 || d < 1 || (n && (!d_out || !d_offsets || !d_buf))) return LH_EINVAL;
  if ((uintptr_t)d_out % 8 || (uintptr_t)d_offsets % 8 || (uintptr_t)d_lengths % 4)
    return LH_EALIGN;
  if (kernel != LH_KERNEL_AUTO && kernel != LH_KERNEL_DIRECT && kernel != LH_KERNEL_RING &&
      kernel != LH_KERNEL_STAGED)
    return LH_EINVAL;
  return sip_ragged_impl(d_buf, d_offsets, d_lengths, n, key, c, d, tree, d_out,
                         (cudaStream_t)stream, kernel == LH_KERNEL_STAGED, nullptr);
}

int lh_siphash_ragged_ordered(const uint8_t* d_buf, const uint64_t* d_offsets,
                              const uint32_t* d_lengths, uint64_t n, const void* d_sched,
                              const uint64_t key[2], int c, int d, int tree, uint64_t* d_out,
                              void* stream) {
  if (!key || c < 1 || d < 1 || (n && (!d_out || !d_offsets || !d_buf || !d_sched)))
    return LH_EINVAL;
  if ((uintptr_t)d_out % 8 || (uintptr_t)d_offsets % 8 || (uintptr_t)d_lengths % 4 ||
      (uintptr_t)d_sched % 16)
    return LH_EALIGN;
  if (n > 0xFFFFFFFFull) return LH_ETOOBIG;
  return sip_ragged_impl(d_buf, d_offsets, d_lengths, n, key, c, d, tree, d_out,
                         (cudaStream_t)stream, false, (const uint4*)d_sched);
}

int lh_highway_ragged_ordered(const uint8_t* d_buf, const uint64_t* d_offsets,
                              const uint32_t* d_lengths, uint64_t n, const void* d_sched,
                              const uint64_t key[4], int width, int rounds, uint64_t* d_out,
                              void* stream) {
  if (!key || !valid_width(width) || rounds < 0 ||
      (n && (!d_out || !d_offsets || !d_buf || !d_sched)))
    return LH_EINVAL;
  if ((uintptr_t)d_out % 8 || (uintptr_t)d_offsets % 8 || (uintptr_t)d_lengths % 4 ||
      (uintptr_t)d_sched % 16)
    return LH_EALIGN;
  if (n > 0xFFFFFFFFull) return LH_ETOOBIG;
  const Highway h = make_highway(key, width, rounds);
  return launch_ring(h, d_buf, d_offsets, d_lengths, 0, n, d_out, (cudaStream_t)stream, (const uint4*)d_sched);
}

int lh_siphash_ragged(const uint8_t* d_buf, const uint64_t* d_offsets, const uint32_t* d_lengths,
                      uint64_t n, const uint64_t key[2], int c, int d, int tree, uint64_t* d_out,
                      void* stream) {
  return lh_siphash_ragged_kernel(d_buf, d_offsets, d_lengths, n, key, c, d, tree, d_out, stream,
                                  LH_KERNEL_AUTO);
}

int lh_highway_prf64(uint64_t start, uint64_t n, const uint64_t key[4], int rounds,
                     uint64_t* d_out, void* stream) {
  if (!key || rounds < 0 || (n && !d_out)) return LH_EINVAL;
  if ((uintptr_t)d_out % 8) return LH_EALIGN;
  int sms = 0;
  int rc = check_device(&sms);
  if (rc) return rc;
  if (n == 0) return LH_OK;
  const PrfProto pp = prf_proto(key, rounds);
  k_prf<<<grid_for(n, 256, sms), 256, 0, (cudaStream_t)stream>>>(pp, start, n, d_out);
  return cuda_err(cudaGetLastError());
}

}  // extern "C"
