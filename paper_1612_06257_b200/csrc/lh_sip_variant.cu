// lh_sip_variant.cu — one Sip-family hasher's kernels (fixed, ragged,
// streaming append), compiled once per variant of lh_sip_variants.h with
// -DLH_VAR_TAG=<tag> -DLH_VAR_C=<c> -DLH_VAR_D=<d> -DLH_VAR_TREE=<0|1>.
#include "lh_kernels.cuh"
#include "lh_sip_variants.h"

#if !defined(LH_VAR_TAG) || !defined(LH_VAR_C) || !defined(LH_VAR_D) || !defined(LH_VAR_TREE)
#error "compile with -DLH_VAR_TAG=.. -DLH_VAR_C=.. -DLH_VAR_D=.. -DLH_VAR_TREE=.."
#endif

#define LH_CAT2(a, b) a##b
#define LH_CAT(a, b) LH_CAT2(a, b)

namespace {
using VarH = std::conditional_t<LH_VAR_TREE != 0, SipTree<LH_VAR_C, LH_VAR_D>,
                                Sip<LH_VAR_C, LH_VAR_D>>;

VarH make_var(const u64 key[2], int c, int d) {
#if LH_VAR_TREE
  return make_siptree<LH_VAR_C, LH_VAR_D>(key, c, d);
#else
  return make_sip<LH_VAR_C, LH_VAR_D>(key, c, d);
#endif
}
}  // namespace

namespace lh {

int LH_CAT(sip_fixed_, LH_VAR_TAG)(const u64 key[2], int c, int d, const uint8_t* msgs, u64 n,
                                   u64 len, u64* out, cudaStream_t st, int kernel) {
  return dispatch_fixed(make_var(key, c, d), msgs, n, len, out, st, kernel);
}

int LH_CAT(sip_ragged_, LH_VAR_TAG)(const u64 key[2], int c, int d, const uint8_t* buf,
                                    const u64* off, const u32* lens, u64 n, u64* out,
                                    cudaStream_t st, bool staged, const uint4* order) {
  return sip_dispatch_ragged(make_var(key, c, d), buf, off, lens, n, out, st, staged, order);
}

// Streaming records carry runtime round counts: only the (0, 0) variants
// take whole-block appends (lh_stream.cu).
int LH_CAT(sip_stream_tma_, LH_VAR_TAG)(void* rec, const uint8_t* chunks, u64 n, u64 len,
                                        cudaStream_t st) {
#if LH_VAR_C == 0 && LH_VAR_D == 0
  return launch_tma_stream((StreamRec<VarH>*)rec, chunks, n, len, st);
#else
  (void)rec, (void)chunks, (void)n, (void)len, (void)st;
  return LH_EINVAL;
#endif
}

}  // namespace lh
