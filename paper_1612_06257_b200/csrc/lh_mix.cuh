// lh_mix.cuh — the SplitMix64 finalizer behind the seeded synthetic
// generator (lh_synth.cu) and the device self-tests (lh_state.cu).
// word(seed, stream, w) = mix64(k + (w + 1) * G), k = mix64(seed * G + stream + 1).
#pragma once
#include <stdint.h>

namespace lh {

constexpr uint64_t kG = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t synth_key(uint64_t seed, uint64_t stream_id) {
  return mix64(seed * kG + stream_id + 1);
}

__host__ __device__ __forceinline__ uint64_t synth_word(uint64_t key, uint64_t w) {
  return mix64(key + (w + 1) * kG);
}

}  // namespace lh
