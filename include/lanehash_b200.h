/*
 * lanehash_b200.h — C ABI of the B200-native batched keyed-hash engine.
 *
 * The drop-in boundary for the reference package `lanehash`'s hash path
 * (/root/reference/pkg, S = pkg/src/lanehash, T = pkg/tests).  Each entry
 * point replaces one reference interface, cited beside it.  Plain pointers
 * and sizes only: every `d_*` pointer is CUDA device memory owned by the
 * caller, `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream) on the caller's current device.  The library never allocates or
 * frees caller memory and keeps no per-call state; launches are
 * asynchronous on `stream` and the caller synchronises.
 *
 * Conventions (identical to the reference):
 *   HighwayHash key: 4 little-endian u64 lanes (S/highway.py:43-57).
 *   SipHash key:     2 little-endian u64 words (S/sip.py:24-37).
 *   Digests: u64 lanes, lane 0 first; width 64 -> 1 lane per message,
 *   128 -> 2, 256 -> 4 (S/highway.py:223-234, 288-295).  Width 128 is not
 *   defined by the reference (S/highway.py:228-229); here it is lanes 0-1 of
 *   the 256-bit lane sum (derived, documented in DESIGN.md).
 *   rounds: HighwayHash finalization rounds (reference default 4,
 *   S/highway.py:223; tests use 1..3, T/test_backends.py:33-38).
 *
 * Return value: LH_OK (0) or a negative LH_E* code; lh_strerror() names it.
 * The Python host maps LH_EINVAL/LH_EALIGN to ValueError (as the reference
 * raises ValueError for bad widths/keys, S/highway.py:49-56, 228-229;
 * S/sip.py:60-62) and the others to RuntimeError.
 */
#ifndef LANEHASH_B200_H
#define LANEHASH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LH_OK 0
#define LH_EINVAL (-1)   /* bad argument: width, rounds, c/d, NULL pointer */
#define LH_EALIGN (-2)   /* misaligned output / offsets / lengths pointer */
#define LH_ECUDA (-3)    /* CUDA runtime error (launch, attribute, ...) */
#define LH_ENODEV (-4)   /* no usable sm_100 device */
#define LH_ETOOBIG (-5)  /* size outside the supported range */

/* Kernel selection for the *_kernel entry points (tests and bench force a
 * path; the plain entry points choose automatically). */
#define LH_KERNEL_AUTO 0
#define LH_KERNEL_DIRECT 1 /* one thread per message, direct global loads */
#define LH_KERNEL_TMA 2    /* TMA-staged shared-memory ring (fixed length) */
#define LH_KERNEL_SPLIT 3  /* HighwayHash only: state split over 2 threads per
                              message (long messages; len % 128 == 0) */
#define LH_KERNEL_STAGED 4 /* HighwayHash: warp-staged short-key kernel
                              (ragged, or fixed rows) */
#define LH_KERNEL_RING 5   /* one thread per message, branch-free 16-byte
                              word reader with packets in flight (fixed or
                              ragged) */

/* Library / build identification. */
const char* lh_version(void);
const char* lh_strerror(int code);

/* HighwayHash over n contiguous messages of `len` bytes each.
 * Replaces: NumpyBackend.hash64_batch (S/backends.py:52-53 ->
 * S/_highway_np.py:116-130), the numba batch _kernels.hash_batch(algo 0)
 * (S/_kernels.py:268-274) and, at n = 1, backend.hash64/hash256
 * (S/backends.py:28-33, 75-80).  d_out holds n * width/64 u64. */
int lh_highway_fixed(const uint8_t* d_msgs, uint64_t n, uint64_t len,
                     const uint64_t key[4], int width, int rounds,
                     uint64_t* d_out, void* stream);
/* kernel: any LH_KERNEL_*.  AUTO: TMA for rows that are 16-byte multiples
 * (>= 1,024 rows), SPLIT for few long rows, STAGED for rows <= 64 B and
 * RING for longer rows that TMA cannot take. */
int lh_highway_fixed_kernel(const uint8_t* d_msgs, uint64_t n, uint64_t len,
                            const uint64_t key[4], int width, int rounds,
                            uint64_t* d_out, void* stream, int kernel);

/* HighwayHash over a packed ragged buffer: message i is
 * d_buf[d_offsets[i] : d_offsets[i] + len_i], len_i = d_lengths[i] when
 * d_lengths != NULL, else d_offsets[i+1] - d_offsets[i] (offsets has n+1
 * entries).  Offsets are byte offsets with no alignment requirement.
 * Replaces: per-message backend.hash64/hash256 (S/backends.py:22-80) over a
 * batch of unequal lengths (the reference has no ragged API). */
int lh_highway_ragged(const uint8_t* d_buf, const uint64_t* d_offsets,
                      const uint32_t* d_lengths, uint64_t n,
                      const uint64_t key[4], int width, int rounds,
                      uint64_t* d_out, void* stream);
/* kernel: LH_KERNEL_AUTO or LH_KERNEL_STAGED = warp-staged short-key kernel
 * (messages <= 64 B packed together; any other warp reads its messages
 * directly);
 * LH_KERNEL_RING (or LH_KERNEL_DIRECT) = one thread per message with a
 * register ring of packets in flight (medium/long messages, e.g. the
 * L = 0..1023 sweep). */
int lh_highway_ragged_kernel(const uint8_t* d_buf, const uint64_t* d_offsets,
                             const uint32_t* d_lengths, uint64_t n,
                             const uint64_t key[4], int width, int rounds,
                             uint64_t* d_out, void* stream, int kernel);

/* SipHash-c-d (tree = 0) or SipTreeHash (tree = 1), n contiguous messages.
 * Replaces: sip.siphash / sip.siptreehash (S/sip.py:89-128) and the numba
 * _kernels.hash_batch algo 1 / 2 (S/_kernels.py:184-244, 268-274). */
int lh_siphash_fixed(const uint8_t* d_msgs, uint64_t n, uint64_t len,
                     const uint64_t key[2], int c, int d, int tree,
                     uint64_t* d_out, void* stream);
/* kernel: LH_KERNEL_AUTO, LH_KERNEL_DIRECT, LH_KERNEL_TMA or LH_KERNEL_RING
 * (SPLIT and STAGED are HighwayHash only). */
int lh_siphash_fixed_kernel(const uint8_t* d_msgs, uint64_t n, uint64_t len,
                            const uint64_t key[2], int c, int d, int tree,
                            uint64_t* d_out, void* stream, int kernel);
int lh_siphash_ragged(const uint8_t* d_buf, const uint64_t* d_offsets,
                      const uint32_t* d_lengths, uint64_t n,
                      const uint64_t key[2], int c, int d, int tree,
                      uint64_t* d_out, void* stream);
/* kernel: LH_KERNEL_AUTO, LH_KERNEL_RING or LH_KERNEL_DIRECT (the same
 * kernel: one thread per message, the register-ring reader described
 * above). */
int lh_siphash_ragged_kernel(const uint8_t* d_buf, const uint64_t* d_offsets,
                             const uint32_t* d_lengths, uint64_t n,
                             const uint64_t key[2], int c, int d, int tree,
                             uint64_t* d_out, void* stream, int kernel);

/* PRF mode: d_out[i] = HighwayHash-64(key, le64(start + i)), i < n.
 * Composition of S/highway.py:247-249 over 8-byte counters (no input
 * buffer). */
int lh_highway_prf64(uint64_t start, uint64_t n, const uint64_t key[4],
                     int rounds, uint64_t* d_out, void* stream);

/* ---- Batched streaming (incremental) hashing ----
 * Replaces: highway.StreamingHasher (S/highway.py:257-285), sip.SipHasher
 * (S/sip.py:131-169) and sip.SipTreeHasher (S/sip.py:172-203), for n
 * messages at once.  d_state holds n records of lh_stream_state_bytes(alg)
 * bytes (16-B aligned, caller-allocated): hasher state, <= 31 pending bytes,
 * total length.  For any split of each message into chunks, init + updates +
 * finish equals the one-shot digest (T/test_highway.py:156-193). */
#define LH_ALG_HIGHWAY 0
#define LH_ALG_SIPHASH 1
#define LH_ALG_SIPTREE 2
size_t lh_stream_state_bytes(int alg);
/* p1, p2 = width, rounds (HighwayHash) or c, d (SipHash / SipTreeHash). */
int lh_stream_init(int alg, void* d_state, uint64_t n, const uint64_t* key,
                   int p1, int p2, void* stream);
/* Append one chunk per message: fixed layout (d_offsets == NULL) chunk i is
 * d_buf[i*chunk_len : (i+1)*chunk_len]; ragged layout as lh_highway_ragged. */
int lh_stream_update(int alg, void* d_state, uint64_t n, const uint8_t* d_buf,
                     const uint64_t* d_offsets, const uint32_t* d_lengths,
                     uint64_t chunk_len, void* stream);
/* Digests of the appended data (state is not consumed).  lanes = 1, 2 or 4
 * (digest width / 64) for HighwayHash -- the absorbed state is
 * width-independent, as in S/highway.py:278-285 -- and 1 for the Sip family. */
int lh_stream_finish(int alg, const void* d_state, uint64_t n, uint64_t* d_out,
                     int lanes, void* stream);

/* ---- Quality harness: avalanche flip tallies ----
 * Replaces: _kernels.avalanche_counts (S/_kernels.py:247-265), the kernel of
 * the avalanche protocol (S/quality.py:105-194) and of the finalization-round
 * experiment (S/quality.py:245-293).  For each of `iters` messages of `size`
 * bytes (1..32) and each input bit b: d_counts[b*64 + ob] += bit ob of
 * hash(msg ^ bit b) ^ hash(msg).  Tallies are ACCUMULATED (caller zeroes).
 * alg: LH_ALG_HIGHWAY (64-bit digest, p1 = finalization rounds),
 * LH_ALG_SIPHASH / LH_ALG_SIPTREE (p1 = c, p2 = d).  d_msgs == NULL: message
 * i is the little-endian bytes of i (exhaustive enumeration). */
int lh_avalanche_counts(int alg, const uint64_t* key, const uint8_t* d_msgs,
                        uint64_t iters, uint32_t size, int p1, int p2,
                        int64_t* d_counts, void* stream);

/* ---- Raw Update and its inverse (test / self-test entries) ----
 * Replaces: update (S/highway.py:130-150) and update_inverse
 * (S/highway.py:153-173), which the reference uses as the bijectivity
 * oracle of T/test_update.py:56-67 and T/test_acceptance.py:42-63.
 * d_states: n x 16 u64 (v0[4], v1[4], mul0[4], mul1[4]), updated in place;
 * d_packets: n x 4 u64.  inverse: 0 = update, 1 = update_inverse.  The
 * device code is the Update every hashing kernel inlines. */
int lh_highway_update_states(uint64_t* d_states, const uint64_t* d_packets,
                             uint64_t n, int inverse, void* stream);
/* update_remainder (S/highway.py:182-199) on n caller states: tail i is
 * d_tails[32i .. 32i + d_r[i]) (bytes beyond are ignored), d_r[i] in 1..31;
 * a state whose d_r[i] is 0 or >= 32 is left unchanged (the reference
 * raises ValueError for such tails, S/highway.py:185-186; the Python
 * wrapper does, before launching). */
int lh_highway_remainder_states(uint64_t* d_states, const uint8_t* d_tails,
                                const uint32_t* d_r, uint64_t n, void* stream);
/* finalize (S/highway.py:223-234) of n caller states: `rounds`
 * PermuteAndUpdates, then width/64 lane sums per state into d_out
 * (n x width/64 u64, lane 0 first).  States are not modified.  width 128
 * is the derived width (lanes 0-1), as everywhere in this library. */
int lh_highway_finalize_states(const uint64_t* d_states, uint64_t n, int width,
                               int rounds, uint64_t* d_out, void* stream);
/* sip_round (S/sip.py:73-86) applied `rounds` times to n caller states
 * (n x 4 u64: v0, v1, v2, v3), in place -- the round every SipHash /
 * SipTreeHash kernel inlines. */
int lh_sip_round_states(uint64_t* d_states, uint64_t n, int rounds, void* stream);
/* Device self-test of the bijection on n synthetic cases: case i is words
 * 20i .. 20i+19 of the synthetic stream (seed, stream_id 0) -- 16 state
 * lanes, then 4 packet lanes.  ACCUMULATES (caller zeroes d_result[0..1]):
 * d_result[0] += #cases with update_inverse(update(s)) != s,
 * d_result[1] ^= XOR of all 16 lanes of update(s) over the cases. */
int lh_highway_bijectivity(uint64_t seed, uint64_t n, uint64_t* d_result,
                           void* stream);

/* One pass over a ragged layout (offsets[n+1] form when d_lengths == NULL):
 * for chunk k = messages [k*chunk_msgs, min(n, (k+1)*chunk_msgs)),
 * d_lo[k] = min start and d_hi[k] = max end (byte offsets; chunks with no
 * message keep lo = UINT64_MAX, hi = 0), and *d_bad = the number of invalid
 * messages: offsets[i+1] < offsets[i], start + length wrapping, or end >
 * buf_len (UINT64_MAX: no bound).  At most 65,535 chunks.  The hashing entry
 * points TRUST offsets/lengths (they read buf + offsets[i] unchecked); the
 * Python host runs this pass first and raises ValueError on *d_bad != 0, and
 * uses the spans to copy only each chunk's bytes.  Replaces: nothing in the
 * reference (it has no ragged API); the reference's per-message calls cannot
 * index out of a Python bytes object. */
int lh_ragged_plan(const uint64_t* d_offsets, const uint32_t* d_lengths, uint64_t n,
                   uint64_t chunk_msgs, uint64_t buf_len, uint64_t* d_lo,
                   uint64_t* d_hi, uint64_t* d_bad, void* stream);

/* lh_ragged_plan plus the lane balance of the natural message order.  With
 * work(i) = (len_i >> unit_shift) + fixed_units (32-byte packets + 5 for
 * HighwayHash, 8-byte words + 3 for SipHash: the per-message finalization),
 * d_stats[0] = sum of work and d_stats[1] = the sum over groups of 32
 * consecutive messages of 32 * max work -- the lane-steps a one-message-per-
 * lane kernel spends.  d_stats[0] / d_stats[1] is the warp efficiency of the
 * natural order; the Python host calls lh_ragged_order when it is below 0.8.
 * d_stats may be NULL (then identical to lh_ragged_plan). */
int lh_ragged_plan_stats(const uint64_t* d_offsets, const uint32_t* d_lengths, uint64_t n,
                         uint64_t chunk_msgs, uint64_t buf_len, uint64_t* d_lo, uint64_t* d_hi,
                         uint64_t* d_bad, uint64_t* d_stats, unsigned unit_shift,
                         unsigned fixed_units, void* stream);

/* Length-class schedule of a ragged batch: d_sched[0..n) becomes the
 * messages as 16-byte records {u64 offset, u32 length, u32 index} grouped by
 * length class, longest first (classes of len >> unit_shift: exact below 128
 * units, then 8 per octave), so that the 32 lanes of a warp of the ordered
 * kernels hash messages of nearly equal length.  A length >= 2^32 - 1 is
 * stored saturated (0xFFFFFFFF: the kernels re-read it from the layout).  A
 * counting sort in three launches; d_sched = 16 * n bytes, 16-byte aligned;
 * d_scratch = 1,024 u32 of device scratch.  n < 2^32.  The order inside a
 * class is unspecified; digests do not depend on it.  Replaces: nothing in
 * the reference (per-message calls have no lanes to balance). */
int lh_ragged_order(const uint64_t* d_offsets, const uint32_t* d_lengths, uint64_t n,
                    unsigned unit_shift, void* d_sched, uint32_t* d_scratch, void* stream);

/* lh_highway_ragged / lh_siphash_ragged with a schedule: thread t hashes the
 * message of record d_sched[t] (lh_ragged_order's output, or any permutation
 * of the batch in that format) and writes its digest to d_out[index] -- the
 * output is in message order, identical to the unordered calls.
 * Register-ring kernel; n < 2^32. */
int lh_highway_ragged_ordered(const uint8_t* d_buf, const uint64_t* d_offsets,
                              const uint32_t* d_lengths, uint64_t n, const void* d_sched,
                              const uint64_t key[4], int width, int rounds, uint64_t* d_out,
                              void* stream);
int lh_siphash_ragged_ordered(const uint8_t* d_buf, const uint64_t* d_offsets,
                              const uint32_t* d_lengths, uint64_t n, const void* d_sched,
                              const uint64_t key[2], int c, int d, int tree, uint64_t* d_out,
                              void* stream);

/* Seeded synthetic input generator (bench/test harness; not a reference
 * interface).  Byte b of the stream is byte (b & 7) of
 * word(seed, stream_id, word_offset + b / 8), see DESIGN.md §Synthetic
 * inputs; fills nbytes bytes.  d_buf must be 8-byte aligned. */
int lh_synth_fill(uint8_t* d_buf, uint64_t nbytes, uint64_t seed,
                  uint64_t stream_id, uint64_t word_offset, void* stream);
/* Lengths uniform in [lo, hi]: len[i] = lo + hi32(word(seed, 0, first+i)) *
 * (hi - lo + 1) >> 32. */
int lh_synth_lengths(uint32_t* d_len, uint64_t n, uint64_t seed,
                     uint64_t first, uint32_t lo, uint32_t hi, void* stream);

/* Harness: stream-read nbytes (16-byte aligned; the tail past the last
 * 16-byte unit is ignored) and XOR-fold them into d_sink[0..63] (zero it
 * first).  bench.py times it to measure the HBM read ceiling in-run. */
int lh_read_probe(const uint8_t* d_buf, uint64_t nbytes, uint64_t* d_sink, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LANEHASH_B200_H */
