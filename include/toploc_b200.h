/*
 * toploc_b200.h -- C ABI of the B200-native TOPLOC rollout-verification path.
 *
 * Drop-in boundary.  The reference binds the path by NAME at three Python
 * import sites (no plugin registry):
 *   - prove:  swarm/worker/rollout.py:51-68      build_commitments(hidden, k=32)
 *             called at rollout.py:112 (generate_group) and adversaries.py:312
 *   - verify: swarm/validator/checks.py:209-213   recompute + digest-list compare
 *   - wire:   swarm/worker/files.py:37,184-186     commitments[] = ceil(T/k) items
 * The Python host layer (paper_2505_07291_b200.api / .swarm_adapter) keeps those
 * names and signatures and calls the entry points below through ctypes; a
 * ctypes / cffi / pybind binding is all a maintainer of the reference adds
 * (INTEGRATION.md).
 *
 * Conventions
 *   - every pointer argument is DEVICE memory unless its name ends in _host;
 *     buffers are caller-owned; the library allocates nothing on the call path;
 *   - calls are stream-ordered and asynchronous on `stream` (a cudaStream_t,
 *     NULL = legacy default stream); no host synchronisation inside;
 *   - return 0 on success or a negative TL_E* code; tl_strerror() names it;
 *   - the library's only device globals are the GF(p) inverse tables (1 MiB, built
 *     once per device by the first tl_commit and immutable afterwards) and a per-kernel
 *     "attribute set" flag on the host; no other global state (safe from many host threads,
 *     one stream per thread / device);
 *   - a workspace (tl_workspace_bytes) serves one call at a time: calls that may
 *     run concurrently need their own.  Between calls it carries the select
 *     kernels' threshold speculation, which only steers speed (any content,
 *     including uninitialised memory, gives the same results).
 *
 * Layout
 *   hidden   : bf16 bit patterns, row-major (n_rows, H), rollouts concatenated
 *              along rows; row_off[n_roll + 1] (int64) delimits rollout r as rows
 *              [row_off[r], row_off[r+1]): non-decreasing, row_off[0] >= 0 and
 *              row_off[n_roll] <= n_rows (device memory, so not validated on the host;
 *              the -DTL_CHECKED build traps on a chunk outside [0, n_rows)).
 *   chunk j  : the j-th block of C rows of a rollout (final block partial),
 *              numbered across rollouts in order; n_chunks = sum ceil(T_r / C).
 *   proofs   : uint8 [n_chunks][2 + 2K]  (K = 128 -> 258 bytes) :
 *              modulus p (u16 BE) then coefficients c_0..c_{K-1} (u16 BE).
 */
#ifndef TOPLOC_B200_H_
#define TOPLOC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TL_OK 0
#define TL_EINVAL (-1)        /* bad shape / argument                         */
#define TL_EUNSUPPORTED (-2)  /* K > 128, C*H >= 2^24, ...                     */
#define TL_EWORKSPACE (-3)    /* workspace too small or misaligned            */
#define TL_ECUDA (-4)         /* kernel launch / CUDA runtime failure          */

#define TL_MAX_K 128
#define TL_PROOF_BYTES(K) (2 + 2 * (K))

/* Verdict thresholds; a chunk is accepted iff all three hold (<=). */
typedef struct tl_thresholds {
  int32_t max_exp_mismatch;
  int32_t _pad;
  double max_mant_mean;
  double max_mant_median;
} tl_thresholds;

/* Per-chunk verification statistics (32 bytes). mean/median = +inf when no
 * exponent matches or the proof is invalid (p is not a prime in [32771, 65497]). */
typedef struct tl_chunk_stats {
  uint32_t exp_mismatch;   /* points whose exponent field differs            */
  uint32_t n_match;        /* points whose exponent field agrees             */
  uint32_t mant_sum;       /* sum |mantissa diff| over matching points       */
  uint32_t flags;          /* bit0 accept, bit1 invalid proof                */
  double mant_mean;
  double mant_median;
} tl_chunk_stats;

#define TL_STAT_ACCEPT 1u
#define TL_STAT_BADPROOF 2u

const char* tl_strerror(int code);
int tl_version(void);

/* Host helper: sum_r ceil((row_off_host[r+1]-row_off_host[r]) / C). */
int64_t tl_count_chunks(const int64_t* row_off_host, int32_t n_roll, int32_t C);

/* Device scratch needed by tl_prove / tl_verify for this problem (bytes). */
size_t tl_workspace_bytes(int32_t n_roll, int64_t n_chunks, int32_t K);

/*
 * PROVE (replaces build_commitments at rollout.py:51-68 / :112).
 * Top-K of every chunk by |bf16| (ties -> lower flat index), GF(p)
 * interpolation, proof serialisation.  idx_out (int32 [n_chunks][K]) and
 * bits_out (uint16 [n_chunks][K]) are optional (NULL); entries past
 * kk = min(K, rows*H) are -1 / 0.
 */
int tl_prove(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
             int32_t H, int32_t C, int32_t K, int64_t n_chunks, uint8_t* proofs_out,
             int32_t* idx_out, uint16_t* bits_out, void* workspace, size_t workspace_bytes,
             void* stream);

/*
 * The two stages of tl_prove, exposed separately (north-star subsystems (a) and
 * (b)); tl_prove == tl_select + tl_commit on the same stream.
 *   tl_select: idx_out / bits_out required (int32 / uint16 [n_chunks][K]).
 *   tl_commit: reads idx / bits as written by tl_select (entries past kk = -1),
 *              writes proofs_out [n_chunks][2 + 2K].
 */
int tl_select(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
              int32_t H, int32_t C, int32_t K, int64_t n_chunks, int32_t* idx_out,
              uint16_t* bits_out, void* workspace, size_t workspace_bytes, void* stream);
int tl_commit(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int32_t K,
              uint8_t* proofs_out, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Launch-shape variants for pipelining a stream of batches (the commitment of
 * batch k on a second stream, beside verify of batch k-1 and select of k+1).
 * ctas_per_sm = 0 leaves the shape to the library: batches of at most one chunk per
 * TMA-ring CTA (2 per SM) with 16-byte aligned chunks (H % 8 == 0) stream through the
 * TMA-ring kernels (tl_ring_grid), larger ones through the one-warp-per-chunk kernels at
 * full occupancy (18 CTAs per SM); -1 always selects the one-warp kernels, -2 the ring
 * kernels wherever the chunks are aligned; > 0 caps the one-warp grid (16 leaves the
 * registers for one commit CTA).  Results are identical;
 * co_resident = 1 runs the commitment with 8 warps (<= 64 registers) and a 64 KiB
 * half inverse table so that CTA fits beside them.  Results are identical.
 */
int tl_select_ex(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
                 int32_t H, int32_t C, int32_t K, int64_t n_chunks, int32_t* idx_out,
                 uint16_t* bits_out, void* workspace, size_t workspace_bytes, int32_t ctas_per_sm,
                 void* stream);
int tl_commit_ex(const int32_t* idx, const uint16_t* bits, int64_t n_chunks, int32_t K,
                 uint8_t* proofs_out, void* workspace, size_t workspace_bytes, int32_t co_resident,
                 void* stream);
/* Build the GF(p) inverse tables of the large-batch commitment on the current device and
 * wait for them (once per device; later calls return at once).  Optional: tl_commit builds
 * them itself on first use (a small batch's tl_commit -- at most 4 chunks per SM -- needs
 * none).  Not callable during stream capture (it synchronises). */
int tl_prepare(void);

/* Grid of the TMA-ring kernel for this call shape (verify = 0: tl_select_ex, 1:
 * tl_verify_ex), or 0 when the one-warp-per-chunk kernels serve it. */
int32_t tl_ring_grid(const uint16_t* hidden, int32_t H, int64_t n_chunks, int32_t ctas_per_sm, int32_t verify,
                     void* stream);
int tl_verify_ex(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
                 int32_t H, int32_t C, int32_t K, int64_t n_chunks, const uint8_t* proofs,
                 const tl_thresholds* thresholds_host, tl_chunk_stats* stats_out,
                 uint8_t* chunk_accept_out, uint8_t* rollout_accept_out, void* workspace,
                 size_t workspace_bytes, int32_t ctas_per_sm, void* stream);

/*
 * VERIFY (replaces the digest compare at checks.py:209-213).
 * Re-selects top-K on the validator's hidden states, evaluates each proof at
 * the validator's indices, computes the exponent / mantissa statistics and the
 * verdicts.  stats_out [n_chunks], chunk_accept_out [n_chunks] (0/1) and
 * rollout_accept_out [n_roll] (0/1, AND over the rollout's chunks) may be NULL
 * individually.
 */
int tl_verify(const uint16_t* hidden, const int64_t* row_off, int32_t n_roll, int64_t n_rows,
              int32_t H, int32_t C, int32_t K, int64_t n_chunks, const uint8_t* proofs,
              const tl_thresholds* thresholds_host, tl_chunk_stats* stats_out,
              uint8_t* chunk_accept_out, uint8_t* rollout_accept_out, void* workspace,
              size_t workspace_bytes, void* stream);

/*
 * SM partition for the pipelined schedule (driver green contexts): streams on two
 * disjoint SM sets of the current device.  streams_out[3]: two streams on the
 * streaming partition (select, verify) and one on the commit_sms partition (rounded
 * up to the driver's granularity, 8 on sm_100); sms_out[2] (nullable): SMs of the
 * streaming and the commitment partition.  Every entry point sizes its grid to the
 * partition of the stream it is given (tl_stream_sms).  Returns TL_EUNSUPPORTED where
 * the driver has no green contexts.  tl_partition_destroy synchronises and frees.
 */
int tl_partition_create(int32_t commit_sms, void** streams_out, int32_t* sms_out);
int tl_partition_destroy(void** streams);
int32_t tl_stream_sms(void* stream);

/*
 * Per-record checks that share the validator's prefill, in the
 * reference's order (checks.py:204-213): termination (checks.py:120-131), then
 * sampling (checks.py:134-142), then the commitment verdict.
 *   probs         : float64 chosen-token probabilities, rollouts concatenated,
 *                   delimited by row_off (device int64 [n_roll + 1]);
 *   prompt_len    : device int32 [n_roll]; ends_with_eos: device uint8 [n_roll]
 *                   (output[-1] == eos_id);
 *   commit_accept : nullable device uint8 [n_roll], e.g. tl_verify's rollout verdicts;
 *   commit_checked: nullable device uint8 [n_roll], 1 = in the commitment sample
 *                   (checks.py:145-151); NULL = every record is checked;
 *   verdict_out   : device int32 [n_roll]: 0 accept, 1 termination, 2 sampling,
 *                   3 commitment (first failing check);
 *   frac_out, p_last_out: nullable device float64 [n_roll]: fraction of probs
 *                   below p_low (exact count / T), probs[T-1] (NaN when T = 0).
 * A record with T = 0 fails termination unless prompt_len >= max_len.
 */
typedef struct tl_record_thresholds {
  int32_t max_len;           /* ModelConfig.max_len                       */
  int32_t min_sampling_len;  /* CheckContext.min_sampling_len (16)         */
  double eos_prob_floor;     /* CheckContext.eos_prob_floor (0.1)          */
  double p_low;              /* CheckContext.p_low (0.005)                 */
  double theta;              /* CheckContext.theta (0.25)                  */
} tl_record_thresholds;

int tl_record_checks(const double* probs, const int64_t* row_off, int32_t n_roll,
                     const int32_t* prompt_len, const uint8_t* ends_with_eos,
                     const tl_record_thresholds* thresholds_host, const uint8_t* commit_accept,
                     const uint8_t* commit_checked, int32_t* verdict_out, double* frac_out,
                     double* p_last_out, void* stream);

/*
 * Exact mode (reference parity shim for build_commitments, rollout.py:65):
 * out[i] = round(in[i], 6) as float64 == rint(x * 1e6) / 1e6 (numpy semantics,
 * NaN payload kept and quieted).  dtype: 0 f64, 1 f32, 2 bf16, 3 f16.
 */
int tl_round6(const void* in, int32_t dtype, int64_t n, double* out, void* stream);

/*
 * Exact mode, whole chains on the GPU: for each rollout r of `hidden` (dtype as
 * tl_round6, rows delimited by row_off, device int64 [n_roll+1]), the reference's
 * commitment chain d_j = SHA-256(d_{j-1} || LE-f64(round(block_j, 6))) over k-row
 * blocks (one digest for T = 0).  digest_off (device int64 [n_roll]) gives each
 * rollout's first digest; digests_out receives 32 bytes per digest.  One lane per
 * rollout (a producer warp packs the message blocks, a SHA warp compresses them):
 * faster than host SHA-NI on all cores from ~700 rollouts.  Replaces
 * swarm/worker/rollout.py:51-68 (build_commitments) for a batch of rollouts.
 */
int tl_exact_chains(const void* hidden, int32_t dtype, const int64_t* row_off, int32_t n_roll,
                    int32_t H, int32_t k, const int64_t* digest_off, uint8_t* digests_out,
                    void* stream);

/*
 * Synthetic bf16 hidden states (bench/test input; counter-based, CPU-replayable,
 * see paper_2505_07291_b200/synth.py).  normal_table: device uint16[65536].
 * massive: 6 channel ids (dist 1).  jitter_thr/65536 of elements get +-1 in
 * the magnitude bits.
 */
int tl_synth_bf16(uint16_t* out, int64_t row0, int64_t n_rows, int32_t H, uint64_t seed_mix,
                  int32_t dist, const uint16_t* normal_table, const int32_t* massive_host,
                  int32_t jitter_thr, uint64_t jitter_mix, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TOPLOC_B200_H_ */
