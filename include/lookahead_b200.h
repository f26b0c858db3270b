/*
 * lookahead_b200.h -- C ABI of the B200-native greedy lookahead-decoding engine.
 *
 * Drop-in boundary for the reference package's hot path
 * (/root/reference/pkg/src/lookahead).  Plain C types only: host pointers,
 * device pointers as `const void*`, sizes as int32, CUDA streams as `void*`
 * (a cudaStream_t; NULL = legacy default stream).  Every entry point returns
 * LA_OK (0) or a negative LA_ERR_* code; la_last_error() returns a
 * thread-local message for the last failure on the calling thread.  The
 * Python host layer maps the codes back to the reference's exception
 * classes (ValueError, LayoutError).
 *
 * Threading (reference SPEC.md:100,332): one engine per (device, thread);
 * decodes on one engine are serialised by the caller; engines are independent.
 */
#ifndef LOOKAHEAD_B200_H
#define LOOKAHEAD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
#define LA_OK 0
#define LA_ERR_INVALID_CONFIG (-1) /* ValueError: types.py:87-97, decoding.py:75-80 */
#define LA_ERR_LAYOUT (-2)         /* LayoutError: types.py:13-15, models.py:46-62   */
#define LA_ERR_CUDA (-3)
#define LA_ERR_NCCL (-4)
#define LA_ERR_CAPACITY (-5) /* a device-side table or buffer would overflow */
#define LA_ERR_UNSUPPORTED (-6)
#define LA_MAX_ACCEPT 9         /* N <= 8: a step accepts <= N tokens */
#define LA_ERR_DEGENERATE (-7) /* DegenerateDistributionError: types.py, sampling.py:52-65,
                                  verification.py:108-110 */

/* Thread-local description of the last error on this thread. */
const char* la_last_error(void);
/* ABI version (bumped on any signature or struct-layout change; 2: la_decode_io.pool_capacity). */
int32_t la_abi_version(void);

/* ------------------------------------------------------------------ model */
#define LA_ARCH_GPT_F32 0    /* reference TinyTransformer, models.py:189-271 */
#define LA_ARCH_LLAMA_F32 1  /* Llama-style decoder, fp32 SIMT (parity model) */
#define LA_ARCH_LLAMA_BF16 2 /* Llama-2-shaped decoder, bf16 tcgen05 path    */

typedef struct la_model_desc {
  int32_t arch;
  int32_t vocab, dim, layers, heads, kv_heads, head_dim, ffn;
  float rope_theta, norm_eps;
  int32_t max_context; /* KV capacity in tokens (prompt + generated) */
} la_model_desc;

/* Number of weight tensors and the name of tensor i, in the order la_create
 * expects their device pointers.  fp32 archs: row-major [out][in] matrices.
 * LA_ARCH_LLAMA_BF16: the embedding is row-major [vocab][dim] bf16; every
 * projection ("*_tiles") is in the packed LA-tile layout produced by
 * la_pack_weight (q/k/v stacked into one matrix, gate/up interleaved per
 * 64 rows); norm vectors are fp32.  Replaces the reference's in-object numpy
 * weights (models.py:219-242). */
int32_t la_weight_count(const la_model_desc* desc);
const char* la_weight_name(const la_model_desc* desc, int32_t i);

/* Packed LA-tile layout of a bf16 [rows][K] matrix (K % 64 == 0): 128-row x
 * 64-column blocks, 16 KB each, tile-major / k-minor, every block stored as
 * its 128-byte-swizzled shared-memory image so the GEMM streams it with one
 * contiguous bulk copy.  la_packed_bytes: size of the packed matrix (rows
 * rounded up to 128; zero the buffer before packing partial tiles).
 * la_pack_weight: pack device matrix src into dst at virtual row offset
 * `row_offset` (mode 0), or as the gate (mode 1) / up (mode 2) half of an
 * interleaved gate/up matrix. */
int64_t la_packed_bytes(int32_t rows, int32_t K);
int32_t la_pack_weight(const void* src, int32_t rows, int32_t K, void* dst, int32_t mode,
                       int32_t row_offset, void* stream);

typedef struct la_engine la_engine;

/* Create an engine on `device`.  Weights are BORROWED device pointers that
 * must outlive the engine; KV cache, pool, window, RNG stream and scratch
 * are engine-owned.  Replaces constructing a ModelInterface
 * (models.py:67-93 / transformer_init models.py:274-284). */
int32_t la_create(const la_model_desc* desc, const void* const* weights, int32_t n_weights,
                  int32_t device, la_engine** out);
int32_t la_destroy(la_engine* e);

/* -------------------------------------------------------------- decoding */
/* GenerationConfig (types.py:70-97); eos_token < 0 means None. */
typedef struct la_gen_config {
  int32_t window, ngram, max_candidates, max_tokens, eos_token, seed_pool_from_prompt;
} la_gen_config;

/* Host-side inputs and outputs of one decode call. */
typedef struct la_decode_io {
  const int32_t* prompt;     /* [n_prompt] */
  int32_t n_prompt;
  const int32_t* rng_stream; /* default_rng(seed).integers(0, V, size=rng_len): the
                                window's only randomness (layout.py:117-125,243-250) */
  int32_t rng_len;
  const int32_t* pool_init;  /* existing pool entries, oldest first, N ints each */
  int32_t pool_init_n;
  int32_t* out_tokens;       /* [out_cap] generated tokens (decoding.py:214-232) */
  int32_t out_cap;
  int32_t n_out;             /* written */
  int32_t* step_records;     /* [rec_cap][4]: accepted, candidates, queries, pool size
                                (StepRecord, types.py:100-111); may be NULL */
  int32_t rec_cap;
  int32_t n_steps;           /* written */
  int32_t* pool_log;         /* [pool_log_cap][N]: every pool insert in order; may be NULL */
  int32_t pool_log_cap;
  int32_t pool_log_n;        /* written (total inserts, may exceed cap) */
  float prefill_ms;          /* written: CUDA-event time of the prompt prefill */
  float decode_ms;           /* written: CUDA-event time of the decode loop */
  int32_t launches;          /* written: kernels launched by the decode loop */
  int32_t pool_capacity;     /* NGramPool(capacity=...): global LRU cap (pool.py:41-61); 0 = none */
} la_decode_io;

/* decode_lookahead (decoding.py:235-255), greedy sampler only. */
int32_t la_decode_lookahead(la_engine* e, const la_gen_config* cfg, la_decode_io* io,
                            void* stream);

/* decode_autoregressive (decoding.py:96-116), greedy. */
int32_t la_decode_autoregressive(la_engine* e, int32_t max_tokens, int32_t eos_token,
                                 la_decode_io* io, void* stream);

/* ------------------------------------------------------ temperature sampler
 * SamplerSpec(mode="temperature") (types.py:43-67): p ** (1/T), top-k, top-p
 * (sampling.py:22-66), distribution-preserving verification
 * (verification.py:74-118).  The random stream is the session's numpy
 * default_rng(seed) (PCG64): the caller draws the initial window exactly like
 * start_session (decoding.py:83-84, window_init layout.py:117-125) into
 * io->rng_stream / rng_len = (N-1)W-1 cells and passes the generator state
 * AFTER those draws -- rng.bit_generator.state's 128-bit `state` and `inc`
 * as hi/lo words, `has_uint32`, `uinteger`.  The device then consumes the
 * identical stream: one random() per verification trial and draw, one
 * integers(0, V) per vacated window cell. */
typedef struct la_sampler {
  double temperature;        /* > 0 */
  int32_t top_k;             /* 0: none */
  double top_p;              /* (0, 1]; 1: none */
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
  int32_t has_uint32;
  uint32_t uinteger;
} la_sampler;

/* decode_lookahead (decoding.py:235-255) under a temperature sampler. */
int32_t la_decode_lookahead_sampled(la_engine* e, const la_gen_config* cfg, const la_sampler* s,
                                    la_decode_io* io, void* stream);

/* decode_autoregressive (decoding.py:96-116) under a temperature sampler:
 * one random() per token (sample_token, sampling.py:77-85); the generator
 * is default_rng(seed) untouched (io->rng_stream unused). */
int32_t la_decode_autoregressive_sampled(la_engine* e, int32_t max_tokens, int32_t eos_token,
                                         const la_sampler* s, la_decode_io* io, void* stream);

/* ------------------------------------------------------------ step session
 * start_session / lookahead_step (decoding.py:67-93,152-211): the decode
 * state stays on the device between steps.  greedy != 0: greedy
 * verification; else sampling verification with s's temperature / top-k /
 * top-p.  Either way s carries the session generator AFTER window_init
 * (io->rng_stream / rng_len = the (N-1)W-1 window cells drawn by the
 * caller); window refills continue that stream on the device.  Steps never
 * stop on EOS / max_tokens (the caller folds tokens, collect_output
 * decoding.py:214-232); a step past the engine's max_context fails with
 * LA_ERR_CAPACITY.  A whole-decode call on the engine ends the session. */
typedef struct la_step_outcome {   /* StepOutcome + StepRecord (decoding.py:44-50, types.py) */
  int32_t accepted[LA_MAX_ACCEPT]; /* 1..N tokens */
  int32_t n_accepted;
  int32_t new_top[64];             /* greedy tokens of the W generator rows */
  int32_t n_new_top;
  int32_t candidate_count, query_count;
  int32_t pool_size;               /* len(pool) after the step's inserts */
  int32_t pool_log_n;              /* pool inserts so far (incl. prompt seeding) */
} la_step_outcome;

int32_t la_session_start(la_engine* e, const la_gen_config* cfg, int32_t greedy,
                         const la_sampler* s, la_decode_io* io, void* stream);
int32_t la_session_step(la_engine* e, la_step_outcome* out, void* stream);
/* what 0: the window's (N-1)W-1 cells (SURVEY A.1 order); what 1: pool-log
 * n-grams [offset, offset + n), N ints each (inserts in order); what 2: the
 * session generator (reference DecodeState.rng, decoding.py:83) as 10 words --
 * PCG64 state lo32/hi32 of its high and low 64-bit halves, increment likewise,
 * has_uint32, uinteger (offset 0, n 10) */
int32_t la_session_read(la_engine* e, int32_t what, int32_t offset, int32_t n, int32_t* out);

/* Parity hooks (tests only).  la_adjust_distributions: adjusted_distribution
 * of n_rows fp64 probability rows [n_rows][V] on the device (host buffers;
 * out may alias probs).  la_verify_sample_dists: verify_sample of c
 * candidates (suffixes [c][S]) over fp64 distributions
 * [1 + c*S][V] = base, then candidate b's S rows; out[<= S+1] accepted. */
int32_t la_adjust_distributions(la_engine* e, const double* probs, int32_t n_rows, int32_t V,
                                const la_sampler* s, double* out, void* stream);
int32_t la_verify_sample_dists(la_engine* e, const double* dists, int32_t V, int32_t S,
                               int32_t c, const int32_t* suffixes, const la_sampler* s,
                               int32_t* out, int32_t* n_out, void* stream);

/* Tests only: a fresh device pool (n-gram size N, LRU capacity or 0, bucket
 * size C >= limit) fed n_grams n-grams in batches of `batch` (<= 64) through the
 * step-finish insert path (pool.py:41-67); after every batch, lookup(lead,
 * limit) (pool.py:69-81) for each of n_leads leads and len(pool):
 * out[batch][lead][limit][N-1], counts[batch][lead], lens[batch]. */
int32_t la_pool_test(int32_t N, int32_t capacity, int32_t C, const int32_t* grams, int32_t n_grams,
                     int32_t batch, const int32_t* leads, int32_t n_leads, int32_t limit,
                     int32_t* out, int32_t* counts, int32_t* lens);

/* The generator as the device advances it, evaluated on the HOST (no GPU):
 * kind 0 random(), kind 1 integers(0, high); writes n values. */
int32_t la_pcg64_draws(const la_sampler* s, int32_t kind, int32_t high, int32_t n, double* out);

/* ModelInterface.forward parity hook (models.py:80-89): logits of n_rows
 * queries after `prefix`.  Row i has token ids[i], relative position rel[i]
 * and sees, in relative-position order, rows chain[i*chain_stride + 0 ..
 * rel[i]-1] (the reference's conditioning chain, models.py:33-64).  Writes
 * fp32 logits[n_rows][vocab] to HOST memory.  Test/parity use only: the
 * decode hot path never goes through this call. */
int32_t la_forward_layout(la_engine* e, const int32_t* prefix, int32_t n_prefix, int32_t n_rows,
                          const int32_t* ids, const int32_t* rel, const int32_t* chain,
                          int32_t chain_stride, float* logits, void* stream);

/* Jacobi decoding (replaces decode_jacobi, decoding.py:119-149): solve the
 * m-token greedy continuation of `prompt` by parallel fixed-point iteration
 * from the initial guess `init` (the caller draws it like the reference:
 * rng.integers(0, V, m)).  Each iteration is one forward of the triangular
 * chain layout (layout.py:185-194), m + 1 rows; stops when an iterate
 * repeats, after at most m iterations.  out_tokens[m] = the fixed point,
 * iterates[n_iterations][m] (may be null) = every iterate after the guess.
 * m + 1 <= 128 rows; ValueError cases as the reference (empty prompt, m < 1). */
int32_t la_decode_jacobi(la_engine* e, const int32_t* prompt, int32_t n_prompt, int32_t m,
                         const int32_t* init, int32_t* out_tokens, int32_t* iterates,
                         int32_t* n_iterations, void* stream);

/* ------------------------------------------------- lookahead parallelism */
/* LP (parallel.py:145-192): rank `rank` of `world` replicas, each holding the
 * full model, evaluates its share of window columns and candidate branches;
 * one NCCL all-gather per step exchanges the argmax ids, a second exchanges
 * the K/V rows of the accepted branch.  `unique_id` is an ncclUniqueId
 * (128 bytes) produced by la_lp_unique_id on rank 0 and broadcast by the
 * caller. */
int32_t la_lp_unique_id(void* out_128_bytes);
int32_t la_lp_init(la_engine* e, const void* unique_id, int32_t rank, int32_t world);

/* In-process LP over `n` engines on ONE device (the reference's simulated
 * decode_lookahead_devices, parallel.py:172-192): engine i acts as rank i;
 * the per-step exchange is a device copy.  All engines must share weights
 * and descriptor.  io is rank 0's; outputs are identical on every rank. */
int32_t la_decode_lookahead_group(la_engine* const* engines, int32_t n, const la_gen_config* cfg,
                                  la_decode_io* io, void* stream);

/* ------------------------------------------------------------ profiling */
/* Per-launch device time of the bf16 path's tcgen05 GEMMs, accumulated in
 * the kernels themselves (globaltimer, first CTA start -> last CTA end) over
 * every launch since the last reset.  out16[4*k + 0] = summed ns,
 * out16[4*k + 1] = launches, for k = 0 QKV, 1 O/down (residual), 2 gate/up,
 * 3 LM head. */
int32_t la_gemm_timing_enable(la_engine* e, int32_t on);   /* off by default (costs ~4 % of a step) */
int32_t la_gemm_timing_reset(la_engine* e);
int32_t la_gemm_timing_read(la_engine* e, double* out16);
/* Device time of the persistent forward kernel (bf16 path): out2 = {summed ns,
 * launches} since la_gemm_timing_reset.  Profiling only; no reference
 * counterpart (the reference has no device). */
int32_t la_forward_timing_read(la_engine* e, double* out2);

/* ------------------------------------------------------------ debugging */
/* Copy an engine buffer to host (tests only): what = 0 argmax table
 * (int32[128]), 1 K cache, 2 V cache ([layer][slot][kv_heads*head_dim]),
 * 3 device decode state, 4 forward plan, 5 per-CTA GEMM trace of the last
 * launch of each GEMM kind (needs LA_GEMM_TRACE=1 at engine creation:
 * uint64[4 kinds][256 CTAs][4] globaltimer stamps).  Synchronises the device. */
int32_t la_debug_read(la_engine* e, int32_t what, void* host, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* LOOKAHEAD_B200_H */
