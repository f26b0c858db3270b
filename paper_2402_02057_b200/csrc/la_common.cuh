// Shared device-side data structures of the B200 lookahead engine.
//
// Everything a decode needs lives in device memory: the 2-D window, the
// n-gram pool, the pre-generated window RNG stream, the output tokens and the
// per-step records.  The host only uploads inputs once per decode and reads
// outputs once at the end (SURVEY.md §8(b) "Ownership").
#pragma once
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define LA_MAX_ROWS 128      // query rows per forward (M_max = (N-1)(W+G) <= 128)
#define LA_MAX_CHAIN 128     // visible step keys per row (chain length)
#define LA_MAX_SUFFIX 7      // N <= 8
#define LA_WARP 32

// ----------------------------------------------------------------- pool
// GPU-resident n-gram pool (reference pool.py:17-90).
//  * lead table: open-addressing hash keyed by the first token; slot i owns a
//    bucket of C most-recent suffixes, newest first.  Keeping C >= G recency
//    slots per lead gives lookups identical to the unbounded reference pool
//    (SURVEY.md appendix A.4).
//  * distinct set: open-addressing hash over the full n-gram; its size is
//    len(pool) (StepRecord.pool_size, types.py:107).
//  * log: every insert in order, replayed on the host into a caller-owned
//    pool object so `decode_lookahead(..., pool=p)` mutates `p` like the
//    reference (decoding.py:72-82).
struct DevPool {
  int ngram;       // N
  int C;           // bucket capacity (unbounded pool): >= G (newest-C per lead suffices
                   // for lookups)
  int lt_mask;     // lead table size - 1 (power of two)
  int st_mask;     // distinct set size - 1 (power of two)
  int log_cap;
  int capacity;    // NGramPool(capacity=...) global LRU cap; 0 = unbounded
  int* lead_keys;  // [LT]   -1 = empty
  int* bkt_cnt;    // [LT]   bucket length (unbounded) / live entries of the lead (capped)
  int* bkt_suf;    // [LT][C][N-1] newest-first suffixes (unbounded pool only)
  // LRU-capped pool: each lead's live entries form a newest-first doubly
  // linked list threaded through the distinct-set slots, so memory stays
  // O(LT + ST) for any capacity and an eviction is an O(1) unlink
  int* lead_head;  // [LT]   newest set slot of the lead, -1 = none
  int* set_prev;   // [ST]   newer entry of the same lead (-1: list head)
  int* set_next;   // [ST]   older entry of the same lead (-1: list tail)
  int* set_keys;   // [ST][N]  key[0] == -1 -> empty
  int* set_stamp;  // [ST] last-touch stamp, -1 = evicted (capacity mode)
  int* fifo;       // [log_cap] set slot touched by stamp s (capacity mode)
  int* counters;   // [0] = distinct n-grams, [1] = log length, [2] = stamps issued, [3] = fifo head
  int* log;        // [log_cap][N]
};

// ------------------------------------------------------- forward plan
// One forward pass = n_rows query rows.  Row m:
//   token ids[m] at absolute position pos[m]; its K/V go to cache slot
//   slot[m]; it attends to cache slots [0, n_prefix) (the confirmed prefix)
//   followed by chain_n[m] step slots chain[m][*] in relative-position order
//   and finally itself.  This chain form is the reference's visibility
//   contract (models.py:33-64): exactly one visible token per relative
//   position below the row's own, so the paper's structured mask is
//   *generated* per row instead of materialised as an M x M matrix.
struct FwdPlan {
  int n_rows;      // 0 -> every forward kernel exits immediately
  int n_pad;       // n_rows rounded up to 16 (MMA N)
  int n_prefix;    // ctx
  int n_global;    // rows of the whole step layout (all LP shards); step keys
                   // sit at slots n_prefix + global row
  int want_logits; // dump fp32 logits (parity hook)
  int ids[LA_MAX_ROWS];
  int pos[LA_MAX_ROWS];
  int slot[LA_MAX_ROWS];
  int grow[LA_MAX_ROWS];   // global row id (lookahead layout row)
  int own[LA_MAX_ROWS];    // 1 if this rank owns the row's output
  int chain_n[LA_MAX_ROWS];
  int chain[LA_MAX_ROWS][LA_MAX_CHAIN];
};

// Deferred RMSNorm statistics: per 128-feature tile partial sums of x^2 of
// each row ([tiles][128]); a consumer scales its projection accumulator by
// rsqrt(sum / d + eps) (the projection consumed bf16(x * g)).
struct LaRowNorm {
  const float* ss;
  int tiles;       // d / 128
  float inv_d;     // 1 / d
  float eps;
};

// ----------------------------------------------------------- decode state
enum { LA_MODE_LOOKAHEAD = 0, LA_MODE_AUTOREGRESSIVE = 1 };

// numpy PCG64 bit-generator state (128-bit LCG + the buffered upper half that
// next_uint32 hands out on its second call); la_sample.cuh advances it
struct LaPcg64 {
  unsigned long long s_hi, s_lo, i_hi, i_lo;
  int has32;
  unsigned u32;
};

struct DevDecode {
  // configuration (GenerationConfig, types.py:70-97)
  int mode, W, N, G, V, max_tokens, eos;   // eos < 0: none
  int rank, world;                         // lookahead parallelism
  int max_steps;
  // status
  int ctx;        // cached tokens = len(prefix) - 1
  int last;       // prefix[-1]
  int n_out;      // emitted tokens (after EOS / budget truncation)
  int done;
  int n_steps;
  int rng_cur, rng_len;
  int c;          // candidates this step
  int M;          // logical rows (N-1)(W+c) of this step
  int k;          // accepted count of the last step
  int winner;     // first surviving branch (-1 none)
  int commit_ctx, commit_n, commit_base;   // KV commit of the last step
  int overflow;   // set if a device capacity was exceeded (host raises)
  // arrays
  int* window;    // (N-1)W - 1 cells (flat)
  const int* rng; // pre-generated integers(0, V) stream (appendix A.3)
  int* out;       // [max_tokens + N]
  int* rec;       // [max_steps][4] = accepted, candidates, queries, pool size
  int* cand;      // [G][N-1] this step's candidate suffixes
  int* amax;      // [LA_MAX_ROWS] argmax per *global* row (-1 = not computed here)
  int* accepted;  // [N]
  DevPool pool;
  // temperature sampler (SamplerSpec, types.py:43-67; sampling.py:22-85);
  // sample == 0: greedy and none of the fields below is read
  int sample;
  int pcg_window;       // window refills from `pcg` (step sessions) instead of the rng stream
  int top_k;            // 0: no top-k
  double temperature;   // p ** (1/T) unless T == 1
  double top_p;         // >= 1: no nucleus
  LaPcg64 pcg;          // the session generator after window_init
  int degenerate;       // DegenerateDistributionError raised on the device
  const float* logits;  // [LA_MAX_ROWS][V] this step's rows (global row order)
  double* adj;          // [1 + G(N-1)][V]: row 0, then branch b offset k at 1 + b(N-1) + k-1
  double* work;         // [V] verification's renormalised distribution
};

// ---------------------------------------------------------------- utils
__device__ __forceinline__ uint32_t la_mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ int la_round16(int x) { return (x + 15) & ~15; }

#define LA_CUDA_CHECK(expr)                                                   \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      la_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                 \
                   cudaGetErrorString(_e));                                   \
      return LA_ERR_CUDA;                                                     \
    }                                                                         \
  } while (0)

// ------------------------------------------------ programmatic dependent launch
// Every kernel of the step graph is launched with programmatic stream
// serialisation: it lets its dependent start (launch_dependents) and then waits
// for its own prerequisites (wait) before touching their outputs.  Without the
// launch attribute both instructions are no-ops.
__device__ __forceinline__ void la_pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Optional in-graph timeline (LA_TIMELINE=1, profiling only): block 0 of
// every kernel stamps globaltimer when its dependency wait returns, with the
// launch shape as a signature.  buf[0] = record count, then pairs.
#define LA_TL_CAP 8192
#ifdef __CUDACC__
static __constant__ unsigned long long* g_la_tl;
#define LA_TL_DEFINE_SETTER(name)                                        \
  void la_tl_set_##name(unsigned long long* p) { cudaMemcpyToSymbol(g_la_tl, &p, sizeof(p)); }
#endif
// timeline record of this kernel's dependency release (profiling only)
__device__ __forceinline__ void la_tl_stamp() {
  if (g_la_tl && (threadIdx.x | threadIdx.y | blockIdx.x | blockIdx.y | blockIdx.z) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(reinterpret_cast<unsigned*>(g_la_tl), 1u);
    if (i < LA_TL_CAP) {
      g_la_tl[1 + 2 * i] = t;
      g_la_tl[2 + 2 * i] = ((unsigned long long)(gridDim.x * gridDim.y) << 16) | blockDim.x;
    }
  }
}
__device__ __forceinline__ void la_pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  la_tl_stamp();
}
#define LA_PDL_ENTRY() \
  do {                 \
    la_pdl_trigger();  \
    la_pdl_wait();     \
  } while (0)

#ifdef __CUDACC__
// cudaFuncSetAttribute is per device: set it once on each device a launch uses
// (a racing second setter is harmless; the bit is published after success)
template <typename F>
static inline cudaError_t la_smem_attr_once(std::atomic<unsigned>& done, F* kernel, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned bit = 1u << (dev & 31);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

// Every kernel of the step runs with the max-shared-memory carveout.  An SM
// whose running CTAs were launched with another L1/smem split cannot host a
// CTA that needs the larger smem partition until it drains, which defeats
// programmatic dependent launch: a GEMM behind a 0-smem epilogue kernel could
// only start (and begin streaming its weights) once the epilogue's CTAs left
// its SM (profiles/microbench/pdl_preload.cu: 0 of 148 secondary CTAs early
// with the default carveout, 148 of 148 with max-smem).  Opt-in
// (LA_CARVEOUT=1): in the decode step it measured +0.8 % -- the epilogue
// kernels' grids are larger than what fits beside a GEMM CTA anyway, and the
// GEMM's MMA issue, not its preload, paces its first units.
static inline void la_carveout_once(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  static const bool on = getenv("LA_CARVEOUT") && atoi(getenv("LA_CARVEOUT")) == 1;
  if (!on) return;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> g(mu);
  if (done.insert({dev, fn}).second)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}

// cudaLaunchKernelEx with the PDL attribute (pdl = false: plain launch)
template <typename... KArgs, typename... Args>
static inline cudaError_t la_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t st, bool pdl, Args... args) {
  la_carveout_once(reinterpret_cast<const void*>(kernel));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
#endif

// ------------------------------------------------------ L2 weight prefetch
// The latency-bound kernels between two GEMMs (epilogues, attention, norms)
// leave HBM idle.  They pull the NEXT GEMM's first weight units into L2
// (cp.async.bulk.prefetch.L2) so HBM keeps streaming while they run: for
// each GEMM CTA c, the first `frac` of its stream-K unit range.
struct LaPrefetch {
  const void* a;   // packed weights of the next GEMM (null: none)
  int n_tiles, kb, tpc, grid;
  float frac;
};

__device__ __forceinline__ void la_l2_prefetch_gemm(const LaPrefetch& pf) {
  if (!pf.a || pf.frac <= 0.f) return;
  // GEMM CTA c is prefetched by block (c mod nblk), thread c / nblk: the bulk
  // prefetches spread over every SM's copy engine instead of one CTA's
  const long nblk = (long)gridDim.x * gridDim.y * gridDim.z;
  const long bid = (long)blockIdx.x + (long)gridDim.x * (blockIdx.y + (long)gridDim.y * blockIdx.z);
  const long U = (long)(pf.n_tiles / pf.tpc) * pf.kb, P = pf.grid;
  const char* base = reinterpret_cast<const char*>(pf.a);
  for (long c = bid + (long)threadIdx.x * nblk; c < P; c += (long)blockDim.x * nblk) {
    const long u0 = c * U / P, u1 = (c + 1) * U / P;
    const long n = (long)((u1 - u0) * pf.frac + 0.999f);
    for (long u = u0; u < u0 + n && u < u1; ++u) {
      size_t off;
      uint32_t bytes;
      if (pf.tpc == 2) {
        off = (size_t)u * 32768;
        bytes = 32768;
      } else {   // single-tile unit inside the pair-interleaved packing
        const long t = u / pf.kb, k = u % pf.kb;
        off = ((size_t)((t / 2) * pf.kb + k) * 2 + (t % 2)) * 16384;
        bytes = 16384;
      }
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(bytes)
                   : "memory");
    }
  }
}

#define LA_PDL_ENTRY_PF(pf)   \
  do {                        \
    la_pdl_trigger();         \
    la_l2_prefetch_gemm(pf);  \
    la_pdl_wait();            \
  } while (0)
