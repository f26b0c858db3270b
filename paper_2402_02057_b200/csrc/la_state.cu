// Standalone kernels of the device step state machine (bf16 multi-kernel path
// and pool seeding).  The logic lives in la_state.cuh and is shared with the
// fp32 megakernel.
#include "la_state.cuh"
#include "la_kernels.h"

// Replay existing pool entries and/or the prompt's n-grams
// (pool.py:83-90 seed_from_prompt) in order, one warp.
__global__ void la_pool_seed_kernel(DevDecode* dp, const int* grams, int n, int log_from) {
  DevDecode& d = *dp;
  const int lane = threadIdx.x;
  for (int i = 0; i < n; ++i) {
    la_pool_insert_warp(d.pool, grams + (size_t)i * d.N, lane, &d.overflow);
    // the first `log_from` inserts replay a caller pool: not new inserts
    if (i + 1 == log_from && lane == 0) d.pool.counters[1] = 0;
    __syncwarp();
  }
}

// Parity hook (tests): replay n-gram batches through the device pool -- the
// K10 insert path (block-parallel, or serial under an LRU cap) -- and after
// every batch record lookup(lead, limit) for each requested lead and len(pool).
__global__ void __launch_bounds__(256) la_pool_test_kernel(DevPool pool, const int* grams, int n_grams,
                                                           int batch, const int* leads, int n_leads,
                                                           int limit, int* out, int* counts, int* lens,
                                                           int* overflow) {
  const int N = pool.ngram, S = N - 1;
  const int nb = (n_grams + batch - 1) / batch;
  for (int b = 0; b < nb; ++b) {
    const int g0 = b * batch, W = min(batch, n_grams - g0);
    if (pool.capacity == 0) {
      la_pool_insert_batch(pool, grams + (size_t)g0 * N, W, overflow);
    } else if (threadIdx.x < 32) {
      for (int j = 0; j < W; ++j) la_pool_insert_warp(pool, grams + (size_t)(g0 + j) * N, threadIdx.x, overflow);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < n_leads; q += blockDim.x) {
      const int slot = la_lead_find(pool, leads[q]);
      counts[(size_t)b * n_leads + q] =
          la_pool_lookup(pool, slot, limit, out + ((size_t)b * n_leads + q) * limit * S);
    }
    if (threadIdx.x == 0) lens[b] = pool.counters[0];
    __syncthreads();
  }
}

// The step kernels run on a shared-memory copy of the decode state (one
// coalesced load, one store back): the state machine reads its scalar fields
// after every barrier, and from global memory each read is an L2 round trip.
__device__ __forceinline__ void la_dec_load(DevDecode& sd, const DevDecode* dp) {
  static_assert(sizeof(DevDecode) % 4 == 0, "DevDecode copy granularity");
  const int* src = reinterpret_cast<const int*>(dp);
  int* dst = reinterpret_cast<int*>(&sd);
  for (int i = threadIdx.x; i < (int)(sizeof(DevDecode) / 4); i += blockDim.x) dst[i] = src[i];
  __syncthreads();
}
__device__ __forceinline__ void la_dec_store(DevDecode* dp, const DevDecode& sd) {
  __syncthreads();
  const int* src = reinterpret_cast<const int*>(&sd);
  int* dst = reinterpret_cast<int*>(dp);
  for (int i = threadIdx.x; i < (int)(sizeof(DevDecode) / 4); i += blockDim.x) dst[i] = src[i];
}

// K1: prepare_step (decoding.py:152-157) as one CTA.
__global__ void __launch_bounds__(256) la_step_build_kernel(DevDecode* dp, FwdPlan* P) {
  __shared__ __align__(16) DevDecode sd;
  LA_PDL_ENTRY();
  la_dec_load(sd, dp);
  la_step_build(sd, *P);
  la_dec_store(dp, sd);
}

// K10: finish_step (decoding.py:160-204) as one CTA.
__global__ void __launch_bounds__(256) la_step_finish_kernel(DevDecode* dp) {
  __shared__ __align__(16) DevDecode sd;
  LA_PDL_ENTRY();
  la_dec_load(sd, dp);
  la_step_finish(sd);
  la_dec_store(dp, sd);
}

// Per-row argmax merge into the global-row array (owned rows only).
__global__ void la_scatter_amax_kernel(DevDecode* dp, const FwdPlan* P, const int* row_amax) {
  LA_PDL_ENTRY();
  const int n = P->n_rows;
  for (int r = threadIdx.x; r < n; r += blockDim.x)
    if (P->own[r]) dp->amax[P->grow[r]] = row_amax[r];
}

// Merge an all-gathered [world][LA_MAX_ROWS] argmax table (LP exchange).
__global__ void la_merge_amax_kernel(DevDecode* dp, const int* gathered, int world) {
  LA_PDL_ENTRY();
  for (int g = threadIdx.x; g < LA_MAX_ROWS; g += blockDim.x) {
    int v = -1;
    for (int r = 0; r < world; ++r) v = max(v, gathered[r * LA_MAX_ROWS + g]);
    dp->amax[g] = v;
  }
}

// KV caches are [layer][slot][row_bytes] (row_bytes = kv_heads*head_dim*elt,
// a multiple of 16).  The three kernels below move whole 16-byte vectors.

// KV commit of the accepted branch rows, in place.
// One thread per (layer, vector), i ascending: the destination slot ctx+i
// can only alias the source of an i' <= i, already read by this thread.
__global__ void la_kv_commit_kernel(const DevDecode* dp, uint8_t* kc, uint8_t* vc, int layers,
                                    int slots, int row_bytes) {
  LA_PDL_ENTRY();
  const int n = dp->commit_n;
  if (dp->mode != LA_MODE_LOOKAHEAD || n <= 0) return;
  const int ctx = dp->commit_ctx, base = dp->commit_base;
  const int per = row_bytes / 16;
  const long total = (long)layers * per;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    int l = (int)(idx / per), e = (int)(idx % per) * 16;
    size_t lb = (size_t)l * slots * row_bytes;
    for (int i = 1; i <= n; ++i) {
      size_t src = lb + (size_t)(ctx + base + i - 1) * row_bytes + e;
      size_t dst = lb + (size_t)(ctx + i) * row_bytes + e;
      *reinterpret_cast<uint4*>(kc + dst) = *reinterpret_cast<const uint4*>(kc + src);
      *reinterpret_cast<uint4*>(vc + dst) = *reinterpret_cast<const uint4*>(vc + src);
    }
  }
}

// LP: the owner of the first surviving branch packs its K/V rows into the
// all-gather send buffer [layers][N-1][2][row_bytes]; other ranks send stale bytes.
__global__ void la_kv_pack_kernel(const DevDecode* dp, const uint8_t* kc, const uint8_t* vc,
                                  uint8_t* send, int layers, int slots, int row_bytes) {
  const DevDecode& d = *dp;
  if (d.mode != LA_MODE_LOOKAHEAD || d.commit_n <= 0 || d.winner < 0) return;
  if ((d.winner % d.world) != d.rank) return;
  const int S = d.N - 1, n = d.commit_n;
  const int per = row_bytes / 16;
  const long total = (long)layers * n * 2 * per;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    int e = (int)(idx % per) * 16;
    long t = idx / per;
    int kv = (int)(t % 2); t /= 2;
    int i = (int)(t % n) + 1;
    int l = (int)(t / n);
    size_t src = (size_t)l * slots * row_bytes +
                 (size_t)(d.commit_ctx + d.commit_base + i - 1) * row_bytes + e;
    size_t dst = (((size_t)l * S + (i - 1)) * 2 + kv) * row_bytes + e;
    const uint8_t* cache = kv ? vc : kc;
    *reinterpret_cast<uint4*>(send + dst) = *reinterpret_cast<const uint4*>(cache + src);
  }
}

// LP: every rank writes the owner's gathered rows into slots ctx+1 .. ctx+n.
__global__ void la_kv_unpack_kernel(const DevDecode* dp, const uint8_t* gathered, size_t seg,
                                    uint8_t* kc, uint8_t* vc, int layers, int slots,
                                    int row_bytes) {
  const DevDecode& d = *dp;
  if (d.mode != LA_MODE_LOOKAHEAD || d.commit_n <= 0 || d.winner < 0) return;
  const int S = d.N - 1, n = d.commit_n, owner = d.winner % d.world;
  const uint8_t* src_base = gathered + (size_t)owner * seg;
  const int per = row_bytes / 16;
  const long total = (long)layers * n * 2 * per;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    int e = (int)(idx % per) * 16;
    long t = idx / per;
    int kv = (int)(t % 2); t /= 2;
    int i = (int)(t % n) + 1;
    int l = (int)(t / n);
    size_t src = (((size_t)l * S + (i - 1)) * 2 + kv) * row_bytes + e;
    size_t dst = (size_t)l * slots * row_bytes + (size_t)(d.commit_ctx + i) * row_bytes + e;
    uint8_t* cache = kv ? vc : kc;
    *reinterpret_cast<uint4*>(cache + dst) = *reinterpret_cast<const uint4*>(src_base + src);
  }
}

LA_TL_DEFINE_SETTER(state)
