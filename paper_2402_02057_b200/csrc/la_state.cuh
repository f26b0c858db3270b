// Device-side step logic: n-gram pool, step build (K1) and step finish (K10).
//
// All functions are block-cooperative: every thread of the calling block must
// enter them (they contain __syncthreads).  They are shared by the fp32
// single-CTA decode megakernel (tiny models) and by the single-CTA step
// kernels of the bf16 multi-kernel path, so both paths run the *same*
// bookkeeping code.
#pragma once
#include "la_common.cuh"
#include "la_sample.cuh"

// ================================================================ pool
__device__ __forceinline__ uint32_t la_gram_hash(const int* g, int n) {
  uint32_t h = 0x9e3779b9u;
  for (int i = 0; i < n; ++i) h = la_mix32(h ^ (uint32_t)g[i]) + 0x85ebca6bu * (i + 1);
  return h;
}

// Lead-table probe (reference pool.py:69-81 `self._buckets.get(last)`).
__device__ __forceinline__ int la_lead_find(const DevPool& p, int lead) {
  uint32_t h = la_mix32((uint32_t)lead) & (uint32_t)p.lt_mask;
  for (int probe = 0; probe <= p.lt_mask; ++probe) {
    int k = p.lead_keys[h];
    if (k == lead) return (int)h;
    if (k < 0) return -1;
    h = (h + 1) & (uint32_t)p.lt_mask;
  }
  return -1;
}

__device__ __forceinline__ int la_lead_find_or_add(const DevPool& p, int lead) {
  uint32_t h = la_mix32((uint32_t)lead) & (uint32_t)p.lt_mask;
  for (int probe = 0; probe <= p.lt_mask; ++probe) {
    int k = p.lead_keys[h];
    if (k == lead) return (int)h;
    if (k < 0) {
      p.lead_keys[h] = lead;
      p.bkt_cnt[h] = 0;
      if (p.lead_head) p.lead_head[h] = -1;
      return (int)h;
    }
    h = (h + 1) & (uint32_t)p.lt_mask;
  }
  return -1;
}

// Bucket helpers for one warp; buckets are newest-first arrays of suffixes and
// may exceed 32 entries in capacity mode, so every pass walks 32-entry chunks.
// first index in [0, cnt) whose suffix equals `suf` (-1: none)
static __device__ int la_bucket_find(const int* B, int cnt, int S, const int* suf, int lane) {
  for (int base = 0; base < cnt; base += 32) {
    bool match = false;
    if (base + lane < cnt) {
      match = true;
      for (int s = 0; s < S; ++s) match &= (B[(base + lane) * S + s] == suf[s]);
    }
    const unsigned m = __ballot_sync(0xffffffffu, match);
    if (m) return base + __ffs(m) - 1;
  }
  return -1;
}

// entries [0, upto) move down one slot (top chunk first: no overwrite before read)
static __device__ void la_bucket_shift_down(int* B, int upto, int S, int lane) {
  int tmp[LA_MAX_SUFFIX];
  for (int base = ((upto - 1) >> 5) << 5; base >= 0 && upto > 0; base -= 32) {
    const bool mv = base + lane < upto;
    if (mv)
      for (int s = 0; s < S; ++s) tmp[s] = B[(base + lane) * S + s];
    __syncwarp();
    if (mv)
      for (int s = 0; s < S; ++s) B[(base + lane + 1) * S + s] = tmp[s];
    __syncwarp();
  }
}

// distinct-set probe in capacity mode: a live entry equal to g (returns its
// slot, *free_slot untouched) or -1 with *free_slot = the first empty or
// evicted slot on g's probe path
static __device__ int la_set_find_live(const DevPool& p, const int* g, int N, int* free_slot) {
  uint32_t h = la_gram_hash(g, N) & (uint32_t)p.st_mask;
  *free_slot = -1;
  for (int probe = 0; probe <= p.st_mask; ++probe) {
    const int* key = p.set_keys + (size_t)h * N;
    if (key[0] < 0) {
      if (*free_slot < 0) *free_slot = (int)h;
      return -1;
    }
    if (p.set_stamp[h] < 0) {
      if (*free_slot < 0) *free_slot = (int)h;
    } else {
      bool eq = true;
      for (int i = 0; i < N; ++i) eq &= (key[i] == g[i]);
      if (eq) return (int)h;
    }
    h = (h + 1) & (uint32_t)p.st_mask;
  }
  return -1;
}

// newest-first bucket update of one suffix (move to front / push front)
static __device__ void la_bucket_insert_warp(const DevPool& p, int slot, const int* suf, int lane) {
  const int S = p.ngram - 1, C = p.C;
  const int cnt = p.bkt_cnt[slot];
  int* B = p.bkt_suf + (size_t)slot * C * S;
  int sl[LA_MAX_SUFFIX];
  for (int s = 0; s < S; ++s) sl[s] = suf[s];
  const int pos = la_bucket_find(B, cnt, S, sl, lane);
  const int upto = pos >= 0 ? pos : min(cnt, C - 1);   // entries [0, upto) move down one
  la_bucket_shift_down(B, upto, S, lane);
  if (lane == 0) {
    for (int s = 0; s < S; ++s) B[s] = sl[s];
    if (pos < 0) p.bkt_cnt[slot] = min(cnt + 1, C);
  }
  __threadfence_block();
  __syncwarp();
}

// LRU-capped pool lists (capacity mode): set slot h is linked into the
// newest-first list of its lead
static __device__ void la_list_unlink(const DevPool& p, int h) {
  const int lead = la_lead_find(p, p.set_keys[(size_t)h * p.ngram]);
  if (lead < 0) return;
  const int pv = p.set_prev[h], nx = p.set_next[h];
  if (pv >= 0) p.set_next[pv] = nx; else p.lead_head[lead] = nx;
  if (nx >= 0) p.set_prev[nx] = pv;
  p.bkt_cnt[lead] -= 1;
}
static __device__ void la_list_push_front(const DevPool& p, int lead, int h) {
  const int hd = p.lead_head[lead];
  p.set_prev[h] = -1;
  p.set_next[h] = hd;
  if (hd >= 0) p.set_prev[hd] = h;
  p.lead_head[lead] = h;
  p.bkt_cnt[lead] += 1;
}

// One n-gram insert by one warp (reference pool.py:41-61): dedup on
// (lead, suffix) with recency refresh, newest-first bucket, distinct count,
// and with a capacity the globally least-recently-touched entry is evicted
// before a new one is added.  `g` may live in shared or global memory.
static __device__ void la_pool_insert_warp(const DevPool& p, const int* g, int lane, int* overflow) {
  const int N = p.ngram;
  int gl[LA_MAX_SUFFIX + 1];
#pragma unroll
  for (int i = 0; i < LA_MAX_SUFFIX + 1; ++i) gl[i] = (i < N) ? g[i] : 0;
  if (p.capacity > 0) {
    // capped pool, one thread: every live entry sits in its lead's list
    if (lane == 0) {
      int free_slot;
      int h = la_set_find_live(p, gl, N, &free_slot);
      if (h >= 0) {
        la_list_unlink(p, h);   // a refresh: re-linked at the front below
      } else {
        if (p.counters[0] >= p.capacity) {
          // _entries.popitem(last=False): the oldest FIFO record still current
          int head = p.counters[3], victim = -1;
          while (head < p.counters[2]) {
            const int v = p.fifo[head];
            const int st = p.set_stamp[v];
            ++head;
            if (st == head - 1) { victim = v; break; }
          }
          p.counters[3] = head;
          if (victim >= 0) {
            // del old_bucket[old_suffix] (pool.py:54-58); the slot becomes a tombstone
            la_list_unlink(p, victim);
            p.set_stamp[victim] = -1;
            p.counters[0] -= 1;
            la_set_find_live(p, gl, N, &free_slot);   // the victim's slot may be first on our path
          } else {
            *overflow = 1;
          }
        }
        h = free_slot;
        if (h >= 0) {
          int* key = p.set_keys + (size_t)h * N;
          for (int i = 0; i < N; ++i) key[i] = gl[i];
          p.counters[0] += 1;
        } else {
          *overflow = 1;
        }
      }
      const int stamp = p.counters[2];
      if (h >= 0 && stamp < p.log_cap) {
        p.set_stamp[h] = stamp;
        p.fifo[stamp] = h;
        p.counters[2] = stamp + 1;
      } else {
        *overflow = 1;
      }
      const int slot = la_lead_find_or_add(p, gl[0]);
      if (slot < 0) *overflow = 1;
      else if (h >= 0) la_list_push_front(p, slot, h);
      const int n = p.counters[1];
      if (n < p.log_cap) {
        for (int i = 0; i < N; ++i) p.log[(size_t)n * N + i] = gl[i];
        p.counters[1] = n + 1;
      } else {
        *overflow = 1;
      }
    }
    __threadfence_block();
    __syncwarp();
    return;
  }
  int slot = 0;
  if (lane == 0) {
    // distinct set (len(pool))
    uint32_t h = la_gram_hash(gl, N) & (uint32_t)p.st_mask;
    bool placed = false;
    for (int probe = 0; probe <= p.st_mask; ++probe) {
      int* key = p.set_keys + (size_t)h * N;
      if (key[0] < 0) {
        for (int i = 0; i < N; ++i) key[i] = gl[i];
        p.counters[0] += 1;
        placed = true;
        break;
      }
      bool eq = true;
      for (int i = 0; i < N; ++i) eq &= (key[i] == gl[i]);
      if (eq) { placed = true; break; }
      h = (h + 1) & (uint32_t)p.st_mask;
    }
    if (!placed) *overflow = 1;
    slot = la_lead_find_or_add(p, gl[0]);
    if (slot < 0) *overflow = 1;
    const int n = p.counters[1];
    if (n < p.log_cap) {
      for (int i = 0; i < N; ++i) p.log[(size_t)n * N + i] = gl[i];
      p.counters[1] = n + 1;
    } else {
      *overflow = 1;
    }
  }
  slot = __shfl_sync(0xffffffffu, slot, 0);
  __syncwarp();
  if (slot < 0) return;
  la_bucket_insert_warp(p, slot, gl + 1, lane);
}

// lookup(lead, limit) (pool.py:69-81) by ONE thread: the <= limit newest
// suffixes of lead-table slot `slot` into out[c][N-1]; returns c
static __device__ int la_pool_lookup(const DevPool& p, int slot, int limit, int* out) {
  const int S = p.ngram - 1;
  if (slot < 0 || limit <= 0) return 0;
  if (p.capacity == 0) {
    const int c = min(p.bkt_cnt[slot], limit);
    const int* B = p.bkt_suf + (size_t)slot * p.C * S;
    for (int i = 0; i < c * S; ++i) out[i] = B[i];
    return c;
  }
  int c = 0;
  for (int h = p.lead_head[slot]; h >= 0 && c < limit; h = p.set_next[h], ++c)
    for (int s = 0; s < S; ++s) out[c * S + s] = p.set_keys[(size_t)h * p.ngram + 1 + s];
  return c;
}

// Ordered insert of one step's W harvested n-grams (insert_all, pool.py:63-67)
// by the whole block, for the unbounded pool: the result equals W serial
// la_pool_insert_warp calls.  In-batch repeats are refreshes of their first
// occurrence; the distinct set and lead table take the remaining (distinct)
// n-grams concurrently (CAS-claimed slots; a half-written key never equals a
// different n-gram); log entries go to fixed positions; bucket updates --
// the only order-dependent part -- run one warp per distinct lead, in column
// order (different leads' buckets commute).
static __device__ void la_pool_insert_batch(const DevPool& p, const int* grams, int W, int* overflow) {
  __shared__ int s_new[64], s_slot[64], s_lfirst[64], s_gfirst[64];
  const int N = p.ngram, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int n0 = p.counters[1];
  if (tid < W) {
    const int j = tid;
    const int* g = grams + j * N;
    int gf = j, lf = j;
    for (int q = j - 1; q >= 0; --q) {
      const int* h = grams + q * N;
      bool eq = true;
      for (int i = 0; i < N; ++i) eq &= (h[i] == g[i]);
      if (eq) gf = q;
      if (h[0] == g[0]) lf = q;
    }
    s_gfirst[j] = gf;
    s_lfirst[j] = lf;
    int is_new = 0;
    if (gf == j) {
      // distinct set (len(pool)): claim an empty slot with CAS on key[0]
      uint32_t h = la_gram_hash(g, N) & (uint32_t)p.st_mask;
      bool placed = false;
      for (int probe = 0; probe <= p.st_mask && !placed; ++probe) {
        int* key = p.set_keys + (size_t)h * N;
        int k0 = atomicCAS(key, -1, g[0]);
        if (k0 == -1) {
          for (int i = 1; i < N; ++i) key[i] = g[i];
          is_new = 1;
          placed = true;
        } else {
          bool eq = (k0 == g[0]);
          for (int i = 1; i < N && eq; ++i) eq &= (((volatile int*)key)[i] == g[i]);
          if (eq) placed = true;
          else h = (h + 1) & (uint32_t)p.st_mask;
        }
      }
      if (!placed) *overflow = 1;
    }
    s_new[j] = is_new;
    // lead table: claim or find with CAS (bucket counts start at 0)
    int slot = -1;
    if (lf == j) {
      uint32_t h = la_mix32((uint32_t)g[0]) & (uint32_t)p.lt_mask;
      for (int probe = 0; probe <= p.lt_mask; ++probe) {
        const int k = atomicCAS(p.lead_keys + h, -1, g[0]);
        if (k == -1 || k == g[0]) { slot = (int)h; break; }
        h = (h + 1) & (uint32_t)p.lt_mask;
      }
      if (slot < 0) *overflow = 1;
    }
    s_slot[j] = slot;
    if (n0 + j < p.log_cap) {
      for (int i = 0; i < N; ++i) p.log[(size_t)(n0 + j) * N + i] = g[i];
    } else {
      *overflow = 1;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int added = 0;
    for (int j = 0; j < W; ++j) added += s_new[j];
    p.counters[0] += added;
    p.counters[1] = min(n0 + W, p.log_cap);
  }
  // bucket updates: warp w serves the distinct leads w, w + nw, ... (first-occurrence order)
  int q = 0;
  for (int j = 0; j < W; ++j) {
    if (s_lfirst[j] != j) continue;
    if (q++ % nw != warp) continue;
    const int slot = s_slot[j];
    if (slot < 0) continue;
    for (int jj = j; jj < W; ++jj)
      if (s_lfirst[jj] == j) la_bucket_insert_warp(p, slot, grams + jj * N + 1, lane);
  }
  __syncthreads();
}

// ================================================= window geometry (A.1)
__device__ __forceinline__ int la_cell_index(int level, int col, int W) {
  return level == 0 ? col - 2 : (W - 1) + (level - 1) * W + (col - 1);
}
__device__ __forceinline__ void la_cell_level_col(int f, int W, int& level, int& col) {
  if (f < W - 1) { level = 0; col = f + 2; return; }
  int f2 = f - (W - 1);
  level = 1 + f2 / W;
  col = 1 + f2 % W;
}

// Global row -> (rel_pos, chain of global rows in rel order).
// Reference build_layout (layout.py:128-182), closed form of appendix A.1.
__device__ __forceinline__ int la_row_chain(int g, int W, int N, int* chain_out) {
  const int nwin = (N - 1) * W;    // q0 + window cells
  if (g == 0) return 0;
  if (g < nwin) {
    int level, col;
    la_cell_level_col(g - 1, W, level, col);
    if (level == 0) {               // q0 + level-0 cells left of col: rows 0..col-2
      for (int r = 0; r < col - 1; ++r) chain_out[r] = r;
      return col - 1;
    }
    int n = 0;
    for (int r = 0; r < col; ++r) chain_out[n++] = r;          // rel 0..col-1
    for (int m = 1; m < level; ++m) chain_out[n++] = la_cell_index(m, col, W) + 1;
    return n;                                                   // = col + level - 1
  }
  int b = (g - nwin) / (N - 1);
  int k = (g - nwin) % (N - 1) + 1;
  int base = nwin + b * (N - 1);
  chain_out[0] = 0;
  for (int r = 1; r < k; ++r) chain_out[r] = base + r - 1;
  return k;
}

__device__ __forceinline__ int la_row_token(const DevDecode& d, int g) {
  const int W = d.W, N = d.N, nwin = (N - 1) * W;
  if (g == 0) return d.last;
  if (g < nwin) return d.window[g - 1];
  int b = (g - nwin) / (N - 1);
  int k = (g - nwin) % (N - 1);
  return d.cand[b * (N - 1) + k];
}

// Lookahead parallelism: does rank `rank` of `world` evaluate global row g,
// and does it own the row's output?  Reference parallel.py:64-116.
__device__ __forceinline__ void la_lp_row_role(int g, int W, int N, int rank, int world,
                                               bool& compute, bool& own) {
  if (world <= 1) { compute = true; own = true; return; }
  const int nwin = (N - 1) * W;
  int base = W / world, extra = W % world;
  int c0 = 1 + rank * base + min(rank, extra);
  int c1 = c0 + base + (rank < extra ? 1 : 0) - 1;
  if (g == 0) { compute = true; own = (rank == 0); return; }
  if (g < nwin) {
    int level, col;
    la_cell_level_col(g - 1, W, level, col);
    bool in_range = (col >= c0 && col <= c1);
    own = in_range;
    compute = in_range || (level == 0 && col < c0);
    return;
  }
  int b = (g - nwin) / (N - 1);
  own = compute = (b % world) == rank;
}

// ====================================================== K1: step build
// prepare_step (decoding.py:152-157): pool lookup + layout rows.
static __device__ void la_step_build(DevDecode& d, FwdPlan& P) {
  __shared__ int s_c, s_slot, s_done, s_n;
  const int tid = threadIdx.x, nth = blockDim.x;
  if (tid == 0) {
    s_done = d.done;
    s_slot = -1;
    s_c = 0;
    if (!s_done && d.mode == LA_MODE_LOOKAHEAD && d.G > 0) {
      const int slot = la_lead_find(d.pool, d.last);
      s_slot = slot;
      s_c = la_pool_lookup(d.pool, slot, d.G, d.cand);
    }
  }
  __syncthreads();
  if (s_done) {
    if (tid == 0) P.n_rows = 0;
    __syncthreads();
    return;
  }
  const int W = d.W, N = d.N, S = N - 1, c = s_c;
  if (d.mode == LA_MODE_AUTOREGRESSIVE) {
    if (tid == 0) {
      P.n_rows = 1; P.n_pad = 16; P.n_prefix = d.ctx; P.n_global = 1;
      P.ids[0] = d.last; P.pos[0] = d.ctx; P.slot[0] = d.ctx; P.grow[0] = 0;
      P.own[0] = 1; P.chain_n[0] = 0;
      d.amax[0] = -1;
      d.c = 0; d.M = 1;
    }
    __syncthreads();
    return;
  }
  if (tid == 0) { d.c = c; d.M = S * (W + c); s_n = 0; }
  __syncthreads();
  const int M = S * (W + c);
  // rows this rank computes, in ascending global order (serial scan: M <= 128)
  if (tid == 0) {
    int n = 0;
    for (int g = 0; g < M; ++g) {
      bool comp, own;
      la_lp_row_role(g, W, N, d.rank, d.world, comp, own);
      if (comp) { P.grow[n] = g; P.own[n] = own ? 1 : 0; ++n; }
    }
    s_n = n;
    P.n_rows = n;
    P.n_pad = la_round16(n);
    P.n_prefix = d.ctx;
    P.n_global = M;
  }
  for (int g = tid; g < LA_MAX_ROWS; g += nth) d.amax[g] = -1;
  __syncthreads();
  for (int m = tid; m < s_n; m += nth) {
    int g = P.grow[m];
    int ch[LA_MAX_CHAIN];
    int n = la_row_chain(g, W, N, ch);
    P.ids[m] = la_row_token(d, g);
    P.pos[m] = d.ctx + n;          // absolute position = len(prefix) + rel_pos
    P.slot[m] = d.ctx + g;         // step K/V scratch right after the prefix
    P.chain_n[m] = n;
    for (int j = 0; j < n; ++j) P.chain[m][j] = d.ctx + ch[j];
  }
  __syncthreads();
}

// ===================================================== K10: step finish
// finish_step (decoding.py:160-204) + collect_output (:214-232):
// verify_greedy, n-gram harvest + ordered pool insert, window shift with
// RNG refills, output folding, StepRecord.  Requires d.amax[] for every
// generator row, row 0 and every branch row.
static __device__ void la_step_finish(DevDecode& d) {
  __shared__ int s_done, s_k;
  __shared__ int s_newtop[64];
  __shared__ int s_grams[64 * (LA_MAX_SUFFIX + 1)];
  __shared__ int s_oldwin[64 * LA_MAX_SUFFIX];
  __shared__ int s_acc[LA_MAX_SUFFIX + 2];
  const int tid = threadIdx.x, nth = blockDim.x;
  if (tid == 0) {
    s_done = d.done;
    if (!s_done && d.degenerate) s_done = d.done = 1;   // host raises DegenerateDistributionError
  }
  __syncthreads();
  if (s_done) return;
  const int W = d.W, N = d.N, S = N - 1;
  if (d.mode == LA_MODE_AUTOREGRESSIVE) {
    // decode_autoregressive (decoding.py:96-116): argmax, or sample_token's
    // draw made by la_verify_sample (sampling.py:77-85)
    if (tid == 0) {
      int t = d.sample ? d.accepted[0] : d.amax[0];
      d.out[d.n_out] = t;
      d.n_out += 1;
      d.ctx += 1;           // q0's K/V already sit at slot ctx
      d.last = t;
      d.n_steps += 1;
      if ((d.eos >= 0 && t == d.eos) || d.n_out >= d.max_tokens || d.n_steps >= d.max_steps)
        d.done = 1;
    }
    __syncthreads();
    return;
  }
  const int c = d.c, nwin = S * W, ncell = S * W - 1;
  for (int j = tid; j < W; j += nth) s_newtop[j] = d.amax[(N - 2) * W + j];
  for (int f = tid; f < ncell; f += nth) s_oldwin[f] = d.window[f];
  __syncthreads();
  if (tid == 0) {
    // verify_greedy (verification.py:43-71) on argmax ids; under a
    // temperature sampler la_verify_sample already ran verify_sample
    int k = 0, win = -1;
    if (d.sample) {
      k = d.k;
      win = d.winner;
      for (int i = 0; i < k; ++i) s_acc[i] = d.accepted[i];
    } else if (c == 0) {
      s_acc[k++] = d.amax[0];
    } else {
      unsigned long long alive = (c >= 64) ? ~0ull : ((1ull << c) - 1ull);
      bool all = true;
      for (int i = 0; i < S; ++i) {
        int lead = __ffsll((long long)alive) - 1;
        int row = (i == 0) ? 0 : nwin + lead * S + i - 1;
        int target = d.amax[row];
        unsigned long long keep = 0;
        for (int b = 0; b < c; ++b)
          if (((alive >> b) & 1ull) && d.cand[b * S + i] == target) keep |= 1ull << b;
        s_acc[k++] = target;
        if (!keep) { all = false; break; }
        alive = keep;
      }
      if (all) {
        win = __ffsll((long long)alive) - 1;
        s_acc[k++] = d.amax[nwin + win * S + S - 1];
      } else if (k >= 2) {
        win = __ffsll((long long)alive) - 1;   // survivors of the accepted prefix
      }
    }
    s_k = k;
    d.k = k;
    d.winner = win;
    d.commit_ctx = d.ctx;
    d.commit_n = k - 1;
    d.commit_base = (win >= 0) ? nwin + win * S : 0;
  }
  // n-gram harvest from the OLD window (layout.py:197-216)
  for (int j = tid; j < W; j += nth) {
    int col = j + 1;
    int* gr = s_grams + j * N;
    gr[0] = (col == 1) ? d.last : s_oldwin[la_cell_index(0, col, W)];
    for (int l = 1; l < N - 1; ++l) gr[l] = s_oldwin[la_cell_index(l, col, W)];
    gr[N - 1] = s_newtop[j];
  }
  __syncthreads();
  // ordered pool insert (pool.py:63-67), column order: block-parallel for the
  // unbounded pool, one warp serially under an LRU cap (evictions are global)
  if (d.pool.capacity == 0) {
    la_pool_insert_batch(d.pool, s_grams, W, &d.overflow);
  } else if (tid < 32) {
    for (int j = 0; j < W; ++j) la_pool_insert_warp(d.pool, s_grams + j * N, tid, &d.overflow);
  }
  // window update (layout.py:219-252) with refills from the RNG stream
  const int sft = s_k - 1;
  const int v0 = min(sft, W - 1), v1 = min(sft, W);
  const int cur = d.rng_cur;
  for (int f = tid; f < ncell; f += nth) {
    int level, col;
    la_cell_level_col(f, W, level, col);
    int sc = col + sft;
    int val;
    if (sc <= W) {
      val = (level + 1 <= N - 2) ? s_oldwin[la_cell_index(level + 1, sc, W)] : s_newtop[sc - 1];
    } else if (d.sample || d.pcg_window) {
      continue;   // drawn below, in cell order, from the session generator
    } else {
      int idx = (level == 0) ? (col - max(2, W - sft + 1))
                             : v0 + (level - 1) * v1 + (col - max(1, W - sft + 1));
      int r = cur + idx;
      val = (r < d.rng_len) ? d.rng[r] : 0;
      if (r >= d.rng_len) d.overflow = 1;
    }
    d.window[f] = val;
  }
  if ((d.sample || d.pcg_window) && tid == 0 && sft > 0) {
    // rng.integers(0, V) per vacated cell, level-major / column-ascending
    // (layout.py:243-250) -- f order is exactly that order
    LaPcg64 g = d.pcg;
    for (int f = 0; f < ncell; ++f) {
      int level, col;
      la_cell_level_col(f, W, level, col);
      if (col + sft > W) d.window[f] = la_pcg_integers(g, (unsigned)d.V);
    }
    d.pcg = g;
  }
  __syncthreads();
  if (tid == 0) {
    const int k = s_k;
    d.rng_cur = cur + v0 + (N - 2) * v1;
    // collect_output: fold accepted tokens, stop at EOS / budget
    bool stop = false;
    for (int i = 0; i < k && !stop; ++i) {
      int t = s_acc[i];
      d.out[d.n_out] = t;
      d.n_out += 1;
      if (d.eos >= 0 && t == d.eos) stop = true;
      else if (d.n_out >= d.max_tokens) stop = true;
    }
    for (int i = 0; i < k; ++i) d.accepted[i] = s_acc[i];
    int st = d.n_steps;
    if (st < d.max_steps) {
      d.rec[st * 4 + 0] = k;
      d.rec[st * 4 + 1] = c;
      d.rec[st * 4 + 2] = d.M;
      d.rec[st * 4 + 3] = d.pool.counters[0];
    }
    d.n_steps = st + 1;
    d.ctx += k;
    d.last = s_acc[k - 1];
    if (stop || d.n_steps >= d.max_steps) d.done = 1;
  }
  __syncthreads();
}
