// Temperature sampling + distribution-preserving verification on the device.
//
// Restates (paths relative to /root/reference/pkg/src/lookahead):
//   la_adjust_row      adjusted_distribution, sampling.py:22-66
//   la_draw            draw (inverse CDF, searchsorted 'right'), sampling.py:69-74
//   la_verify_sample   verify_sample, verification.py:74-118
// and numpy's PCG64 Generator stream (random(): 53-bit double; integers(0, V):
// 32-bit Lemire rejection on next_uint32, which hands out the buffered upper
// half of a 64-bit draw on every second call) so that a session seeded like
// the reference consumes the identical random stream.
//
// Every function below except the PCG64 scalar ones is block-cooperative:
// all threads of the block must enter (blockDim.x a multiple of 32, <= 1024).
// Distributions are fp64 [V] arrays in global memory.  Reductions and scans
// run in a fixed order (per-thread contiguous chunks, warp trees, warps in
// order), so results do not depend on scheduling; the top-p mass histogram
// uses 2^-60 fixed point with integer atomics for the same reason.
#pragma once
#include "la_common.cuh"

// ------------------------------------------------------------------ PCG64
__host__ __device__ __forceinline__ unsigned long long la_mulhi64(unsigned long long a,
                                                                  unsigned long long b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (unsigned long long)(((unsigned __int128)a * b) >> 64);
#endif
}

// state = state * PCG_DEFAULT_MULTIPLIER_128 + inc; XSL-RR of the new state
__host__ __device__ __forceinline__ unsigned long long la_pcg_next64(LaPcg64& g) {
  const unsigned long long mhi = 0x2360ED051FC65DA4ull, mlo = 0x4385DF649FCCF645ull;
  const unsigned long long lo = g.s_lo * mlo;
  unsigned long long hi = la_mulhi64(g.s_lo, mlo) + g.s_lo * mhi + g.s_hi * mlo;
  const unsigned long long nlo = lo + g.i_lo;
  hi += g.i_hi + (nlo < lo ? 1ull : 0ull);
  g.s_lo = nlo;
  g.s_hi = hi;
  const unsigned long long x = hi ^ nlo;
  const unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__host__ __device__ __forceinline__ unsigned la_pcg_next32(LaPcg64& g) {
  if (g.has32) {
    g.has32 = 0;
    return g.u32;
  }
  const unsigned long long v = la_pcg_next64(g);
  g.has32 = 1;
  g.u32 = (unsigned)(v >> 32);
  return (unsigned)v;
}

// Generator.random()
__host__ __device__ __forceinline__ double la_pcg_random(LaPcg64& g) {
  return (double)(la_pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// Generator.integers(0, high), 1 <= high < 2^32 (buffered_bounded_lemire_uint32)
__host__ __device__ __forceinline__ int la_pcg_integers(LaPcg64& g, unsigned high) {
  const unsigned rng = high - 1u;
  if (rng == 0u) return 0;
  const unsigned excl = rng + 1u;
  unsigned long long m = (unsigned long long)la_pcg_next32(g) * excl;
  unsigned left = (unsigned)m;
  if (left < excl) {
    const unsigned thr = (0xFFFFFFFFu - rng) % excl;
    while (left < thr) {
      m = (unsigned long long)la_pcg_next32(g) * excl;
      left = (unsigned)m;
    }
  }
  return (int)(m >> 32);
}

#ifdef __CUDACC__
// ------------------------------------------------------- block primitives
struct LaSampleSmem {
  unsigned long long hist[32][16];   // per-warp radix histograms (4-bit digits)
  unsigned long long tot[16];
  unsigned long long xt[2][16];      // cluster scope: published histograms (double-buffered)
  double xd[2];                      // cluster scope: published partials (double-buffered)
  long long xl[2];
  double red[32];
  unsigned long long ured[32];
  int ired[32];
  double u;
  unsigned long long sel_acc;
  int sel;
  int idx;
  int flag;
};

__device__ __forceinline__ double la_bsum_d(double v, LaSampleSmem& sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm.red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += sm.red[i];
  return t;
}

__device__ __forceinline__ float la_bmax_f(float v, LaSampleSmem& sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm.red[w] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int i = 0; i < nw; ++i) t = fmaxf(t, (float)sm.red[i]);
  return t;
}

// exclusive prefix (thread order) of one double per thread; *total = sum
__device__ __forceinline__ double la_bscan_d(double v, LaSampleSmem& sm, double* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  __syncthreads();
  if (lane == 31) sm.red[w] = inc;
  __syncthreads();
  double base = 0.0, t = 0.0;
  for (int i = 0; i < nw; ++i) {
    if (i == w) base = t;
    t += sm.red[i];
  }
  *total = t;
  return base + inc - v;
}

__device__ __forceinline__ int la_bscan_i(int v, LaSampleSmem& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  __syncthreads();
  if (lane == 31) sm.ired[w] = inc;
  __syncthreads();
  int base = 0;
  for (int i = 0; i < w; ++i) base += sm.ired[i];
  return base + inc - v;
}

// Reduction scopes of the row functions below.  A row is processed by one
// CTA (LaBlockScope: the fp32 single-CTA decode, parity hooks) or by the CTAs
// of a thread-block cluster, each owning a contiguous slice of the vocabulary
// (LaClusterScope: the bf16 path's adjust kernel).  Cluster partials are
// exchanged through distributed shared memory and combined in rank order, so
// results are deterministic; every call is collective over the scope.
struct LaBlockScope {
  int lo, hi;   // [0, V)
  __device__ double sum(double v, LaSampleSmem&) { return v; }
  __device__ float max(float v, LaSampleSmem&) { return v; }
  __device__ void combine16(LaSampleSmem&) {}
  __device__ long long prefix(long long, LaSampleSmem&) { return 0; }
  __device__ void finish() {}
};

#if defined(__CUDACC__)
__device__ __forceinline__ void la_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <typename T>
__device__ __forceinline__ T la_dsmem_ld(const T* local, unsigned rank) {
  // address of `local`'s counterpart in CTA `rank` of the cluster
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  T v;
  if constexpr (sizeof(T) == 8) {
    unsigned long long u;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(u) : "r"(r) : "memory");
    memcpy(&v, &u, 8);
  } else {
    unsigned u;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(u) : "r"(r) : "memory");
    memcpy(&v, &u, 4);
  }
  return v;
}

struct LaClusterScope {
  int lo, hi;             // this CTA's slice
  unsigned rank, size;
  int ph = 0;             // exchange parity: a slot is rewritten only two exchanges
                          // later, after an intervening barrier every CTA has passed
  __device__ double sum(double v, LaSampleSmem& sm) {
    const int b = ph; ph ^= 1;
    if (threadIdx.x == 0) sm.xd[b] = v;
    la_cluster_sync();
    double t = 0.0;
    for (unsigned r = 0; r < size; ++r) t += la_dsmem_ld(&sm.xd[b], r);
    return t;
  }
  __device__ float max(float v, LaSampleSmem& sm) {
    const int b = ph; ph ^= 1;
    if (threadIdx.x == 0) sm.xd[b] = (double)v;
    la_cluster_sync();
    float t = -INFINITY;
    for (unsigned r = 0; r < size; ++r) t = fmaxf(t, (float)la_dsmem_ld(&sm.xd[b], r));
    return t;
  }
  // sm.tot[16] (this CTA) -> sm.tot[16] (whole cluster)
  __device__ void combine16(LaSampleSmem& sm) {
    const int b = ph; ph ^= 1;
    if (threadIdx.x < 16) sm.xt[b][threadIdx.x] = sm.tot[threadIdx.x];
    la_cluster_sync();
    if (threadIdx.x < 16) {
      unsigned long long t = 0ull;
      for (unsigned r = 0; r < size; ++r) t += la_dsmem_ld(&sm.xt[b][threadIdx.x], r);
      sm.tot[threadIdx.x] = t;
    }
    __syncthreads();
  }
  // exclusive prefix over the cluster's ranks of a per-CTA value
  __device__ long long prefix(long long v, LaSampleSmem& sm) {
    const int b = ph; ph ^= 1;
    if (threadIdx.x == 0) sm.xl[b] = v;
    la_cluster_sync();
    long long t = 0;
    for (unsigned r = 0; r < rank; ++r) t += la_dsmem_ld(&sm.xl[b], r);
    return t;
  }
  // before the CTA may exit: no peer still reads this CTA's slots
  __device__ void finish() { la_cluster_sync(); }
};
#endif

__device__ __forceinline__ unsigned long long la_pbits(double p) {
  return (unsigned long long)__double_as_longlong(p);   // p >= 0: order preserving
}

// Radix select over the order (-p, id) restricted to values: finds the value
// key T with  weight(p > T) < need <= weight(p >= T), weight = 1 per element
// (mass == false) or floor(p * scale) (mass == true).  Returns false when the
// total weight stays below `need`.  *above = weight(p > T).  4-bit digits
// counted in per-thread registers and reduced by warp shuffles: near-uniform
// distributions put almost every element in the same top digits, where
// shared-memory atomics would serialise the CTA on one address.
template <typename Scope>
static __device__ bool la_radix_select(const double* p, Scope& sc, bool mass, double scale,
                                unsigned long long need, LaSampleSmem& sm,
                                unsigned long long* T, unsigned long long* above) {
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, w = tid >> 5;
  const int V = sc.hi;
  const int nw = nth >> 5;
  unsigned long long prefix = 0ull, mask = 0ull, acc_above = 0ull;
  for (int shift = 60; shift >= 0; shift -= 4) {
    unsigned long long loc[16];
#pragma unroll
    for (int d = 0; d < 16; ++d) loc[d] = 0ull;
    for (int i0 = sc.lo + tid; i0 < V; i0 += 8 * nth) {
      double vb[8];   // 8 loads in flight per thread (the pass is L2-latency bound)
#pragma unroll
      for (int u = 0; u < 8; ++u) vb[u] = (i0 + u * nth < V) ? p[i0 + u * nth] : -1.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double v = vb[u];
        const unsigned long long b = la_pbits(v);
        if (v >= 0.0 && (b & mask) == prefix) {
          const unsigned long long wgt = mass ? (unsigned long long)(v * scale) : 1ull;
          const int dg = (int)((b >> shift) & 15ull);
#pragma unroll
          for (int d = 0; d < 16; ++d) loc[d] += (dg == d) ? wgt : 0ull;
        }
      }
    }
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      unsigned long long v = loc[d];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      loc[d] = v;
    }
    if (lane == 0) {
#pragma unroll
      for (int d = 0; d < 16; ++d) sm.hist[w][d] = loc[d];
    }
    __syncthreads();
    if (tid < 16) {
      unsigned long long t = 0ull;
      for (int j = 0; j < nw; ++j) t += sm.hist[j][tid];
      sm.tot[tid] = t;
    }
    __syncthreads();
    sc.combine16(sm);
    if (tid == 0) {
      unsigned long long acc = acc_above;
      int sel = -1;
      for (int dg = 15; dg >= 0; --dg) {
        if (acc + sm.tot[dg] >= need) { sel = dg; break; }
        acc += sm.tot[dg];
      }
      sm.sel = sel;
      sm.sel_acc = acc;
    }
    __syncthreads();
    const int sel = sm.sel;
    if (sel < 0) return false;
    acc_above = sm.sel_acc;
    prefix |= (unsigned long long)sel << shift;
    mask |= 15ull << shift;
  }
  *T = prefix;
  *above = acc_above;
  return true;
}

// keep p[i] with value key > T, and the first `m` (lowest ids) with key == T;
// zero the rest (the (-p, id) order prefix of lexsort, sampling.py:43)
template <typename Scope>
static __device__ void la_keep_prefix(double* p, Scope& sc, unsigned long long T, long long m,
                               LaSampleSmem& sm) {
  const int n = sc.hi - sc.lo;
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int lo = sc.lo + min(n, (int)threadIdx.x * chunk), hi = min(sc.hi, lo + chunk);
  int ties = 0;
  for (int i = lo; i < hi; ++i) ties += la_pbits(p[i]) == T;
  long long r = la_bscan_i(ties, sm);
  r += sc.prefix((long long)la_bsum_d((double)ties, sm), sm);   // ties in lower-ranked slices
  for (int i = lo; i < hi; ++i) {
    const unsigned long long b = la_pbits(p[i]);
    bool keep = b > T;
    if (b == T) keep = (r++ < m);
    if (!keep) p[i] = 0.0;
  }
  __syncthreads();
}

// adjusted_distribution(softmax(logits), spec) into out[V] (sampling.py:22-66;
// the model's probabilities are exp(l - max) / sum, models.py:268-271).
// lg == nullptr: out[] already holds the probabilities.  Returns false
// (DegenerateDistributionError) when all mass is truncated.
template <typename Scope>
static __device__ bool la_adjust_row_s(const float* lg, Scope& sc, int V, double temperature,
                                       int top_k, double top_p, double* out, LaSampleSmem& sm) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lo = sc.lo, hi = sc.hi;
  double Z = 1.0;
  if (lg) {
    float mx = -INFINITY;
    for (int i = lo + tid; i < hi; i += nth) mx = fmaxf(mx, lg[i]);
    mx = sc.max(la_bmax_f(mx, sm), sm);
    double s = 0.0;
    for (int i = lo + tid; i < hi; i += nth) {
      const double e = exp((double)lg[i] - (double)mx);
      out[i] = e;
      s += e;
    }
    Z = sc.sum(la_bsum_d(s, sm), sm);
  }
  const bool powr = temperature != 1.0;
  const double inv = 1.0 / temperature;
  for (int i = lo + tid; i < hi; i += nth) {
    double p = lg ? out[i] / Z : out[i];
    if (powr) p = pow(p, inv);
    out[i] = p;
  }
  __syncthreads();
  unsigned long long T, above;
  if (top_k > 0 && top_k < V) {
    if (la_radix_select(out, sc, false, 0.0, (unsigned long long)top_k, sm, &T, &above))
      la_keep_prefix(out, sc, T, (long long)top_k - (long long)above, sm);
  }
  if (top_p < 1.0) {
    double t = 0.0;
    for (int i = lo + tid; i < hi; i += nth) t += out[i];
    t = sc.sum(la_bsum_d(t, sm), sm);
    if (!(t > 0.0)) return false;
    const double one = 1152921504606846976.0;   // 2^60: the total's fixed-point weight
    const double scale = one / t;
    const unsigned long long need = (unsigned long long)ceil(top_p * one);
    if (need > 0 && la_radix_select(out, sc, true, scale, need, sm, &T, &above)) {
      const unsigned long long f = (unsigned long long)(__longlong_as_double((long long)T) * scale);
      long long m = f ? (long long)((need - above + f - 1) / f) : 1;
      la_keep_prefix(out, sc, T, m < 1 ? 1 : m, sm);
    }
  }
  double t = 0.0;
  for (int i = lo + tid; i < hi; i += nth) t += out[i];
  t = sc.sum(la_bsum_d(t, sm), sm);
  if (!(t > 0.0)) return false;
  for (int i = lo + tid; i < hi; i += nth) out[i] = out[i] / t;
  __syncthreads();
  return true;
}

static __device__ bool la_adjust_row(const float* lg, int V, double temperature, int top_k, double top_p,
                                     double* out, LaSampleSmem& sm) {
  LaBlockScope sc{0, V};
  return la_adjust_row_s(lg, sc, V, temperature, top_k, top_p, out, sm);
}

// draw(p, rng): u = random(); first i with cumsum(p)[i] > u * cumsum(p)[-1]
// (searchsorted right), clamped to V - 1.  Thread 0 owns the generator.
static __device__ int la_draw(const double* p, int V, LaPcg64& g, LaSampleSmem& sm) {
  const int tid = threadIdx.x;
  if (tid == 0) { sm.u = la_pcg_random(g); sm.idx = V; }
  const int chunk = (V + blockDim.x - 1) / blockDim.x;
  const int lo = min(V, tid * chunk), hi = min(V, lo + chunk);
  double loc = 0.0;
  for (int i = lo; i < hi; ++i) loc += p[i];
  double total;
  double c = la_bscan_d(loc, sm, &total);   // its barriers publish sm.u / sm.idx
  const double tgt = sm.u * total;
  for (int i = lo; i < hi; ++i) {
    c += p[i];
    if (c > tgt) { atomicMin(&sm.idx, i); break; }
  }
  __syncthreads();
  const int r = min(sm.idx, V - 1);
  __syncthreads();
  return r;
}

// verify_sample (verification.py:74-118) on this step's adjusted rows:
// adj row 0 = base, branch b offset k = 1 + b*S + k - 1.  Writes d.accepted,
// d.k, d.winner (first surviving branch whose K/V rows are committed).
// Returns false on DegenerateDistributionError.
static __device__ bool la_verify_sample(DevDecode& d, LaSampleSmem& sm) {
  __shared__ int s_alive[64], s_na, s_out[LA_MAX_SUFFIX + 2], s_k, s_win, s_acc;
  __shared__ LaPcg64 s_g;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int V = d.V, S = d.N - 1;
  const int c = d.mode == LA_MODE_LOOKAHEAD ? d.c : 0;
  if (tid == 0) {
    s_g = d.pcg;
    s_na = c;
    for (int b = 0; b < c; ++b) s_alive[b] = b;
    s_k = 0;
    s_win = -1;
  }
  __syncthreads();
  bool ok = true;
  if (c == 0) {
    const int t = la_draw(d.adj, V, s_g, sm);
    if (tid == 0) { s_out[0] = t; s_k = 1; }
  } else {
    bool all = true;
    for (int i = 0; i < S && ok; ++i) {
      const double* src = d.adj + (size_t)(i == 0 ? 0 : 1 + s_alive[0] * S + i - 1) * V;
      for (int v = tid; v < V; v += nth) d.work[v] = src[v];
      __syncthreads();
      bool accepted = false;
      for (int j = 0; j < s_na; ++j) {
        const int tok = d.cand[s_alive[j] * S + i];
        if (tid == 0) {
          const double r = la_pcg_random(s_g);
          const double ps = d.work[tok];
          s_acc = (ps > 0.0 && r <= ps);
        }
        __syncthreads();
        if (s_acc) {
          if (tid == 0) {
            s_out[s_k++] = tok;
            int n = 0;
            for (int b = j; b < s_na; ++b)
              if (d.cand[s_alive[b] * S + i] == tok) s_alive[n++] = s_alive[b];
            s_na = n;
          }
          accepted = true;
          __syncthreads();
          break;
        }
        if (tid == 0) d.work[tok] = 0.0;
        __syncthreads();
        double t = 0.0;
        for (int v = tid; v < V; v += nth) t += d.work[v];
        t = la_bsum_d(t, sm);
        if (!(t > 0.0)) { ok = false; break; }
        for (int v = tid; v < V; v += nth) d.work[v] = d.work[v] / t;
        __syncthreads();
      }
      if (!ok) break;
      if (!accepted) {
        const int t = la_draw(d.work, V, s_g, sm);
        if (tid == 0) {
          s_out[s_k++] = t;
          s_win = i > 0 ? s_alive[0] : -1;
        }
        all = false;
        __syncthreads();
        break;
      }
    }
    if (ok && all) {
      const int t = la_draw(d.adj + (size_t)(1 + s_alive[0] * S + S - 1) * V, V, s_g, sm);
      if (tid == 0) { s_out[s_k++] = t; s_win = s_alive[0]; }
    }
  }
  __syncthreads();
  if (tid == 0) {
    d.pcg = s_g;
    if (ok) {
      for (int i = 0; i < s_k; ++i) d.accepted[i] = s_out[i];
      d.k = s_k;
      d.winner = s_win;
    } else {
      d.degenerate = 1;
    }
  }
  __syncthreads();
  return ok;
}

// Rows whose adjusted distribution verification may read: row 0 and every
// branch row (decoding.py:181-185 adjusts exactly these).  j -> global row.
__device__ __forceinline__ int la_sample_row(const DevDecode& d, int j) {
  return j == 0 ? 0 : (d.N - 1) * d.W + (j - 1);
}
__device__ __forceinline__ int la_sample_rows(const DevDecode& d) {
  return d.mode == LA_MODE_LOOKAHEAD ? 1 + d.c * (d.N - 1) : 1;
}
#endif  // __CUDACC__
