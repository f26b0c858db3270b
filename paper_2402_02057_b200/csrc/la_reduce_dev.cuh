// Device helpers shared by the split-K reduce / epilogue kernels
// (la_reduce.cu) and the fused attention kernel (la_attn_fused.cu).
#pragma once
#include <cuda_bf16.h>

#include "la_gemm.cuh"
#include "la_reduce.cuh"

constexpr int kMaxSegUnroll = 10;   // ~the piece count of the narrow projections (O / down)

// sum over segments of 4 consecutive features (f4 = f/4) of token tok, tile t
static __device__ __forceinline__ float4 seg_sum4(const float* ws, int t, int max_segs, int nseg, int tok,
                                           int f) {
  const float4* p = reinterpret_cast<const float4*>(ws + ((size_t)t * max_segs * 128 + tok) * 128 + f);
  constexpr size_t stride = 128 * 128 / 4;
  float4 v[kMaxSegUnroll];
#pragma unroll
  for (int s = 0; s < kMaxSegUnroll; ++s)
    if (s < nseg) v[s] = __ldcg(p + s * stride);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int s = 0; s < kMaxSegUnroll; ++s)
    if (s < nseg) { acc.x += v[s].x; acc.y += v[s].y; acc.z += v[s].z; acc.w += v[s].w; }
  for (int s = kMaxSegUnroll; s < nseg; ++s) {   // rare: very narrow GEMMs
    float4 w = __ldcg(p + s * stride);
    acc.x += w.x; acc.y += w.y; acc.z += w.z; acc.w += w.w;
  }
  return acc;
}

// Entry of an epilogue kernel.  With per-tile readiness (ready != null) the
// CTA polls its tile's piece counter instead of waiting for the whole GEMM
// grid: the counter only grows (every contributor adds 1 per launch, also
// when a launch has no rows), and this CTA's own launch count -- a slot only
// it writes -- gives the target.  Every GEMM CTA passed its own dependency
// wait before counting in, so everything before the GEMM is complete and
// visible once the counter is reached (acquire), as after a grid wait.
static __device__ __forceinline__ void la_epi_enter(const int* ready, int* runs, const LaSplit& sp, int tile,
                                                    const LaPrefetch& pf) {
  la_pdl_trigger();
  if (!ready) {
    la_l2_prefetch_gemm(pf);
    la_pdl_wait();
    return;
  }
  if (threadIdx.x == 0) {
    const int slot = blockIdx.y * gridDim.x + blockIdx.x;
    const int r = runs[slot] + 1;
    runs[slot] = r;
    long c0;
    int n;
    la_tile_segs(tile, sp.kb, sp.n_tiles, sp.grid, c0, n, sp.tpc);
    const int target = r * n;
    const int* cnt = ready + tile / sp.tpc;
    int v;
    for (unsigned n = 0;; ++n) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
      if (v - target >= 0) break;
      // a GEMM / epilogue pair out of lockstep would wait forever: fail the
      // launch instead (seconds; a normal wait is microseconds)
      if (n > (1u << 26)) __trap();
      __nanosleep(64);
    }
    la_tl_stamp();
  }
  __syncthreads();
}

static __device__ __forceinline__ int tile_nseg(const LaSplit& sp, int t) {
  long c0;
  int n;
  la_tile_segs(t, sp.kb, sp.n_tiles, sp.grid, c0, n, sp.tpc);
  return n;
}

static __device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Single-round-trip variants: every load of the pieces (and of the norm
// statistics) is issued before the first use, so a kernel pays one L2 latency.
// (kSegBatch loads per group in flight: ~the piece count of the wide
// projections; more would cost registers and occupancy)
constexpr int kSegBatch = 4;
// sums over the stream-K pieces of two 4-feature groups (f0, f1) of token tok
static __device__ __forceinline__ void seg_sum4x2(const float* ws, int t, int max_segs, int nseg, int tok, int f0,
                                                  int f1, float4& a, float4& b) {
  const float* base = ws + ((size_t)t * max_segs * 128 + tok) * 128;
  const float4* p0 = reinterpret_cast<const float4*>(base + f0);
  const float4* p1 = reinterpret_cast<const float4*>(base + f1);
  constexpr size_t stride = 128 * 128 / 4;
  float4 va[kSegBatch], vb[kSegBatch];
#pragma unroll
  for (int s = 0; s < kSegBatch; ++s)
    if (s < nseg) {
      va[s] = __ldcg(p0 + s * stride);
      vb[s] = __ldcg(p1 + s * stride);
    }
  a = make_float4(0.f, 0.f, 0.f, 0.f);
  b = a;
#pragma unroll
  for (int s = 0; s < kSegBatch; ++s)
    if (s < nseg) {
      a.x += va[s].x; a.y += va[s].y; a.z += va[s].z; a.w += va[s].w;
      b.x += vb[s].x; b.y += vb[s].y; b.z += vb[s].z; b.w += vb[s].w;
    }
  for (int s = kSegBatch; s < nseg; ++s) {   // narrow projections (O / down)
    const float4 x = __ldcg(p0 + s * stride), y = __ldcg(p1 + s * stride);
    a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
    b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
  }
}

// deferred-norm statistics of a token in two halves: issue the loads of the
// per-tile sums (the LANES threads of the token -- aligned lane groups --
// split the tiles) ...
struct LaSsLoads {
  float v[8];
};
template <int LANES = 16>
static __device__ __forceinline__ LaSsLoads rstd_issue(const LaRowNorm& n, int tok) {
  LaSsLoads r;
  const int l = threadIdx.x & (LANES - 1);
#pragma unroll
  for (int i = 0; i < 64 / LANES; ++i) {
    const int t = l + LANES * i;
    r.v[i] = t < n.tiles ? __ldcg(n.ss + t * 128 + tok) : 0.f;
  }
  return r;
}
// ... and finish: sum, reduce over the lane group, rsqrt
template <int LANES = 16>
static __device__ __forceinline__ float rstd_finish(const LaRowNorm& n, int tok, const LaSsLoads& r) {
  const unsigned mask = ((LANES == 32) ? 0xffffffffu : ((1u << LANES) - 1u)) << (threadIdx.x & 31 & ~(LANES - 1));
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 64 / LANES; ++i) s += r.v[i];
  for (int t = (threadIdx.x & (LANES - 1)) + 64; t < n.tiles; t += LANES) s += __ldcg(n.ss + t * 128 + tok);   // d > 8192
#pragma unroll
  for (int o = LANES / 2; o > 0; o >>= 1) s += __shfl_xor_sync(mask, s, o);
  return rsqrtf(s * n.inv_d + n.eps);
}
static __device__ __forceinline__ LaSsLoads rstd16_issue(const LaRowNorm& n, int tok) { return rstd_issue<16>(n, tok); }
static __device__ __forceinline__ float rstd16_finish(const LaRowNorm& n, int tok, const LaSsLoads& r) {
  return rstd_finish<16>(n, tok, r);
}

// rsqrt(mean(x^2) + eps) of token tok from the per-tile sums; the 16 threads
// of a half-warp (one token) split the tiles
static __device__ __forceinline__ float rstd16(const LaRowNorm& n, int tok) {
  const int l16 = threadIdx.x & 15;
  const unsigned mask = 0xffffu << (threadIdx.x & 16);
  float s = 0.f;
  for (int t = l16; t < n.tiles; t += 16) s += __ldcg(n.ss + t * 128 + tok);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(mask, s, o);
  return rsqrtf(s * n.inv_d + n.eps);
}

// QKV epilogue of feature tile t, token tok, on the 16 threads of a half-warp
// (lane & 15 -> 4 rotary pairs): piece sums in piece order, deferred-norm
// scale, rotate-half RoPE on q / k; q to the Q buffer, k / v to the cache slot
static __device__ __forceinline__ void la_qkv_fix(const LaQkvEpi& e, const FwdPlan* P, int t, int tok) {
  const int nseg = tile_nseg(e.sp, t);
  const int i0 = (threadIdx.x & 15) * 4;
  const bool v_tile = t >= e.H + e.KVH;
  // every independent load first: norm statistics, RoPE tables, pieces
  const LaSsLoads ssl = rstd16_issue(e.nrm, tok);
  const int pos = P->pos[tok];
  float4 c = make_float4(1.f, 1.f, 1.f, 1.f), sn = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!v_tile) {
    c = __ldg(reinterpret_cast<const float4*>(e.rope_cos + (size_t)pos * 64 + i0));
    sn = __ldg(reinterpret_cast<const float4*>(e.rope_sin + (size_t)pos * 64 + i0));
  }
  float4 a, b;
  seg_sum4x2(e.ws, t, e.sp.max_segs, nseg, tok, i0, i0 + 64, a, b);
  const float rs = rstd16_finish(e.nrm, tok, ssl);   // deferred RMSNorm of the projection input
  a.x *= rs; a.y *= rs; a.z *= rs; a.w *= rs;
  b.x *= rs; b.y *= rs; b.z *= rs; b.w *= rs;
  __nv_bfloat16* dst;
  if (t < e.H) dst = e.q_out + ((size_t)tok * e.H + t) * 128;
  else if (!v_tile) dst = e.kc + ((size_t)P->slot[tok] * e.KVH + (t - e.H)) * 128;
  else dst = e.vc + ((size_t)P->slot[tok] * e.KVH + (t - e.H - e.KVH)) * 128;
  if (!v_tile) {
    // rotate-half RoPE at the row's absolute position
    const float4 a2 = make_float4(a.x * c.x - b.x * sn.x, a.y * c.y - b.y * sn.y,
                                  a.z * c.z - b.z * sn.z, a.w * c.w - b.w * sn.w);
    const float4 b2 = make_float4(b.x * c.x + a.x * sn.x, b.y * c.y + a.y * sn.y,
                                  b.z * c.z + a.z * sn.z, b.w * c.w + a.w * sn.w);
    a = a2;
    b = b2;
  }
  *reinterpret_cast<uint2*>(dst + i0) = make_uint2(pack2(a.x, a.y), pack2(a.z, a.w));
  *reinterpret_cast<uint2*>(dst + i0 + 64) = make_uint2(pack2(b.x, b.y), pack2(b.z, b.w));
}
