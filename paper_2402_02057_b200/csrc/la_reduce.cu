// Split-K reduction + fused epilogues of the tcgen05 GEMM (la_gemm.cu).
//
// Each output element is the sum of its tile's fp32 segment partials taken in
// segment order -- fixed by the stream-K geometry alone, so the result is
// deterministic and identical for every step layout / LP shard.  The
// epilogues are the ops that follow each projection in the reference model
// (models.py:253-265 restated for the Llama family):
//   QKV     -> rotate-half RoPE on q, k; q to the Q buffer, k/v to the cache slot
//   O, down -> residual add + the next RMSNorm (one CTA per row)
//   gate/up -> SwiGLU
//   LM head -> per-row (max, argmax) via one 64-bit atomicMax per (tile, row)
// Every thread handles 4 consecutive features and issues the loads of all
// segments before summing (latency-bound otherwise: ~10 segments per element
// for the narrow O / down projections).
#include <cuda_bf16.h>

#include "la_gemm.cuh"
#include "la_reduce.cuh"
#include "la_reduce_dev.cuh"

namespace {

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// order-preserving key: larger value wins, then the LOWER index
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (uint32_t)(0x7fffffff - idx);
}

}  // namespace

// grid = (H + 2*KVH tiles, rows/8), block = 128: thread = (token, 4 rotary pairs)
__global__ void __launch_bounds__(128, 8) la_qkv_epi_kernel(LaQkvEpi e) {
  la_epi_enter(e.ready, e.runs, e.sp, blockIdx.x, e.pf);
  const FwdPlan* P = e.plan;
  const int tok = blockIdx.y * 8 + (threadIdx.x >> 4);
  if (tok >= P->n_rows) return;
  la_qkv_fix(e, P, blockIdx.x, tok);
}

// grid = (d/128 tiles, rows/8), block = 256: warp = (row, 128-feature tile),
// lane = 4 features.  x (+)= sum of segment partials (or := embedding row);
// next GEMM input bf16(x * g) (deferred RMSNorm) and the tile's sum of x^2
__global__ void __launch_bounds__(256, 4) la_resid_norm_kernel(LaResidNorm e) {
  la_epi_enter(e.ready, e.runs, e.sp, blockIdx.x, e.pf);
  const FwdPlan* P = e.plan;
  const int r = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (r >= P->n_rows) return;
  const int t = blockIdx.x;
  const int f = t * 128 + (threadIdx.x & 31) * 4;
  float* xr = e.x + (size_t)r * e.d;
  const float4 g = __ldg(reinterpret_cast<const float4*>(e.g + f));
  float4 v;
  if (e.embed) {
    const __nv_bfloat16* er = e.embed + (size_t)P->ids[r] * e.d + f;
    const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(er));
    const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(er + 2));
    v = make_float4(lo.x, lo.y, hi.x, hi.y);
  } else {
    v = *reinterpret_cast<const float4*>(xr + f);
    if (e.ws) {
      const float4 p = seg_sum4(e.ws, t, e.sp.max_segs, tile_nseg(e.sp, t), r, f & 127);
      v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
    }
  }
  *reinterpret_cast<float4*>(xr + f) = v;
  *reinterpret_cast<uint2*>(e.h + la_act_off(r, f)) =
      make_uint2(pack2(v.x * g.x, v.y * g.y), pack2(v.z * g.z, v.w * g.w));
  float ss = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) e.ss[t * 128 + r] = ss;
}

// grid = (ffn/64 tiles, rows/16), block = 128: thread = (token, 8 outputs),
// 8 threads per token -- one wave over the GPU, every load issued before use
__global__ void __launch_bounds__(128, 8) la_swiglu_epi_kernel(LaSwigluEpi e) {
  la_epi_enter(e.ready, e.runs, e.sp, blockIdx.x, e.pf);
  const FwdPlan* P = e.plan;
  const int t = blockIdx.x;
  const int tok = blockIdx.y * 16 + (threadIdx.x >> 3);
  if (tok >= P->n_rows) return;
  const int nseg = tile_nseg(e.sp, t);
  const int i0 = (threadIdx.x & 7) * 8;
  const LaSsLoads ssl = rstd_issue<8>(e.nrm, tok);
  float4 g0, u0, g1, u1;
  seg_sum4x2(e.ws, t, e.sp.max_segs, nseg, tok, i0, i0 + 64, g0, u0);
  seg_sum4x2(e.ws, t, e.sp.max_segs, nseg, tok, i0 + 4, i0 + 68, g1, u1);
  const float rs = rstd_finish<8>(e.nrm, tok, ssl);
  const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
  const float u[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
  float w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float gg = g[i] * rs, uu = u[i] * rs;
    w[i] = gg / (1.0f + __expf(-gg)) * uu;
  }
  *reinterpret_cast<uint4*>(e.act + la_act_off(tok, t * 64 + i0)) =
      make_uint4(pack2(w[0], w[1]), pack2(w[2], w[3]), pack2(w[4], w[5]), pack2(w[6], w[7]));
}

// grid = (LM-head tiles, rows/8), block = 128: thread = (token, 8 vocabulary
// rows); the row's argmax is folded with one 64-bit atomicMax per (tile, row)
// whose key orders by value then by LOWER index (sampling.py:17-19), so the
// result does not depend on arrival order.
__global__ void __launch_bounds__(128, 8) la_logits_epi_kernel(LaLogitsEpi e) {
  la_epi_enter(e.ready, e.runs, e.sp, blockIdx.x, LaPrefetch{});
  const FwdPlan* P = e.plan;
  const int tok = blockIdx.y * 8 + (threadIdx.x >> 4);
  const bool valid = tok < P->n_rows;
  const int t = blockIdx.x;
  const int nseg = tile_nseg(e.sp, t);
  const int f0 = (threadIdx.x & 15) * 8;
  unsigned long long best = 0ull;
  if (valid) {
    const LaSsLoads ssl = rstd16_issue(e.nrm, tok);
    float4 a, b;
    seg_sum4x2(e.ws, t, e.sp.max_segs, nseg, tok, f0, f0 + 4, a, b);
    const float rs = rstd16_finish(e.nrm, tok, ssl);
    const float v[8] = {a.x * rs, a.y * rs, a.z * rs, a.w * rs, b.x * rs, b.y * rs, b.z * rs, b.w * rs};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int fg = t * 128 + f0 + q;
      if (fg < e.V) {
        if (e.logits) e.logits[(size_t)tok * e.V + fg] = v[q];
        unsigned long long k = argmax_key(v[q], fg);
        best = k > best ? k : best;
      }
    }
  }
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    unsigned long long k = __shfl_xor_sync(0xffffffffu, best, o);
    best = k > best ? k : best;
  }
  if (valid && (threadIdx.x & 15) == 0 && best) atomicMax(e.keys + tok, best);
}

// per-row winner of the atomicMax keys -> row argmax; owned rows go to the
// decode state's global-row table; keys are reset for the next forward
__global__ void la_argmax_finish_kernel(const FwdPlan* P, unsigned long long* keys, int* row_amax,
                                        DevDecode* dp) {
  LA_PDL_ENTRY();
  const int r = threadIdx.x;
  if (r >= LA_MAX_ROWS) return;
  const unsigned long long k = keys[r];
  keys[r] = 0ull;
  if (r >= P->n_rows) return;
  const int idx = 0x7fffffff - (int)(uint32_t)(k & 0xffffffffu);
  row_amax[r] = idx;
  if (dp && P->own[r]) dp->amax[P->grow[r]] = idx;
}

LA_TL_DEFINE_SETTER(reduce)
