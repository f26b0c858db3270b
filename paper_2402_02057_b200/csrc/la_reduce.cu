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
//   LM head -> per-tile (max, argmax) (+ optional fp32 logits dump)
#include <cuda_bf16.h>

#include "la_gemm.cuh"
#include "la_reduce.cuh"

namespace {

__device__ __forceinline__ float seg_sum(const float* ws, int t, int max_segs, int nseg, int tok, int f) {
  const float* p = ws + ((size_t)t * max_segs * 128 + tok) * 128 + f;
  float acc = 0.f;
  for (int s = 0; s < nseg; ++s) acc += __ldcg(p + (size_t)s * 128 * 128);
  return acc;
}

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

}  // namespace

// grid = H + 2*KVH tiles (one attention head each), block = 256
__global__ void __launch_bounds__(256) la_qkv_epi_kernel(LaQkvEpi e) {
  const FwdPlan* P = e.plan;
  const int n = P->n_rows;
  if (n == 0) return;
  const int t = blockIdx.x;
  long c0;
  int nseg;
  la_tile_segs(t, e.sp.kb, e.sp.n_tiles, e.sp.grid, c0, nseg);
  const int i = threadIdx.x & 63;
  const bool v_tile = t >= e.H + e.KVH;
  for (int tok = threadIdx.x >> 6; tok < n; tok += blockDim.x >> 6) {
    float a = seg_sum(e.ws, t, e.sp.max_segs, nseg, tok, i);
    float b = seg_sum(e.ws, t, e.sp.max_segs, nseg, tok, i + 64);
    __nv_bfloat16* dst;
    if (t < e.H) dst = e.q_out + ((size_t)tok * e.H + t) * 128;
    else if (!v_tile) dst = e.kc + ((size_t)P->slot[tok] * e.KVH + (t - e.H)) * 128;
    else dst = e.vc + ((size_t)P->slot[tok] * e.KVH + (t - e.H - e.KVH)) * 128;
    if (!v_tile) {
      // rotate-half RoPE at the row's absolute position
      const float c = e.rope_cos[(size_t)P->pos[tok] * 64 + i];
      const float s = e.rope_sin[(size_t)P->pos[tok] * 64 + i];
      const float a2 = a * c - b * s, b2 = b * c + a * s;
      a = a2;
      b = b2;
    }
    dst[i] = __float2bfloat16_rn(a);
    dst[i + 64] = __float2bfloat16_rn(b);
  }
}

// grid = rows, block = 256: x (+)= sum of segment partials (or := embedding
// row), then RMSNorm -> bf16 GEMM input
__global__ void __launch_bounds__(256) la_resid_norm_kernel(LaResidNorm e) {
  const FwdPlan* P = e.plan;
  const int r = blockIdx.x;
  if (r >= P->n_rows) return;
  __shared__ float red[8];
  float* xr = e.x + (size_t)r * e.d;
  float ss = 0.f;
  for (int f = threadIdx.x; f < e.d; f += blockDim.x) {
    float v;
    if (e.embed) {
      v = __bfloat162float(e.embed[(size_t)P->ids[r] * e.d + f]);
    } else {
      v = xr[f];
      if (e.ws) {
        const int t = f >> 7;
        long c0;
        int nseg;
        la_tile_segs(t, e.sp.kb, e.sp.n_tiles, e.sp.grid, c0, nseg);
        v += seg_sum(e.ws, t, e.sp.max_segs, nseg, r, f & 127);
      }
    }
    xr[f] = v;
    ss += v * v;
  }
  const float inv = rsqrtf(block_sum(ss, red) / e.d + e.eps);
  for (int f = threadIdx.x; f < e.d; f += blockDim.x)
    e.h[la_act_off(r, f)] = __float2bfloat16_rn(xr[f] * inv * e.g[f]);
}

// grid = ffn/64 tiles (64 gate + 64 up rows each), block = 256
__global__ void __launch_bounds__(256) la_swiglu_epi_kernel(LaSwigluEpi e) {
  const FwdPlan* P = e.plan;
  const int n = P->n_rows;
  if (n == 0) return;
  const int t = blockIdx.x;
  long c0;
  int nseg;
  la_tile_segs(t, e.sp.kb, e.sp.n_tiles, e.sp.grid, c0, nseg);
  const int i = threadIdx.x & 63;
  for (int tok = threadIdx.x >> 6; tok < n; tok += blockDim.x >> 6) {
    const float g = seg_sum(e.ws, t, e.sp.max_segs, nseg, tok, i);
    const float u = seg_sum(e.ws, t, e.sp.max_segs, nseg, tok, i + 64);
    e.act[la_act_off(tok, t * 64 + i)] = __float2bfloat16_rn(g / (1.0f + __expf(-g)) * u);
  }
}

// grid = LM-head tiles, block = 128 (thread = token): per-tile (max, argmax)
// over the tile's 128 vocabulary rows, ties -> lowest id (sampling.py:17-19)
__global__ void __launch_bounds__(128) la_logits_epi_kernel(LaLogitsEpi e) {
  const FwdPlan* P = e.plan;
  const int tok = threadIdx.x;
  if (tok >= P->n_rows) return;
  const int t = blockIdx.x;
  long c0;
  int nseg;
  la_tile_segs(t, e.sp.kb, e.sp.n_tiles, e.sp.grid, c0, nseg);
  float best = -INFINITY;
  int bi = 0x7fffffff;
  const float* base = e.ws + ((size_t)t * e.sp.max_segs * 128 + tok) * 128;
  for (int f4 = 0; f4 < 32; ++f4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nseg; ++s) {
      float4 v = __ldcg(reinterpret_cast<const float4*>(base + (size_t)s * 128 * 128) + f4);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const float vals[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int fg = t * 128 + f4 * 4 + q;
      if (fg < e.V) {
        if (e.logits) e.logits[(size_t)tok * e.V + fg] = vals[q];
        if (vals[q] > best) { best = vals[q]; bi = fg; }
      }
    }
  }
  e.pmax[(size_t)t * 128 + tok] = make_float2(best, __int_as_float(bi));
}
