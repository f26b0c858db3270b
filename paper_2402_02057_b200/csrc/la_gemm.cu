// tcgen05 swap-AB stream-K GEMM for the lookahead step's projections
// (reference models.py:253-265 -- q/k/v, o, MLP -- and 268 -- unembedding --
// computed here for <= 128 step rows at once against bf16 weights).
//
// CTA = 6 warps: warp 0 TMA producer, warp 1 TMEM allocator + single-thread
// MMA issuer, warps 2-5 epilogue (TMEM lanes 32*(warp%4)...).  One CTA per SM,
// a 6-stage TMA ring of {weight tile 128x64, step-row tile n_pad x 64}
// (128-byte swizzle), two TMEM accumulators (128 lanes x n_pad fp32 columns)
// so the epilogue of one tile overlaps the MMAs of the next.
#include <cudaTypedefs.h>

#include <algorithm>

#include "../../include/lookahead_b200.h"
#include "la_gemm.cuh"
#include "la_ptx.cuh"

void la_set_error(const char* fmt, ...);

namespace {

constexpr int kStages = 6;
constexpr int kABytes = 128 * 128;   // 128 rows x 64 bf16
constexpr int kBBytes = 128 * 128;   // <= 128 rows x 64 bf16
constexpr int kEpiLd = 33;
constexpr int kThreads = 192;
constexpr int kTmemCols = 256;
constexpr size_t kSmemBytes =
    1024 + kStages * (kABytes + kBBytes) + 128 * kEpiLd * 4 + 2 * kStages * 8 + 4 * 8 + 16;

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ long cta_of(long u, long U, long P) { return ((u + 1) * P + U - 1) / U - 1; }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Apply the fused epilogue for one 32-token chunk held in sEpi[f][j].
// Thread et (0..127) owns token j = et/4 and a quarter p = et%4 of the tile.
template <int EPI>
__device__ __forceinline__ void epi_apply(const LaGemmArgs& a, const FwdPlan* P, int tile, int c0,
                                          int n_rows, const float* sEpi, int et) {
  const int j = et >> 2, p = et & 3;
  const int tok = c0 + j;
  const bool valid = tok < n_rows;
  if constexpr (EPI == LA_EPI_QKV) {
    if (!valid) return;
    __nv_bfloat16* dst;
    bool rope = true;
    if (tile < a.H) {
      dst = a.q_out + (size_t)tok * a.H * 128 + tile * 128;
    } else if (tile < a.H + a.KVH) {
      dst = a.kc + (size_t)P->slot[tok] * a.KVH * 128 + (tile - a.H) * 128;
    } else {
      dst = a.vc + (size_t)P->slot[tok] * a.KVH * 128 + (tile - a.H - a.KVH) * 128;
      rope = false;
    }
    if (rope) {
      // rotate-half RoPE: (x_i, x_{i+64}) -> (x_i c - x_{i+64} s, x_{i+64} c + x_i s)
      const int pos = P->pos[tok];
      const float* cs = a.rope_cos + (size_t)pos * 64;
      const float* sn = a.rope_sin + (size_t)pos * 64;
      uint32_t lo[8], hi[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        int i0 = p * 16 + 2 * q, i1 = i0 + 1;
        float x0 = sEpi[i0 * kEpiLd + j], x1 = sEpi[i1 * kEpiLd + j];
        float y0 = sEpi[(i0 + 64) * kEpiLd + j], y1 = sEpi[(i1 + 64) * kEpiLd + j];
        float c0v = cs[i0], c1v = cs[i1], s0 = sn[i0], s1 = sn[i1];
        lo[q] = pack_bf16(x0 * c0v - y0 * s0, x1 * c1v - y1 * s1);
        hi[q] = pack_bf16(y0 * c0v + x0 * s0, y1 * c1v + x1 * s1);
      }
      uint4* d0 = reinterpret_cast<uint4*>(dst + p * 16);
      uint4* d1 = reinterpret_cast<uint4*>(dst + 64 + p * 16);
      d0[0] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      d0[1] = make_uint4(lo[4], lo[5], lo[6], lo[7]);
      d1[0] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      d1[1] = make_uint4(hi[4], hi[5], hi[6], hi[7]);
    } else {
      uint32_t w[16];
#pragma unroll
      for (int q = 0; q < 16; ++q)
        w[q] = pack_bf16(sEpi[(p * 32 + 2 * q) * kEpiLd + j], sEpi[(p * 32 + 2 * q + 1) * kEpiLd + j]);
      uint4* d = reinterpret_cast<uint4*>(dst + p * 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) d[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
  } else if constexpr (EPI == LA_EPI_RESID) {
    if (!valid) return;
    float* xr = a.x + (size_t)tok * a.x_ld + tile * 128 + p * 32;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 v = reinterpret_cast<float4*>(xr)[q];
      v.x += sEpi[(p * 32 + 4 * q + 0) * kEpiLd + j];
      v.y += sEpi[(p * 32 + 4 * q + 1) * kEpiLd + j];
      v.z += sEpi[(p * 32 + 4 * q + 2) * kEpiLd + j];
      v.w += sEpi[(p * 32 + 4 * q + 3) * kEpiLd + j];
      reinterpret_cast<float4*>(xr)[q] = v;
    }
  } else if constexpr (EPI == LA_EPI_SWIGLU) {
    if (!valid) return;
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int i0 = p * 16 + 2 * q;
      float g0 = sEpi[i0 * kEpiLd + j], g1 = sEpi[(i0 + 1) * kEpiLd + j];
      float u0 = sEpi[(64 + i0) * kEpiLd + j], u1 = sEpi[(64 + i0 + 1) * kEpiLd + j];
      w[q] = pack_bf16(g0 / (1.0f + __expf(-g0)) * u0, g1 / (1.0f + __expf(-g1)) * u1);
    }
    uint4* d = reinterpret_cast<uint4*>(a.act + (size_t)tok * a.act_ld + tile * 64 + p * 16);
    d[0] = make_uint4(w[0], w[1], w[2], w[3]);
    d[1] = make_uint4(w[4], w[5], w[6], w[7]);
  } else {  // LA_EPI_LOGITS
    float best = -INFINITY;
    int bi = 0x7fffffff;
    if (valid) {
#pragma unroll 8
      for (int q = 0; q < 32; ++q) {
        int f = p * 32 + q, fg = tile * 128 + f;
        if (fg < a.V) {
          float v = sEpi[f * kEpiLd + j];
          if (a.logits) a.logits[(size_t)tok * a.V + fg] = v;
          if (v > best) { best = v; bi = fg; }   // ascending fg: ties keep the lowest
        }
      }
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      float v2 = __shfl_xor_sync(0xffffffffu, best, o);
      int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (v2 > best || (v2 == best && i2 < bi)) { best = v2; bi = i2; }
    }
    if (valid && p == 0) a.pmax[(size_t)tile * 128 + tok] = make_float2(best, __int_as_float(bi));
  }
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    la_gemm_kernel(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
                   const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mB,
                   const LaGemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  const FwdPlan* P = args.plan;
  const int n_rows = P->n_rows;
  if (n_rows == 0) return;                       // decode finished: nothing to do
  const int n_pad = P->n_pad;
  uint8_t* sm = smem_raw + ((1024 - (ptx::smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = sm;
  uint8_t* sB = sA + kStages * kABytes;
  float* sEpi = reinterpret_cast<float*>(sB + kStages * kBBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + 128 * kEpiLd);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (args.timing && threadIdx.x == 0) {
    if (atomicAdd(&args.timing[3], 1ull) == 0ull) args.timing[0] = globaltimer();
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&tfull[b], 1); ptx::mbar_init(&tempty[b], 128); }
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&mA0);
    ptx::tma_prefetch_desc(&mB);
    if (args.a_mode) { ptx::tma_prefetch_desc(&mA1); }
    if (args.a_mode == 1) { ptx::tma_prefetch_desc(&mA2); }
  }
  if (warp == 1) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int kb = args.kb;
  const long U = (long)args.n_tiles * kb;
  const long Pn = gridDim.x;
  const long u_begin = (long)blockIdx.x * U / Pn;
  const long u_end = (long)(blockIdx.x + 1) * U / Pn;

  if (warp == 0) {
    // ---------------------------------------------------- TMA producer
    if (lane == 0) {
      const uint64_t pol_w = ptx::policy_evict_first();   // weights: streamed once
      const uint64_t pol_x = ptx::policy_evict_last();    // step rows: re-read by every CTA
      const uint32_t bbytes = (uint32_t)n_pad * 128;
      long it = 0;
      for (long u = u_begin; u < u_end; ++u, ++it) {
        const int tile = (int)(u / kb), k = (int)(u % kb);
        const int s = (int)(it % kStages);
        const uint32_t r = (uint32_t)(it / kStages);
        if (r > 0) ptx::mbar_wait(&empty[s], (r - 1) & 1);
        ptx::mbar_expect_tx(&full[s], kABytes + bbytes);
        uint8_t* a = sA + s * kABytes;
        uint8_t* b = sB + s * kBBytes;
        const int kc = k * 64;
        if (args.a_mode == 0) {
          ptx::tma_load_2d(a, &mA0, &full[s], kc, tile * 128, pol_w);
        } else if (args.a_mode == 1) {
          if (tile < args.t0) ptx::tma_load_2d(a, &mA0, &full[s], kc, tile * 128, pol_w);
          else if (tile < args.t1) ptx::tma_load_2d(a, &mA1, &full[s], kc, (tile - args.t0) * 128, pol_w);
          else ptx::tma_load_2d(a, &mA2, &full[s], kc, (tile - args.t1) * 128, pol_w);
        } else {
          ptx::tma_load_2d(a, &mA0, &full[s], kc, tile * 64, pol_w);
          ptx::tma_load_2d(a + 64 * 128, &mA1, &full[s], kc, tile * 64, pol_w);
        }
        for (int jb = 0; jb < n_pad / 16; ++jb)
          ptx::tma_load_2d(b + jb * 2048, &mB, &full[s], kc, jb * 16, pol_x);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = ptx::umma_idesc_bf16(128, (uint32_t)n_pad);
      long it = 0, u = u_begin;
      int use[2] = {0, 0}, buf = 0;
      while (u < u_end) {
        const int tile = (int)(u / kb);
        const long seg_start = u, seg_end = std::min(u_end, (long)(tile + 1) * kb);
        if (use[buf] > 0) {
          ptx::mbar_wait(&tempty[buf], (use[buf] - 1) & 1);
          ptx::tc_fence_after();
        }
        const uint32_t d_tmem = tmem + buf * 128;
        for (; u < seg_end; ++u, ++it) {
          const int s = (int)(it % kStages);
          ptx::mbar_wait(&full[s], (uint32_t)(it / kStages) & 1);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sA + s * kABytes);
          const uint32_t b_addr = ptx::smem_u32(sB + s * kBBytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::umma_bf16(d_tmem, ptx::umma_desc_sw128(a_addr + kk * 32),
                           ptx::umma_desc_sw128(b_addr + kk * 32), idesc,
                           (u > seg_start || kk > 0) ? 1u : 0u);
          ptx::umma_commit(&empty[s]);
        }
        ptx::umma_commit(&tfull[buf]);
        use[buf]++;
        buf ^= 1;
      }
    }
  } else {
    // -------------------------------------------------------- epilogue
    const int et = threadIdx.x - 64;              // 0..127
    const int row_base = 32 * (warp & 3);
    const int f = row_base + lane;                // accumulator lane = output feature in tile
    int use[2] = {0, 0}, buf = 0;
    long u = u_begin;
    while (u < u_end) {
      const int tile = (int)(u / kb);
      const long seg_start = u, seg_end = std::min(u_end, (long)(tile + 1) * kb);
      const bool whole = seg_start == (long)tile * kb && seg_end == (long)(tile + 1) * kb;
      ptx::mbar_wait(&tfull[buf], use[buf] & 1);
      ptx::tc_fence_after();
      const uint32_t t_base = tmem + ((uint32_t)row_base << 16) + buf * 128;
      if (whole) {
        for (int c0 = 0; c0 < n_pad; c0 += 32) {
          float v[32];
          ptx::tmem_ld32(t_base + c0, v);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) sEpi[f * kEpiLd + jj] = v[jj];
          ptx::named_bar_sync(1, 128);
          epi_apply<EPI>(args, P, tile, c0, n_rows, sEpi, et);
          ptx::named_bar_sync(1, 128);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[buf]);
      } else {
        // stream-K partial: write fp32 partial, last arriver reduces in segment order
        const long c_first = cta_of((long)tile * kb, U, Pn);
        const int seg = (int)(blockIdx.x - c_first);
        float* wsp = args.ws + ((size_t)tile * args.max_segs + seg) * 128 * 128;
        for (int c0 = 0; c0 < n_pad; c0 += 32) {
          float v[32];
          ptx::tmem_ld32(t_base + c0, v);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) __stcg(wsp + (size_t)(c0 + jj) * 128 + f, v[jj]);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[buf]);
        __threadfence();
        ptx::named_bar_sync(1, 128);
        if (et == 0) {
          const int nseg = (int)(cta_of((long)(tile + 1) * kb - 1, U, Pn) - c_first + 1);
          const int old = atomicAdd(&args.counters[tile], 1);
          *flag = (old == nseg - 1) ? nseg : 0;
        }
        ptx::named_bar_sync(1, 128);
        const int nseg = *flag;
        if (nseg) {
          __threadfence();
          const float* base = args.ws + (size_t)tile * args.max_segs * 128 * 128;
          for (int c0 = 0; c0 < n_pad; c0 += 32) {
#pragma unroll 4
            for (int jj = 0; jj < 32; ++jj) {
              float acc = 0.f;
              for (int sg = 0; sg < nseg; ++sg)
                acc += __ldcg(base + ((size_t)sg * 128 + c0 + jj) * 128 + f);
              sEpi[f * kEpiLd + jj] = acc;
            }
            ptx::named_bar_sync(1, 128);
            epi_apply<EPI>(args, P, tile, c0, n_rows, sEpi, et);
            ptx::named_bar_sync(1, 128);
          }
          if (et == 0) args.counters[tile] = 0;
        }
        ptx::named_bar_sync(1, 128);
      }
      use[buf]++;
      buf ^= 1;
      u = seg_end;
    }
    ptx::tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem);
  }
  if (args.timing && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&args.timing[4], 1ull) == (unsigned long long)gridDim.x - 1) {
      unsigned long long t1 = globaltimer();
      args.timing[1] += t1 - args.timing[0];
      args.timing[2] += 1;
      args.timing[3] = 0;
      args.timing[4] = 0;
    }
  }
}

}  // namespace

// ------------------------------------------------------------------ host
int la_sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int la_make_tmap(CUtensorMap* map, const void* base, int rows, int K, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || !fn) {
      la_set_error("cuTensorMapEncodeTiled unavailable");
      return LA_ERR_CUDA;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    la_set_error("cuTensorMapEncodeTiled failed (%d) rows=%d K=%d box=%d", (int)r, rows, K, box_rows);
    return LA_ERR_CUDA;
  }
  return LA_OK;
}

int la_gemm_workspace_segs(int n_tiles, int kb, int grid) {
  long U = (long)n_tiles * kb, P = grid, mx = 1;
  for (int t = 0; t < n_tiles; ++t) {
    long c0 = ((long)t * kb + 1) * P / U, c1 = ((long)(t + 1) * kb) * P / U;
    // cta_of(u) = ceil((u+1)P/U) - 1
    c0 = (((long)t * kb + 1) * P + U - 1) / U - 1;
    c1 = (((long)(t + 1) * kb) * P + U - 1) / U - 1;
    mx = std::max(mx, c1 - c0 + 1);
  }
  return (int)mx;
}

template <int EPI>
static int launch_epi(const LaGemm& g, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(la_gemm_kernel<EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e != cudaSuccess) { la_set_error("gemm smem attr: %s", cudaGetErrorString(e)); return LA_ERR_CUDA; }
    attr = true;
  }
  la_gemm_kernel<EPI><<<g.grid, kThreads, kSmemBytes, st>>>(g.a0, g.a1, g.a2, g.b, g.args);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { la_set_error("gemm launch: %s", cudaGetErrorString(e)); return LA_ERR_CUDA; }
  return LA_OK;
}

int la_gemm_launch(const LaGemm& g, cudaStream_t st) {
  switch (g.epi) {
    case LA_EPI_QKV: return launch_epi<LA_EPI_QKV>(g, st);
    case LA_EPI_RESID: return launch_epi<LA_EPI_RESID>(g, st);
    case LA_EPI_SWIGLU: return launch_epi<LA_EPI_SWIGLU>(g, st);
    default: return launch_epi<LA_EPI_LOGITS>(g, st);
  }
}
