// tcgen05 swap-AB stream-K GEMM for the lookahead step's projections
// (reference models.py:253-265 -- q/k/v, o, MLP -- and 268 -- unembedding --
// computed for <= 128 step rows at once against packed bf16 weight tiles).
//
// CTA = 6 warps: warp 0 producer (1-D bulk copy of the contiguous 16 KB
// weight tile + TMA of the step-row tile), warp 1 TMEM allocator + single-
// thread MMA issuer, warps 2-5 drain TMEM (lanes 32*(warp%4)..) to the fp32
// partial workspace.  One CTA per SM, 6-stage smem ring, two TMEM
// accumulators so draining one segment overlaps the MMAs of the next.
#include <cudaTypedefs.h>

#include <algorithm>

#include "../../include/lookahead_b200.h"
#include "la_gemm.cuh"
#include "la_ptx.cuh"
#include "la_reduce_dev.cuh"

void la_set_error(const char* fmt, ...);

namespace {

constexpr int kStages = 4;                     // stages of 2-tile units (48 KB each)
constexpr int kMaxStages = 6;                  // stages of 1-tile units (32 KB each), same ring
constexpr int kTileBytes = 128 * 128;          // 128 rows x 64 bf16
constexpr int kABytes = LA_TPC * kTileBytes;   // weight tiles per unit
constexpr int kBBytes = 128 * 128;             // <= 128 rows x 64 bf16
constexpr int kThreads = 192;
constexpr int kTmemCols = 512;                 // 2 buffers x LA_TPC tiles x 128 columns
constexpr int kEpiLd = 33;                     // fused-epilogue staging [128 f][33]
constexpr int kStageFloats = 4 * 32 * 36;      // >= 128 * kEpiLd: also the pieces' transpose staging
constexpr size_t kSmemBytes =
    1024 + kStages * (kABytes + kBBytes) + kStageFloats * 4 + 2 * kMaxStages * 8 + 5 * 8 + 16 + 128 + 128 * 4;

constexpr bool is_fx(int epi) { return epi >= LA_EPI_FX_QKV && epi <= LA_EPI_FX_RESID; }

// ------------------------------------------------ in-GEMM split-K fix-up
// Staging image of one unit tile's row slice: S[s][tt][rr][128 f] fp32 for
// pieces s < nseg, tiles tt < tpc, slice rows rr < nr.
__device__ __forceinline__ const float* fx_piece(const float* S, int s, int tt, int rr, int tpc, int nr) {
  return S + ((size_t)(s * tpc + tt) * nr + rr) * 128;
}
// sum over the pieces, in piece order, of 4 consecutive features (as seg_sum4)
__device__ __forceinline__ float4 fx_sum4(const float* S, int nseg, int tt, int rr, int tpc, int nr, int f) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < nseg; ++s) {
    const float4 v = *reinterpret_cast<const float4*>(fx_piece(S, s, tt, rr, tpc, nr) + f);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  return acc;
}

// Epilogue of rows [r0, r0 + nr) of unit tile ut on the 128 drain threads
// (et = 0..127).  The arithmetic is exactly that of the standalone epilogue
// kernels (la_reduce.cu) -- same piece order, same lane grouping for the norm
// statistics -- so the fused and unfused paths agree bit for bit.
template <int EPI>
__device__ void fx_finish(const LaGemmArgs& a, const FwdPlan* P, int ut, int r0, int nr, int nseg,
                          const float* S, int et) {
  const int lane = et & 31;
  const int tpc = a.tpc, items = tpc * nr;
  if constexpr (EPI == LA_EPI_FX_RESID) {
    // warp = (tile, row), lane = 4 features (la_resid_norm_kernel)
    for (int it = et >> 5; it < items; it += 4) {
      const int tt = it / nr, rr = it % nr;
      const int t = ut * tpc + tt;
      if (t >= a.n_real) continue;
      const int r = r0 + rr, fl = lane * 4, f = t * 128 + fl;
      const float4 p = fx_sum4(S, nseg, tt, rr, tpc, nr, fl);
      float* xr = a.x + (size_t)r * a.d + f;
      const float4 g = __ldg(reinterpret_cast<const float4*>(a.gain + f));
      float4 v = *reinterpret_cast<const float4*>(xr);
      v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
      *reinterpret_cast<float4*>(xr) = v;
      *reinterpret_cast<uint2*>(a.h_out + la_act_off(r, f)) =
          make_uint2(pack2(v.x * g.x, v.y * g.y), pack2(v.z * g.z, v.w * g.w));
      float ss = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) a.ss_out[t * 128 + r] = ss;
    }
  } else if constexpr (EPI == LA_EPI_FX_QKV) {
    // half-warp = (tile, row), lane & 15 = 4 rotary pairs (la_qkv_fix)
    for (int it = et >> 4; it < items; it += 8) {
      const int tt = it / nr, rr = it % nr;
      const int t = ut * tpc + tt;
      if (t >= a.n_real) continue;
      const int tok = r0 + rr;
      const int i0 = (et & 15) * 4;
      const bool v_tile = t >= a.H + a.KVH;
      const LaSsLoads ssl = rstd16_issue(a.nrm, tok);
      const int pos = P->pos[tok];
      float4 c = make_float4(1.f, 1.f, 1.f, 1.f), sn = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!v_tile) {
        c = __ldg(reinterpret_cast<const float4*>(a.rope_cos + (size_t)pos * 64 + i0));
        sn = __ldg(reinterpret_cast<const float4*>(a.rope_sin + (size_t)pos * 64 + i0));
      }
      float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
      for (int s = 0; s < nseg; ++s) {
        const float* pp = fx_piece(S, s, tt, rr, tpc, nr);
        const float4 u = *reinterpret_cast<const float4*>(pp + i0);
        const float4 w = *reinterpret_cast<const float4*>(pp + i0 + 64);
        x0.x += u.x; x0.y += u.y; x0.z += u.z; x0.w += u.w;
        x1.x += w.x; x1.y += w.y; x1.z += w.z; x1.w += w.w;
      }
      const float rs = rstd16_finish(a.nrm, tok, ssl);
      x0.x *= rs; x0.y *= rs; x0.z *= rs; x0.w *= rs;
      x1.x *= rs; x1.y *= rs; x1.z *= rs; x1.w *= rs;
      __nv_bfloat16* dst;
      if (t < a.H) dst = a.q_out + ((size_t)tok * a.H + t) * 128;
      else if (!v_tile) dst = a.kc + ((size_t)P->slot[tok] * a.KVH + (t - a.H)) * 128;
      else dst = a.vc + ((size_t)P->slot[tok] * a.KVH + (t - a.H - a.KVH)) * 128;
      if (!v_tile) {
        const float4 a2 = make_float4(x0.x * c.x - x1.x * sn.x, x0.y * c.y - x1.y * sn.y,
                                      x0.z * c.z - x1.z * sn.z, x0.w * c.w - x1.w * sn.w);
        const float4 b2 = make_float4(x1.x * c.x + x0.x * sn.x, x1.y * c.y + x0.y * sn.y,
                                      x1.z * c.z + x0.z * sn.z, x1.w * c.w + x0.w * sn.w);
        x0 = a2;
        x1 = b2;
      }
      *reinterpret_cast<uint2*>(dst + i0) = make_uint2(pack2(x0.x, x0.y), pack2(x0.z, x0.w));
      *reinterpret_cast<uint2*>(dst + i0 + 64) = make_uint2(pack2(x1.x, x1.y), pack2(x1.z, x1.w));
    }
  } else if constexpr (EPI == LA_EPI_FX_SWIGLU) {
    // 8 threads = (tile, row), 8 outputs each (la_swiglu_epi_kernel)
    for (int it = et >> 3; it < items; it += 16) {
      const int tt = it / nr, rr = it % nr;
      const int t = ut * tpc + tt;
      if (t >= a.n_real) continue;
      const int tok = r0 + rr;
      const int i0 = (et & 7) * 8;
      const LaSsLoads ssl = rstd_issue<8>(a.nrm, tok);
      float4 g0 = make_float4(0.f, 0.f, 0.f, 0.f), u0 = g0, g1 = g0, u1 = g0;
      for (int s = 0; s < nseg; ++s) {
        const float* pp = fx_piece(S, s, tt, rr, tpc, nr);
        const float4 a0 = *reinterpret_cast<const float4*>(pp + i0);
        const float4 b0 = *reinterpret_cast<const float4*>(pp + i0 + 64);
        const float4 a1 = *reinterpret_cast<const float4*>(pp + i0 + 4);
        const float4 b1 = *reinterpret_cast<const float4*>(pp + i0 + 68);
        g0.x += a0.x; g0.y += a0.y; g0.z += a0.z; g0.w += a0.w;
        u0.x += b0.x; u0.y += b0.y; u0.z += b0.z; u0.w += b0.w;
        g1.x += a1.x; g1.y += a1.y; g1.z += a1.z; g1.w += a1.w;
        u1.x += b1.x; u1.y += b1.y; u1.z += b1.z; u1.w += b1.w;
      }
      const float rs = rstd_finish<8>(a.nrm, tok, ssl);
      const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float u[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
      float w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gg = g[i] * rs, uu = u[i] * rs;
        w[i] = gg / (1.0f + __expf(-gg)) * uu;
      }
      *reinterpret_cast<uint4*>(a.act + la_act_off(tok, t * 64 + i0)) =
          make_uint4(pack2(w[0], w[1]), pack2(w[2], w[3]), pack2(w[4], w[5]), pack2(w[6], w[7]));
    }
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// order-preserving argmax key: larger value wins, then the LOWER index
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (uint32_t)(0x7fffffff - idx);
}

// Fused epilogue of one 32-token chunk of feature tile `ftile` held in
// sEpi[f][j]; thread et (0..127) owns token j = et/4, quarter p = et%4.
template <int EPI>
__device__ __forceinline__ void epi_apply(const LaGemmArgs& a, const FwdPlan* P, int ftile, int c0,
                                          int n_rows, const float* sEpi, int et) {
  const int j = et >> 2, p = et & 3;
  const int tok = c0 + j;
  const bool valid = tok < n_rows;
  if constexpr (EPI == LA_EPI_QKV) {
    if (!valid) return;
    __nv_bfloat16* dst;
    bool rope = true;
    if (ftile < a.H) {
      dst = a.q_out + ((size_t)tok * a.H + ftile) * 128;
    } else if (ftile < a.H + a.KVH) {
      dst = a.kc + ((size_t)P->slot[tok] * a.KVH + (ftile - a.H)) * 128;
    } else if (ftile < a.H + 2 * a.KVH) {
      dst = a.vc + ((size_t)P->slot[tok] * a.KVH + (ftile - a.H - a.KVH)) * 128;
      rope = false;
    } else {
      return;   // zero padding tile
    }
    if (rope) {
      // rotate-half RoPE: (x_i, x_{i+64}) -> (x_i c - x_{i+64} s, x_{i+64} c + x_i s)
      const float* cs = a.rope_cos + (size_t)P->pos[tok] * 64;
      const float* sn = a.rope_sin + (size_t)P->pos[tok] * 64;
      uint32_t lo[8], hi[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i0 = p * 16 + 2 * q, i1 = i0 + 1;
        const float x0 = sEpi[i0 * kEpiLd + j], x1 = sEpi[i1 * kEpiLd + j];
        const float y0 = sEpi[(i0 + 64) * kEpiLd + j], y1 = sEpi[(i1 + 64) * kEpiLd + j];
        lo[q] = pack_bf16(x0 * cs[i0] - y0 * sn[i0], x1 * cs[i1] - y1 * sn[i1]);
        hi[q] = pack_bf16(y0 * cs[i0] + x0 * sn[i0], y1 * cs[i1] + x1 * sn[i1]);
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
  } else if constexpr (EPI == LA_EPI_SWIGLU) {
    if (!valid) return;
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i0 = p * 16 + 2 * q;
      const float g0 = sEpi[i0 * kEpiLd + j], g1 = sEpi[(i0 + 1) * kEpiLd + j];
      const float u0 = sEpi[(64 + i0) * kEpiLd + j], u1 = sEpi[(64 + i0 + 1) * kEpiLd + j];
      w[q] = pack_bf16(g0 / (1.0f + __expf(-g0)) * u0, g1 / (1.0f + __expf(-g1)) * u1);
    }
    // 16 outputs = 2 swizzled 16-byte chunks of the packed LA-row layout
    __nv_bfloat16* base = a.act;
    const int k0 = ftile * 64 + p * 16;
    *reinterpret_cast<uint4*>(base + la_act_off(tok, k0)) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(base + la_act_off(tok, k0 + 8)) = make_uint4(w[4], w[5], w[6], w[7]);
  } else if constexpr (EPI == LA_EPI_LOGITS) {
    unsigned long long best = 0ull;
    if (valid) {
#pragma unroll 8
      for (int q = 0; q < 32; ++q) {
        const int f = p * 32 + q, fg = ftile * 128 + f;
        if (fg < a.V) {
          const float v = sEpi[f * kEpiLd + j];
          if (a.logits) a.logits[(size_t)tok * a.V + fg] = v;
          const unsigned long long k = argmax_key(v, fg);
          best = k > best ? k : best;
        }
      }
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const unsigned long long k = __shfl_xor_sync(0xffffffffu, best, o);
      best = k > best ? k : best;
    }
    if (valid && p == 0 && best) atomicMax(a.keys + tok, best);
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Per-unit stream trace (LaGemmArgs::utrace): compiled in only with
// -DLA_GEMM_UTRACE (LA_NVCC_DEFS=-DLA_GEMM_UTRACE python -m ..._build --force):
// its checks inside the producer / MMA loops cost ~2.5 % of a decode step
#ifdef LA_GEMM_UTRACE
#define LA_UT(cond, idx)                                         \
  do {                                                           \
    if (args.utrace && (cond)) args.utrace[idx] = globaltimer(); \
  } while (0)
#else
#define LA_UT(cond, idx) \
  do {                   \
  } while (0)
#endif

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    la_gemm_kernel(const LaGemmArgs args) {
  const unsigned long long t_entry = args.trace ? globaltimer() : 0ull;   // trace: CTA start
  extern __shared__ uint8_t smem_raw[];
  const FwdPlan* P = args.plan;
  uint8_t* sm = smem_raw + ((1024 - (ptx::smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = sm;
  // one 192 KB ring: nst stages of (weights a_bytes | step rows 16 KB), the
  // weight and row halves in two contiguous regions (1024-B aligned)
  constexpr bool multi = EPI == LA_EPI_MULTI;        // prefill: row blocks per weight stage
  // decode split-K pieces: accumulate (step rows x weight rows) -- see the MMA issuer
  constexpr bool nt = EPI == LA_EPI_PARTIAL;
  const int nblk = multi ? args.nblk : 1;
  const int nbuf = nblk > 2 ? 1 : 2;                 // TMEM accumulator buffers
  const int nst = args.nst > 0 ? args.nst : multi ? (nblk > 2 ? 2 : kStages)
                                                  : (args.tpc == LA_TPC ? kStages : kMaxStages);
  const uint32_t a_stage = (uint32_t)args.tpc * kTileBytes;
  const uint32_t b_stage = (uint32_t)nblk * kBBytes;
  uint8_t* sB = sA + nst * a_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sA + nst * (a_stage + b_stage));
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* fxbar = tempty + 2;                     // fix-up staging (LA_EPI_FX_*)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fxbar + 1);
  int* sflag = reinterpret_cast<int*>(tmem_slot + 1);
  // (pointer + offset, not an integer round trip: keeps the shared address
  // space visible to the compiler -- STS/LDS instead of generic ST/LD)
  uint8_t* epi_base = reinterpret_cast<uint8_t*>(tmem_slot) + 16;
  float* sEpi = reinterpret_cast<float*>(epi_base + ((128 - (ptx::smem_u32(epi_base) & 127)) & 127));
  float* sRstd = sEpi + kStageFloats;   // fused epilogues: per-row deferred-norm scale

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = args.kb;
  const int tpc = args.tpc;
  const int n_units_t = args.n_tiles / tpc;      // unit tiles (pairs when tpc == 2)
  const long U = (long)n_units_t * kb;
  const long Pn = gridDim.x;
  const long u_begin = (long)blockIdx.x * U / Pn;
  const long u_end = (long)(blockIdx.x + 1) * U / Pn;
  const int n_pre = (int)min((long)nst, u_end - u_begin);
  // weight block of unit u: packed tiles are pair-interleaved per k-block, so
  // a 2-tile unit is one 32 KB copy and a 1-tile unit one 16 KB copy
  const uint32_t a_bytes = (uint32_t)tpc * kTileBytes;
  auto a_src = [&](long u) -> const __nv_bfloat16* {
    if (tpc == LA_TPC) return args.a + (size_t)u * (kABytes / 2);
    const long t = u / kb, k = u % kb;
    return args.a + ((size_t)((t / LA_TPC) * kb + k) * LA_TPC + (t % LA_TPC)) * (kTileBytes / 2);
  };
  // PDL: the weights do not depend on the previous kernel, so the first
  // stages' weight tiles stream in while the previous kernel drains -- issued
  // right after the barrier init, overlapping warp 1's TMEM allocation
  la_pdl_trigger();
  uint64_t pol_w = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&tfull[b], 1); ptx::mbar_init(&tempty[b], 128); }
    ptx::mbar_init(fxbar, 1);
    ptx::fence_barrier_init();
    pol_w = ptx::policy_evict_first();   // weights: streamed once
    for (int i = 0; i < n_pre; ++i) {
      ptx::mbar_expect_tx_noarrive(&full[i], a_bytes);
      ptx::bulk_load(sA + i * a_stage, a_src(u_begin + i), a_bytes, &full[i], pol_w);
    }
    LA_UT(true, (gridDim.x + blockIdx.x) * 32 + 31);
  }
  if (warp == 1) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0 && lane == 0 && args.l2pf > 0) {
    // keep HBM streaming while the previous kernel finishes: the units just
    // beyond the smem ring go to L2 (a cache hint, always safe)
    for (long u = u_begin + n_pre; u < min(u_end, u_begin + n_pre + args.l2pf); ++u)
      ptx::bulk_prefetch_l2(a_src(u), a_bytes);
  }
  la_pdl_wait();
  if (args.timing && threadIdx.x == 0) {
    if (atomicAdd(&args.timing[3], 1ull) == 0ull) args.timing[0] = globaltimer();
  }
  // trace: [0] CTA entry (before the dependency wait), [1] wait returned
  if (args.trace && threadIdx.x == 0) {
    args.trace[blockIdx.x * 8 + 0] = t_entry;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (!is_fx(EPI)) args.trace[blockIdx.x * 8 + 5] = smid;   // (fix-up slot unused)
  }
  const int n_rows = P->n_rows;
  const int n_pad = P->n_pad;
  int n_rows_x[3] = {0, 0, 0}, n_pad_x[3] = {0, 0, 0};
  if constexpr (multi)
    for (int j = 1; j < nblk; ++j) { n_rows_x[j - 1] = args.planx[j - 1]->n_rows; n_pad_x[j - 1] = args.planx[j - 1]->n_pad; }
  if (args.trace && threadIdx.x == 0) args.trace[blockIdx.x * 8 + 1] = globaltimer();

  if (n_rows == 0) {
    // decode finished: drain the prefetched weight tiles before exiting
    if (warp == 0 && lane == 0)
      for (int i = 0; i < n_pre; ++i) {
        ptx::mbar_arrive(&full[i]);
        ptx::mbar_wait(&full[i], 0);
      }
    // the epilogue counts every launch's contributions: count the empty pieces in
    if (args.ready && threadIdx.x == 0)
      for (long u = u_begin; u < u_end; u = ((u / kb) + 1) * kb) atomicAdd(args.ready + (int)(u / kb), 1);
  } else if (warp == 0) {
    // --------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol_x = ptx::policy_evict_last();    // step rows: re-read by every CTA
      uint32_t bbytes_all = (uint32_t)n_pad * 128;
      if constexpr (multi)
        for (int j = 1; j < nblk; ++j) bbytes_all += (uint32_t)n_pad_x[j - 1] * 128;
      const uint32_t bbytes = (uint32_t)n_pad * 128;
      long it = 0;
      for (long u = u_begin; u < u_end; ++u, ++it) {
        const int k = (int)(u % kb);
        const int s = (int)(it % nst);
        const uint32_t r = (uint32_t)(it / nst);
        const bool load_b = !(args.debug & 1);
        const uint32_t bb = load_b ? bbytes_all : 0;
        if (it < n_pre) {
          ptx::mbar_expect_tx(&full[s], bb);   // weights already in flight
        } else {
          ptx::mbar_wait(&empty[s], (r - 1) & 1);
          ptx::mbar_expect_tx(&full[s], a_bytes + bb);
          ptx::bulk_load(sA + s * a_stage, a_src(u), a_bytes, &full[s], pol_w);
        }
        LA_UT(it < 24, (gridDim.x + blockIdx.x) * 32 + it);
        if (load_b) {
          ptx::bulk_load(sB + s * b_stage, args.b + (size_t)k * (kBBytes / 2), bbytes, &full[s], pol_x);
          if constexpr (multi)
            for (int j = 1; j < nblk; ++j)
              ptx::bulk_load(sB + s * b_stage + j * kBBytes, args.bx[j - 1] + (size_t)k * (kBBytes / 2),
                             (uint32_t)n_pad_x[j - 1] * 128, &full[s], pol_x);
        }
      }
      // every load of this CTA is issued: stream the following GEMMs' first
      // units into L2 while the kernels between them run
#pragma unroll 1
      for (int j = 0; j < 2; ++j) {
        const LaNextPf& q = args.npf[j];
        if (!q.a || q.units <= 0) continue;
        const long Uq = (long)(q.n_tiles / q.tpc) * q.kb, Pq = q.grid;
        for (long c = blockIdx.x; c < Pq; c += gridDim.x) {
          const long v0 = c * Uq / Pq, v1 = (c + 1) * Uq / Pq;
          for (long v = v0 + q.skip; v < min(v1, v0 + q.skip + q.units); ++v) {
            const char* base = reinterpret_cast<const char*>(q.a);
            if (q.tpc == LA_TPC) {
              ptx::bulk_prefetch_l2(base + (size_t)v * kABytes, kABytes);
            } else {
              const long t = v / q.kb, k = v % q.kb;
              ptx::bulk_prefetch_l2(base + ((size_t)((t / LA_TPC) * q.kb + k) * LA_TPC + (t % LA_TPC)) * kTileBytes,
                                    kTileBytes);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = nt ? ptx::umma_idesc_bf16(128, (uint32_t)(128 * tpc)) : ptx::umma_idesc_bf16(128, (uint32_t)n_pad);
      uint32_t idesc_x[3] = {0u, 0u, 0u};
      if constexpr (multi)
        for (int j = 0; j < 3; ++j) idesc_x[j] = ptx::umma_idesc_bf16(128, (uint32_t)(n_pad_x[j] > 0 ? n_pad_x[j] : 16));
      long it = 0, u = u_begin;
      int use[2] = {0, 0}, buf = 0;
      while (u < u_end) {
        const int tile = (int)(u / kb);
        const long seg_start = u, seg_end = std::min(u_end, (long)(tile + 1) * kb);
        if (use[buf] > 0) {
          ptx::mbar_wait(&tempty[buf], (use[buf] - 1) & 1);
          ptx::tc_fence_after();
        }
        const uint32_t d_tmem = tmem + buf * (LA_TPC * 128);   // TMEM sized for LA_TPC (single buffer: buf = 0)
        for (; u < seg_end; ++u, ++it) {
          const int s = (int)(it % nst);
          ptx::mbar_wait(&full[s], (uint32_t)(it / nst) & 1);
#ifdef LA_GEMM_UTRACE
          {   // first 24 units, then the last 8
            const long nu = u_end - u_begin;
            const long slot = it < 24 ? it : it >= nu - 8 ? 24 + (it - (nu - 8)) : -1;
            LA_UT(slot >= 0, blockIdx.x * 32 + slot);
          }
#endif
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sA + s * a_stage);
          const uint32_t b_addr = ptx::smem_u32(sB + s * b_stage);
          if (args.debug & 2) {
            ptx::mbar_arrive(&empty[s]);
            continue;
          }
          if constexpr (nt) {
            // step rows x weight rows: A = the step rows' k-block (M = 128
            // lanes; rows >= n_pad hold stale data and are never read back),
            // B = the unit's tpc contiguous weight tiles (N = 128 tpc), so a
            // unit is 4 MMAs instead of 4 tpc (the tensor core's per-MMA cost
            // hardly depends on N at these sizes: profiles/microbench/mma_rate.cu)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              ptx::umma_bf16(d_tmem, ptx::umma_desc_sw128(b_addr + kk * 32), ptx::umma_desc_sw128(a_addr + kk * 32),
                             idesc, (u > seg_start || kk > 0) ? 1u : 0u);
          } else {
            for (int tt = 0; tt < tpc; ++tt)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                ptx::umma_bf16(d_tmem + tt * 128, ptx::umma_desc_sw128(a_addr + tt * kTileBytes + kk * 32),
                               ptx::umma_desc_sw128(b_addr + kk * 32), idesc,
                               (u > seg_start || kk > 0) ? 1u : 0u);
          }
          if constexpr (multi)
          for (int j = 1; j < nblk; ++j)   // row block j into columns [128 j, 128 j + 128)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              ptx::umma_bf16(d_tmem + 128 * j, ptx::umma_desc_sw128(a_addr + kk * 32),
                             ptx::umma_desc_sw128(b_addr + j * kBBytes + kk * 32), idesc_x[j - 1],
                             (u > seg_start || kk > 0) ? 1u : 0u);
          ptx::umma_commit(&empty[s]);
          LA_UT(it < 24, (2 * gridDim.x + blockIdx.x) * 32 + it);
        }
        ptx::umma_commit(&tfull[buf]);
        use[buf]++;
        buf = nbuf == 2 ? buf ^ 1 : 0;
      }
      if (args.trace) args.trace[blockIdx.x * 8 + 2] = globaltimer();
    }
  } else {
    // ------------------------------------------- drain TMEM / epilogue
    const int et = threadIdx.x - 64;              // 0..127
    const int row_base = 32 * (warp & 3);
    const int f = row_base + lane;                // accumulator lane = feature in tile
    int use[2] = {0, 0}, buf = 0;
    long u = u_begin;
    while (u < u_end) {
      const int tile = (int)(u / kb);             // unit tile
      const long seg_end = std::min(u_end, (long)(tile + 1) * kb);
      const long c_first = la_cta_of((long)tile * kb, U, Pn);
      const int seg = (int)(blockIdx.x - c_first);
      ptx::mbar_wait(&tfull[buf], use[buf] & 1);
      ptx::tc_fence_after();
#ifdef LA_GEMM_UTRACE
      const int dseg = use[0] + use[1];
#endif
      LA_UT(et == 128 - 64 && dseg < 4, (2 * gridDim.x + blockIdx.x) * 32 + 24 + 2 * dseg);   // warp 4: drain start
      if constexpr (nt) {
        // lane = step row, columns = the unit's 128 tpc features: each thread
        // writes its row's 32-feature runs (128 B) of the piece
        const int q4 = warp & 3;   // lanes 32 q4 .. 32 q4 + 31 = step rows
        if (32 * q4 < n_rows) {
          // transpose each 32 x 32 block through the warp's smem slice so a
          // store instruction writes one row's 32 features (128 B, coalesced)
          // (rows 36 floats apart: 16-B aligned, conflict-free float4 writes
          // and reads); a store instruction then covers 4 rows x 128 B
          float* tw = sEpi + q4 * 32 * 36;
          const int rr = lane >> 3, cc = (lane & 7) * 4;
          for (int tt = 0; tt < tpc; ++tt) {
            float* wsp = args.ws + ((size_t)(tile * tpc + tt) * args.max_segs + seg) * 128 * 128;
            const uint32_t t_base = tmem + ((uint32_t)row_base << 16) + buf * (LA_TPC * 128) + tt * 128;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              const int c0 = 32 * c;
              uint32_t v[32];
              ptx::tmem_ld32_nowait(t_base + c0, v);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int q = 0; q < 8; ++q)
                *reinterpret_cast<uint4*>(tw + lane * 36 + 4 * q) = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
              __syncwarp();
#pragma unroll
              for (int p = 0; p < 8; ++p) {
                const int i = 4 * p + rr;
                const int row = 32 * q4 + i;
                if (row < n_rows && !(args.debug & 4))
                  __stcg(reinterpret_cast<float4*>(wsp + (size_t)row * 128 + c0 + cc),
                         *reinterpret_cast<const float4*>(tw + i * 36 + cc));
              }
              __syncwarp();
            }
          }
        }
        LA_UT(et == 128 - 64 && dseg < 4, (2 * gridDim.x + blockIdx.x) * 32 + 25 + 2 * dseg);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[buf]);
        if (args.ready) {
          // this unit tile's piece is written: release it to the epilogue kernel
          ptx::named_bar_sync(1, 128);
          if (et == 0) {
            __threadfence();
            atomicAdd(args.ready + tile, 1);
          }
        }
      } else if (EPI == LA_EPI_PARTIAL_SW || multi || is_fx(EPI) || seg != 0) {
        // write this piece's fp32 partial (multi-chunk mode: every row block)
        const int nout = multi ? nblk : tpc;
        for (int tt = 0; tt < nout; ++tt) {
          const uint32_t t_base = tmem + ((uint32_t)row_base << 16) + buf * (LA_TPC * 128) + tt * 128;
          const int ftile = multi ? tile : tile * tpc + tt;
          float* wsp = (multi && tt ? args.wsx[tt - 1] : args.ws) + ((size_t)ftile * args.max_segs + seg) * 128 * 128 + f;
          const int nr = multi && tt ? n_rows_x[tt - 1] : n_rows, np = multi && tt ? n_pad_x[tt - 1] : n_pad;
          for (int c0 = 0; c0 < np; c0 += 32) {
            float v[32];
            ptx::tmem_ld32(t_base + c0, v);
            const int nj = min(32, nr - c0);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (jj < nj) __stcg(wsp + (size_t)(c0 + jj) * 128, v[jj]);
          }
        }
        LA_UT(et == 128 - 64 && dseg < 4, (2 * gridDim.x + blockIdx.x) * 32 + 25 + 2 * dseg);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[buf]);
        if constexpr (is_fx(EPI)) {
          // this piece is complete: count it in for the unit tile's fix-up
          // (one cumulative fence by the signalling thread after the barrier;
          // a fence per thread stalls the drain -- and so the MMAs -- mid-stream)
          ptx::named_bar_sync(1, 128);
          if (et == 0) {
            __threadfence();
            atomicAdd(args.fx_arrive + tile, 1);
          }
        } else if (EPI == LA_EPI_PARTIAL_SW && args.ready) {
          // this unit tile's piece is written: release it to the epilogue kernel
          ptx::named_bar_sync(1, 128);
          if (et == 0) {
            __threadfence();
            atomicAdd(args.ready + tile, 1);
          }
        } else if (EPI != LA_EPI_PARTIAL_SW && !multi) {
          ptx::named_bar_sync(1, 128);
          if (et == 0) {
            __threadfence();
            atomicAdd(args.counters + tile, 1);
          }
        }
      } else if constexpr (EPI != LA_EPI_PARTIAL_SW && EPI != LA_EPI_MULTI && !is_fx(EPI)) {
        // owner of the tile's k = 0 piece: wait for the other pieces, sum them
        // in piece order onto the accumulator, apply the fused epilogue
        const int nseg = (int)(la_cta_of((long)(tile + 1) * kb - 1, U, Pn) - c_first + 1);
        if (nseg > 1) {
          if (et == 0) {
            while (atomicAdd(args.counters + tile, 0) < nseg - 1) __nanosleep(64);
            args.counters[tile] = 0;
          }
          ptx::named_bar_sync(1, 128);
          __threadfence();
        }
        if (et < n_rows) {
          float s = 0.f;
          for (int t = 0; t < args.nrm.tiles; ++t) s += __ldcg(args.nrm.ss + t * 128 + et);
          sRstd[et] = rsqrtf(s * args.nrm.inv_d + args.nrm.eps);
        }
        ptx::named_bar_sync(1, 128);
        for (int tt = 0; tt < tpc; ++tt) {
          const uint32_t t_base = tmem + ((uint32_t)row_base << 16) + buf * (LA_TPC * 128) + tt * 128;
          const int ftile = tile * tpc + tt;
          const float* wsp = args.ws + (size_t)ftile * args.max_segs * 128 * 128 + f;
          for (int c0 = 0; c0 < n_pad; c0 += 32) {
            float v[32];
            ptx::tmem_ld32(t_base + c0, v);
            const int nj = min(32, n_rows - c0);
            for (int sg = 1; sg < nseg; ++sg) {
              const float* pp = wsp + ((size_t)sg * 128 + c0) * 128;
#pragma unroll
              for (int jj = 0; jj < 32; ++jj)
                if (jj < nj) v[jj] += __ldcg(pp + (size_t)jj * 128);
            }
            // deferred RMSNorm of the projection input: scale token columns
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              sEpi[f * kEpiLd + jj] = jj < nj ? v[jj] * sRstd[c0 + jj] : 0.f;
            ptx::named_bar_sync(1, 128);
            epi_apply<EPI>(args, P, ftile, c0, n_rows, sEpi, et);
            ptx::named_bar_sync(1, 128);
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[buf]);
      }
      use[buf]++;
      buf = nbuf == 2 ? buf ^ 1 : 0;
      u = seg_end;
    }
    if (args.trace && et == 0) args.trace[blockIdx.x * 8 + 4] = globaltimer();   // last piece written
    if constexpr (is_fx(EPI)) {
      // ---- fix-up: every MMA of this CTA has completed (its last TMEM
      // buffer was drained above), so the smem ring is free for staging
      float* S = reinterpret_cast<float*>(sA);
      const uint64_t pol = ptx::policy_evict_first();
      uint32_t fx_phase = 0;
      for (long ut = u_begin / kb; ut <= (u_end - 1) / kb; ++ut) {
        long c0;
        int nseg;
        la_tile_segs((int)(ut * tpc), kb, args.n_tiles, Pn, c0, nseg, tpc);
        const int j = (int)(blockIdx.x - c0);
        const int r0 = j * n_rows / nseg, nr = (j + 1) * n_rows / nseg - r0;
        if (et == 0) {
          while (ld_acquire(args.fx_arrive + ut) < nseg) __nanosleep(32);
          if (args.trace && ut == u_begin / kb) args.trace[blockIdx.x * 8 + 5] = globaltimer();
        }
        ptx::named_bar_sync(1, 128);
        if (nr > 0) {
          if (et == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");   // generic-proxy pieces -> bulk copies
            const uint32_t bytes = (uint32_t)nr * 512;
            ptx::mbar_expect_tx(fxbar, bytes * (uint32_t)(nseg * tpc));
            for (int sg = 0; sg < nseg; ++sg)
              for (int tt = 0; tt < tpc; ++tt)
                ptx::bulk_load(S + (size_t)(sg * tpc + tt) * nr * 128,
                               args.ws + (((size_t)(ut * tpc + tt) * args.max_segs + sg) * 128 + r0) * 128,
                               bytes, fxbar, pol);
          }
          ptx::mbar_wait(fxbar, fx_phase);
          fx_phase ^= 1;
          if (args.trace && et == 0 && ut == u_begin / kb) args.trace[blockIdx.x * 8 + 6] = globaltimer();
          fx_finish<EPI>(args, P, (int)ut, r0, nr, nseg, S, et);
        }
        ptx::named_bar_sync(1, 128);   // S is restaged for the next unit tile
        if (et == 0 && atomicAdd(args.fx_depart + ut, 1) == nseg - 1) {
          // every contributor is past its wait: reset for the next launch
          args.fx_arrive[ut] = 0;
          args.fx_depart[ut] = 0;
        }
      }
      if (args.trace && et == 0) args.trace[blockIdx.x * 8 + 7] = globaltimer();
    }
  }
  if (args.trace && !is_fx(EPI)) {   // which role reaches the final barrier last
    if (threadIdx.x == 0) args.trace[blockIdx.x * 8 + 6] = globaltimer();
    if (threadIdx.x == 96) args.trace[blockIdx.x * 8 + 7] = globaltimer();
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem);
  }
  if (args.trace && threadIdx.x == 0) args.trace[blockIdx.x * 8 + 3] = globaltimer();
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

// ------------------------------------------ data-parallel + stream-K GEMM
// (LA_EPI_DPSK_SWIGLU: the gate/up projection when its 128-row tiles
// outnumber the CTAs).  CTA c owns the dpc = T / P whole tiles
// [c dpc, (c + 1) dpc) (full K in one TMEM accumulator: no split-K pieces,
// SwiGLU straight from TMEM) and first streams its stream-K share of the
// R = T - P dpc remaining tiles, whose pieces it writes and later fixes up (its
// row slice of every remainder tile it touched; those pieces were all written
// at the start of every CTA's stream, so the wait is normally already over).
// One-tile units (16 KB weights + the k-block's step rows), 6-stage ring.
// The stream-K split and the piece order depend on the shape only, so every
// row's arithmetic is the same for any row count / layout / LP shard.
__device__ __forceinline__ float dpsk_rstd(const LaRowNorm& n, int tok) {
  // the exact summation order of rstd_issue<8> / rstd_finish<8> (la_reduce_dev.cuh),
  // so a row's scale is bit-identical for whole and remainder tiles
  float p[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int t = l + 8 * i;
      v += t < n.tiles ? __ldcg(n.ss + t * 128 + tok) : 0.f;
    }
    for (int t = l + 64; t < n.tiles; t += 8) v += __ldcg(n.ss + t * 128 + tok);
    p[l] = v;
  }
  const float s = ((p[0] + p[4]) + (p[2] + p[6])) + ((p[1] + p[5]) + (p[3] + p[7]));
  return rsqrtf(s * n.inv_d + n.eps);
}

__global__ void __launch_bounds__(kThreads, 1) la_gemm_dpsk_kernel(const LaGemmArgs args) {
  const unsigned long long t_entry = args.trace ? globaltimer() : 0ull;
  // optional per-CTA trace [gridDim][8]: 0 entry, 1 wait returned, 2 last MMA
  // issued, 3 exit, 4 remainder pieces written, 5 whole tile's act written,
  // 6 fix-up pieces complete, 7 fix-up done
  auto tr = [&](int k, bool cond) {
    if (args.trace && cond) args.trace[blockIdx.x * 8 + k] = globaltimer();
  };
  extern __shared__ uint8_t smem_raw[];
  const FwdPlan* P = args.plan;
  uint8_t* sm = smem_raw + ((1024 - (ptx::smem_u32(smem_raw) & 1023)) & 1023);
  constexpr int nst = kMaxStages;
  uint8_t* sA = sm;
  uint8_t* sB = sA + nst * kTileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + nst * kBBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* fxbar = tempty + 2;
  uint64_t* tdp = fxbar + 1;                   // the whole tile's accumulators are complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tdp + 1);
  uint8_t* epi_base = reinterpret_cast<uint8_t*>(tmem_slot) + 16;
  float* sEpi = reinterpret_cast<float*>(epi_base + ((128 - (ptx::smem_u32(epi_base) & 127)) & 127));
  float* sRstd = sEpi + kStageFloats;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = args.kb;
  const int T = args.n_real;
  const int Pn = gridDim.x;
  const int dpc = T / Pn;                      // whole tiles per CTA
  const int R = T - dpc * Pn;                  // remainder tiles [dpc Pn, T)
  const long Ur = (long)R * kb;
  const long ur0 = (long)blockIdx.x * Ur / Pn, ur1 = (long)(blockIdx.x + 1) * Ur / Pn;
  const int n_rem = (int)(ur1 - ur0);
  const int n_all = n_rem + dpc * kb;
  auto unit_tile = [&](int it) -> int {
    return it < n_rem ? dpc * Pn + (int)((ur0 + it) / kb) : (int)blockIdx.x * dpc + (it - n_rem) / kb;
  };
  auto unit_k = [&](int it) -> int { return it < n_rem ? (int)((ur0 + it) % kb) : (it - n_rem) % kb; };
  auto a_src = [&](int t, int k) -> const __nv_bfloat16* {
    return args.a + ((size_t)((t / LA_TPC) * kb + k) * LA_TPC + (t % LA_TPC)) * (kTileBytes / 2);
  };
  auto seg_end_of = [&](int it) -> int {   // units of one tile are contiguous in the sequence
    const int t = unit_tile(it);
    if (it < n_rem) {
      const long tile_end = (long)(t - dpc * Pn + 1) * kb;   // remainder-space end of tile t
      return (int)(min(ur1, tile_end) - ur0);
    }
    return n_rem + ((it - n_rem) / kb + 1) * kb;
  };
  const int n_pre = min(nst, n_all);
  la_pdl_trigger();
  uint64_t pol_w = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&tfull[b], 1); ptx::mbar_init(&tempty[b], 128); }
    ptx::mbar_init(fxbar, 1);
    ptx::mbar_init(tdp, 1);
    ptx::fence_barrier_init();
    pol_w = ptx::policy_evict_first();
    for (int i = 0; i < n_pre; ++i) {
      ptx::mbar_expect_tx_noarrive(&full[i], kTileBytes);
      ptx::bulk_load(sA + i * kTileBytes, a_src(unit_tile(i), unit_k(i)), kTileBytes, &full[i], pol_w);
    }
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  la_pdl_wait();
  if (args.timing && threadIdx.x == 0) {
    if (atomicAdd(&args.timing[3], 1ull) == 0ull) args.timing[0] = globaltimer();
  }
  if (args.trace && threadIdx.x == 0) args.trace[blockIdx.x * 8 + 0] = t_entry;
  tr(1, threadIdx.x == 0);
  const int n_rows = P->n_rows;
  const int n_pad = P->n_pad;
  // TMEM: columns [0, 256) = two buffers for the remainder segments, [256, 512)
  // = the whole tile's two accumulators (even / odd k-blocks: two independent
  // MMA chains keep the tensor pipe busy; summed even + odd in the epilogue)
  const uint32_t dp_acc = tmem + 256;

  if (n_rows == 0) {
    if (warp == 0 && lane == 0)
      for (int i = 0; i < n_pre; ++i) {
        ptx::mbar_arrive(&full[i]);
        ptx::mbar_wait(&full[i], 0);
      }
  } else if (warp == 0) {
    // --------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol_x = ptx::policy_evict_last();
      const uint32_t bbytes = (uint32_t)n_pad * 128;
      for (int it = 0; it < n_all; ++it) {
        const int s = it % nst;
        const uint32_t r = (uint32_t)(it / nst);
        const int t = unit_tile(it), k = unit_k(it);
        if (it < n_pre) {
          ptx::mbar_expect_tx(&full[s], bbytes);
        } else {
          ptx::mbar_wait(&empty[s], (r - 1) & 1);
          ptx::mbar_expect_tx(&full[s], kTileBytes + bbytes);
          ptx::bulk_load(sA + s * kTileBytes, a_src(t, k), kTileBytes, &full[s], pol_w);
        }
        ptx::bulk_load(sB + s * kBBytes, args.b + (size_t)k * (kBBytes / 2), bbytes, &full[s], pol_x);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = ptx::umma_idesc_bf16(128, (uint32_t)n_pad);
      int use[2] = {0, 0}, buf = 0;
      for (int it = 0; it < n_all;) {
        const int first = it, end = seg_end_of(it);
        const bool whole = it >= n_rem;
        if (!whole && use[buf] > 0) {
          ptx::mbar_wait(&tempty[buf], (use[buf] - 1) & 1);
          ptx::tc_fence_after();
        }
        for (; it < end; ++it) {
          const int s = it % nst;
          ptx::mbar_wait(&full[s], (uint32_t)(it / nst) & 1);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sA + s * kTileBytes);
          const uint32_t b_addr = ptx::smem_u32(sB + s * kBBytes);
          const int q = it - first;
          const uint32_t d_tmem = whole ? dp_acc + (q & 1) * 128 : tmem + buf * 128;
          const bool acc = whole ? q >= 2 : q > 0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::umma_bf16(d_tmem, ptx::umma_desc_sw128(a_addr + kk * 32), ptx::umma_desc_sw128(b_addr + kk * 32),
                           idesc, (acc || kk > 0) ? 1u : 0u);
          ptx::umma_commit(&empty[s]);
        }
        ptx::umma_commit(whole ? tdp : &tfull[buf]);
        tr(2, whole);
        if (!whole) {
          use[buf]++;
          buf ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------- drain TMEM / epilogue
    const int et = threadIdx.x - 64;              // 0..127
    const int row_base = 32 * (warp & 3);
    const int f = row_base + lane;                // accumulator lane = feature in tile
    if (et < n_rows) sRstd[et] = dpsk_rstd(args.nrm, et);
    ptx::named_bar_sync(1, 128);
    int use[2] = {0, 0}, buf = 0;
    for (int it = 0; it < n_all;) {
      const int tile = unit_tile(it), end = seg_end_of(it);
      const bool whole = it >= n_rem;
      if (whole) ptx::mbar_wait(tdp, 0);
      else ptx::mbar_wait(&tfull[buf], use[buf] & 1);
      ptx::tc_fence_after();
      const uint32_t t_base = tmem + ((uint32_t)row_base << 16) + buf * 128;
      if (!whole) {
        // remainder piece of tile `tile`: its contributor index = piece order
        const long c_first = la_cta_of((long)(tile - dpc * Pn) * kb, Ur, Pn);
        const int seg = (int)(blockIdx.x - c_first);
        float* wsp = args.ws + ((size_t)tile * args.max_segs + seg) * 128 * 128 + f;
        for (int c0 = 0; c0 < n_pad; c0 += 32) {
          float v[32];
          ptx::tmem_ld32(t_base + c0, v);
          const int nj = min(32, n_rows - c0);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            if (jj < nj) __stcg(wsp + (size_t)(c0 + jj) * 128, v[jj]);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[buf]);
        use[buf]++;
        buf ^= 1;
        ptx::named_bar_sync(1, 128);
        if (et == 0) {
          __threadfence();
          atomicAdd(args.fx_arrive + tile, 1);
        }
        tr(4, et == 0);
      } else {
        // whole tile: even + odd accumulators, deferred-norm scale, SwiGLU,
        // act -- straight from TMEM
        const uint32_t e_base = dp_acc + ((uint32_t)row_base << 16);
        for (int c0 = 0; c0 < n_pad; c0 += 32) {
          float v[32], w[32];
          ptx::tmem_ld32(e_base + c0, v);
          ptx::tmem_ld32(e_base + 128 + c0, w);
          const int nj = min(32, n_rows - c0);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) sEpi[f * kEpiLd + jj] = jj < nj ? (v[jj] + w[jj]) * sRstd[c0 + jj] : 0.f;
          ptx::named_bar_sync(1, 128);
          epi_apply<LA_EPI_SWIGLU>(args, P, tile, c0, n_rows, sEpi, et);
          ptx::named_bar_sync(1, 128);
        }
        tr(5, et == 0);
      }
      it = end;
    }
    // ---- fix-up of this CTA's row slice of every remainder tile it touched
    // (every MMA of this CTA has completed: the ring is free for staging)
    float* S = reinterpret_cast<float*>(sA);
    const uint64_t pol = ptx::policy_evict_first();
    uint32_t fx_phase = 0;
    for (int it = 0; it < n_rem;) {
      const int tile = unit_tile(it), end = seg_end_of(it);
      it = end;
      long c0;
      int nseg;
      la_tile_segs(tile - dpc * Pn, kb, R, Pn, c0, nseg, 1);
      const int j = (int)(blockIdx.x - c0);
      const int r0 = j * n_rows / nseg, nr = (j + 1) * n_rows / nseg - r0;
      if (et == 0)
        while (ld_acquire(args.fx_arrive + tile) < nseg) __nanosleep(32);
      tr(6, et == 0);
      ptx::named_bar_sync(1, 128);
      if (nr > 0) {
        if (et == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");   // generic-proxy pieces -> bulk copies
          const uint32_t bytes = (uint32_t)nr * 512;
          ptx::mbar_expect_tx(fxbar, bytes * (uint32_t)nseg);
          for (int sg = 0; sg < nseg; ++sg)
            ptx::bulk_load(S + (size_t)sg * nr * 128, args.ws + (((size_t)tile * args.max_segs + sg) * 128 + r0) * 128,
                           bytes, fxbar, pol);
        }
        ptx::mbar_wait(fxbar, fx_phase);
        fx_phase ^= 1;
        fx_finish<LA_EPI_FX_SWIGLU>(args, P, tile, r0, nr, nseg, S, et);
      }
      ptx::named_bar_sync(1, 128);   // S is restaged for the next tile
      if (et == 0 && atomicAdd(args.fx_depart + tile, 1) == nseg - 1) {
        args.fx_arrive[tile] = 0;    // every contributor is past its wait: reset for the next launch
        args.fx_depart[tile] = 0;
      }
    }
    tr(7, et == 0);
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  tr(3, threadIdx.x == 0);
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

size_t la_packed_elems(int rows, int K) {
  const int tiles = ((rows + 127) / 128 + LA_TPC - 1) / LA_TPC * LA_TPC;
  return (size_t)tiles * (K / 64) * 128 * 64;
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

// the fix-up stages nseg pieces x tpc tiles x ceil(rows / nseg) rows of 512 B
// in the smem ring: check the worst case (128 rows) against the ring
bool la_gemm_fx_fits(const LaGemm& g) {
  const int tpc = g.args.tpc;
  const int nst = g.args.nst > 0 ? g.args.nst : (tpc == LA_TPC ? kStages : kMaxStages);
  const size_t ring = (size_t)nst * (tpc * kTileBytes + kBBytes);
  const int U = g.args.n_tiles / tpc;
  for (int ut = 0; ut < U; ++ut) {
    long c0;
    int n;
    la_tile_segs(ut * tpc, g.args.kb, g.args.n_tiles, g.grid, c0, n, tpc);
    const size_t need = (size_t)n * tpc * ((LA_MAX_ROWS + n - 1) / n) * 512;
    if (need > ring) return false;
  }
  return true;
}

// LA_EPI_DPSK_SWIGLU geometry: pieces per remainder tile (0: not applicable,
// fewer real tiles than CTAs); the remainder fix-up stages nseg slices of
// ceil(128 / nseg) rows in the ring
int la_gemm_dpsk_segs(int n_real, int kb, int grid) {
  const int dpc = n_real / grid, R = n_real - dpc * grid;
  if (dpc != 1) return 0;   // one whole tile per CTA (its accumulator pair is not double-buffered)
  if (R == 0) return 1;
  if ((long)R * kb < grid) return 0;   // every CTA needs a remainder unit: the piece count of a tile
                                       // is the CTA span of its units (la_tile_segs)
  const int mx = la_gemm_workspace_segs(R, kb, grid, 1);
  const size_t ring = (size_t)kMaxStages * (kTileBytes + kBBytes);
  if ((size_t)mx * ((LA_MAX_ROWS + mx - 1) / mx) * 512 > ring) return 0;
  return mx;
}

int la_gemm_workspace_segs(int n_tiles, int kb, int grid, int tpc) {
  long mx = 1;
  for (int t = 0; t < n_tiles; ++t) {
    long c0;
    int n;
    la_tile_segs(t, kb, n_tiles, grid, c0, n, tpc);
    mx = std::max<long>(mx, n);
  }
  return (int)mx;
}

template <int EPI>
static cudaError_t launch_epi(const LaGemm& g, cudaStream_t st, bool pdl) {
  static std::atomic<unsigned> attr{0};
  {
    cudaError_t e = la_smem_attr_once(attr, la_gemm_kernel<EPI>, (int)kSmemBytes);
    if (e != cudaSuccess) return e;
  }
  // the ring (nst stages), barriers / TMEM slot, and the fused epilogue's staging
  const int nblk = g.args.nblk > 1 ? g.args.nblk : 1;
  const int nst = g.args.nst > 0 ? g.args.nst : nblk > 1 ? (nblk > 2 ? 2 : kStages)
                                                         : (g.args.tpc == LA_TPC ? kStages : kMaxStages);
  const size_t smem = 1024 + (size_t)nst * (g.args.tpc * kTileBytes + nblk * kBBytes) + 2 * kMaxStages * 8 +
                      5 * 8 + 16 +
                      (EPI == LA_EPI_MULTI || EPI == LA_EPI_PARTIAL_SW || is_fx(EPI) ? 0 : 128 + kStageFloats * 4 + 128 * 4);
  return la_launch(la_gemm_kernel<EPI>, dim3(g.grid), dim3(kThreads), smem, st, pdl, g.args);
}

static cudaError_t launch_dpsk(const LaGemm& g, cudaStream_t st, bool pdl) {
  const size_t smem = 1024 + (size_t)kMaxStages * (kTileBytes + kBBytes) + 2 * kMaxStages * 8 + 6 * 8 + 16 + 128 +
                      kStageFloats * 4 + 128 * 4;
  static std::atomic<unsigned> attr{0};
  cudaError_t e = la_smem_attr_once(attr, la_gemm_dpsk_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  return la_launch(la_gemm_dpsk_kernel, dim3(g.grid), dim3(kThreads), smem, st, pdl, g.args);
}

int la_gemm_launch(const LaGemm& g, cudaStream_t st, bool pdl) {
  cudaError_t e;
  switch (g.epi) {
    case LA_EPI_DPSK_SWIGLU: e = launch_dpsk(g, st, pdl); break;
    case LA_EPI_QKV: e = launch_epi<LA_EPI_QKV>(g, st, pdl); break;
    case LA_EPI_SWIGLU: e = launch_epi<LA_EPI_SWIGLU>(g, st, pdl); break;
    case LA_EPI_LOGITS: e = launch_epi<LA_EPI_LOGITS>(g, st, pdl); break;
    case LA_EPI_FX_QKV: e = launch_epi<LA_EPI_FX_QKV>(g, st, pdl); break;
    case LA_EPI_FX_SWIGLU: e = launch_epi<LA_EPI_FX_SWIGLU>(g, st, pdl); break;
    case LA_EPI_FX_RESID: e = launch_epi<LA_EPI_FX_RESID>(g, st, pdl); break;
    case LA_EPI_PARTIAL_SW: e = launch_epi<LA_EPI_PARTIAL_SW>(g, st, pdl); break;
    default: e = g.args.nblk > 1 ? launch_epi<LA_EPI_MULTI>(g, st, pdl) : launch_epi<LA_EPI_PARTIAL>(g, st, pdl); break;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) { la_set_error("gemm launch: %s", cudaGetErrorString(e)); return LA_ERR_CUDA; }
  return LA_OK;
}

// ---------------------------------------------------------------- packing
// Packed "LA tile" layout: matrix rows grouped in 128-row tiles (tile count
// rounded up to LA_TPC), K in 64-wide blocks; block (t, kb) is 16 KB at
// (((t / LA_TPC) * KB + kb) * LA_TPC + t % LA_TPC) * 8192 elements -- the
// LA_TPC tiles of one stream-K unit are adjacent -- holding
// rows r = 0..127 as 128-byte lines with 16-byte chunk c stored at chunk
// position c ^ (r & 7) -- exactly the SWIZZLE_128B shared-memory image the
// UMMA descriptor expects, so a 1-D bulk copy lands it ready to multiply.
// mode 0: virtual row = row_offset + r; 1: gate row r -> (r/64)*128 + r%64;
// 2: up row r -> (r/64)*128 + 64 + r%64 (gate/up interleaved per tile).
__global__ void la_pack_kernel(const __nv_bfloat16* __restrict__ src, int rows, int K,
                               __nv_bfloat16* __restrict__ dst, int mode, int row_offset) {
  const int chunks = K / 8;
  const long total = (long)rows * chunks;
  const int KB = K / 64;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / chunks), c = (int)(i % chunks);
    int vr;
    if (mode == 0) vr = row_offset + r;
    else if (mode == 1) vr = (r / 64) * 128 + (r % 64);
    else vr = (r / 64) * 128 + 64 + (r % 64);
    const int t = vr / 128, rr = vr % 128, kb = c / 8, cc = c % 8;
    const size_t blk = ((size_t)(t / LA_TPC) * KB + kb) * LA_TPC + (t % LA_TPC);
    const size_t off = blk * 8192 + (size_t)rr * 64 + ((cc ^ (rr & 7)) * 8);
    *reinterpret_cast<uint4*>(dst + off) = *reinterpret_cast<const uint4*>(src + (size_t)r * K + c * 8);
  }
}

extern "C" int64_t la_packed_bytes(int32_t rows, int32_t K) {
  if (rows < 1 || K < 64 || K % 64) return -1;
  return (int64_t)la_packed_elems(rows, K) * 2;
}

extern "C" int32_t la_pack_weight(const void* src, int32_t rows, int32_t K, void* dst, int32_t mode,
                                  int32_t row_offset, void* stream) {
  if (!src || !dst || rows < 1 || K < 64 || K % 64 || mode < 0 || mode > 2 || row_offset < 0 ||
      (mode && rows % 64)) {
    la_set_error("la_pack_weight: bad arguments (K %% 64 == 0; gate/up rows %% 64 == 0)");
    return LA_ERR_INVALID_CONFIG;
  }
  long total = (long)rows * (K / 8);
  int grid = (int)std::min<long>(4096, (total + 255) / 256);
  la_pack_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(src), rows, K, reinterpret_cast<__nv_bfloat16*>(dst),
      mode, row_offset);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { la_set_error("pack launch: %s", cudaGetErrorString(e)); return LA_ERR_CUDA; }
  return LA_OK;
}

LA_TL_DEFINE_SETTER(gemm)
