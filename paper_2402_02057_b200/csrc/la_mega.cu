// Persistent whole-forward kernel of the bf16 lookahead step (see la_mega.cuh
// for the warp roles).  Reference semantics: one next-token distribution per
// query row (models.py:80-89) of a Llama-family decoder restated from the
// reference model contract (models.py:244-271: embed -> blocks -> final norm
// -> unembedding), greedy argmax with ties to the lowest id (sampling.py:17-19).
//
// Correctness of the dataflow (why no grid barrier is needed):
//  * every tile's split-K fix-up is done by the last CTA to finish a piece of
//    it; pieces are summed in piece order, so results are deterministic and
//    independent of arrival order and of the step layout / LP shard;
//  * a consumer waits only for the producing tiles it reads (per 128-feature
//    tile readiness counters; attention per KV head);
//  * every buffer is rewritten only by a phase that transitively depends on
//    every tile of the phase that read it, and the smem ring
//    of the activation operand is lent to the attention units only between
//    the CTA's last QKV MMA and its first O-projection load.
// Counters are monotonic across launches: a launch's targets are offset by
// the generation `gen` (completed launches), read once at entry.
#include <cuda_bf16.h>

#include "../../include/lookahead_b200.h"
#include "la_mega.cuh"
#include "la_ptx.cuh"

namespace {

constexpr int kThreads = 352;        // 11 warps
constexpr int kAStages = 8;          // 128 KB of weights in flight per SM
constexpr int kBStages = 4;
constexpr int kTile = 16384;         // bytes of one 128 x 64 bf16 weight tile
constexpr int kAStage = kTile;       // one tile per stream-K unit
constexpr int kBStage = 16384;       // <= 128 rows x 64 bf16
constexpr int kEpiLd = 33;
constexpr int kKeyTile = 64;
constexpr float kLog2e = 1.4426950408889634f;
constexpr unsigned kSpinLimit = 1u << 24;
constexpr int kSlices = 4;           // reduction slices (32 tokens) per 128-feature tile

constexpr size_t kOffA = 0;
constexpr size_t kOffB = kOffA + (size_t)kAStages * kAStage;
constexpr size_t kOffEpi = kOffB + (size_t)kBStages * kBStage;
constexpr size_t kOffBar = kOffEpi + 128 * kEpiLd * 4;
constexpr int kNumBars = 2 * kAStages + 2 * kBStages + 2 + 2;
constexpr size_t kOffMisc = kOffBar + 32 * 8;
constexpr size_t kOffRstd = kOffMisc + 64;
constexpr size_t kSmemBytes = 1024 + kOffRstd + 128 * 4;
static_assert(kNumBars <= 32, "barrier area");
static_assert(2 * 2 * kKeyTile * 256 <= kBStages * kBStage, "attention K/V stages live in the B ring");

// ------------------------------------------------------------ primitives
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// spin until *p - target >= 0 (wrapping); a timeout flags the launch as
// failed and proceeds (garbage results, but the GPU is never hung)
__device__ __forceinline__ void wait_ge(const unsigned* p, unsigned target, unsigned* err) {
  unsigned n = 0;
  while ((int)(ld_acquire(p) - target) < 0) {
    if (++n > kSpinLimit) { atomicExch(err, 1u); return; }
    if ((n & 255u) == 0 && *reinterpret_cast<volatile unsigned*>(err)) return;
    __nanosleep(32);
  }
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (uint32_t)(0x7fffffff - idx);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// [rows][128] bf16 K/V tile, 16-byte chunks XOR-swizzled by (row & 7)
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 256 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void tr(const LaMegaArgs& A, int slot, int k) {
  if (A.trace) A.trace[((size_t)blockIdx.x * A.trace_slots + slot) * 8 + k] = globaltimer();
}

// ------------------------------------------------------------- phases
// A GEMM phase's work: optionally one whole "data-parallel" tile per CTA
// (geo.dp = gridDim.x tiles [0, dp), epilogue straight from TMEM, no
// partials) plus a stream-K split of the remaining tiles [dp, n_tiles).
// A CTA walks its stream-K units first, then its data-parallel tile, as
// "virtual units" v in [0, n_virtual).
struct Ph {
  int kind, l;
  const __nv_bfloat16* a;   // packed weights
  const __nv_bfloat16* b;   // packed step rows
  LaMegaGeo g;
  float* ws;
  long U, u0, u1;           // stream-K units of the phase / this CTA's range
};

__device__ __forceinline__ Ph phase_of(const LaMegaArgs& A, int i) {
  Ph p;
  if (i == 4 * A.L) {
    p.kind = LA_MK_HEAD; p.l = A.L;
    p.a = A.lm_head; p.b = A.h_attn;
  } else {
    p.l = i >> 2; p.kind = i & 3;
    const LaMegaLayer& w = A.layers[p.l];
    switch (p.kind) {
      case LA_MK_QKV: p.a = w.wqkv; p.b = A.h_attn; break;
      case LA_MK_O: p.a = w.wo; p.b = A.attn_out; break;
      case LA_MK_GU: p.a = w.wgu; p.b = A.h_mlp; break;
      default: p.a = w.wd; p.b = A.act; break;
    }
  }
  p.g = A.geo[p.kind];
  p.ws = A.ws[p.kind];
  const long P = gridDim.x;
  p.U = (long)((p.g.n_tiles - p.g.dp) / p.g.tpc) * p.g.kb;
  p.u0 = (long)blockIdx.x * p.U / P;
  p.u1 = (long)(blockIdx.x + 1) * p.U / P;
  return p;
}

__device__ __forceinline__ long n_virtual(const Ph& p) { return (p.u1 - p.u0) + (p.g.dp ? p.g.kb : 0); }

// unit tile (tpc feature tiles) and k-block of virtual unit v
__device__ __forceinline__ void unit_of(const Ph& p, long v, int& tu, int& k) {
  const long ns = p.u1 - p.u0;
  if (v < ns) {
    const long u = p.u0 + v;
    tu = (int)(u / p.g.kb) + p.g.dp / p.g.tpc;
    k = (int)(u % p.g.kb);
  } else {
    tu = blockIdx.x;           // data-parallel tile (dp > 0 implies tpc == 1)
    k = (int)(v - ns);
  }
}

// end (exclusive) of the segment -- run of units of one unit tile -- at v
__device__ __forceinline__ long seg_end_of(const Ph& p, long v) {
  const long ns = p.u1 - p.u0;
  if (v >= ns) return n_virtual(p);
  const long u = p.u0 + v;
  return min(p.u1, (u / p.g.kb + 1) * p.g.kb) - p.u0;
}

__device__ __forceinline__ unsigned* layer_sync(const LaMegaArgs& A, int l) {
  return A.sync + (size_t)l * A.sm.layer_stride;
}

// packed LA-tile address of weight tile t, k-block k (la_gemm.cu layout:
// tiles grouped in pairs per k-block)
__device__ __forceinline__ const __nv_bfloat16* a_src(const Ph& p, int t, int k) {
  return p.a + ((size_t)((t / LA_TPC) * p.g.kb + k) * LA_TPC + (t % LA_TPC)) * (kTile / 2);
}

// readiness counter guarding k-block k of phase p's step-row operand
__device__ __forceinline__ const unsigned* b_dep(const LaMegaArgs& A, const Ph& p, int k, unsigned gen,
                                                 unsigned& target, int& key) {
  // a finished 128-feature tile bumps its readiness by kSlices in total
  // (once per reduction slice, or kSlices at once); the embedding once
  target = (gen + 1) * (unsigned)kSlices;
  switch (p.kind) {
    case LA_MK_QKV:
      key = k >> 1;
      if (p.l == 0) {
        target = gen + 1;
        return A.sync + A.sm.h0 + key;
      }
      return layer_sync(A, p.l - 1) + A.sm.rdy_h + key;
    case LA_MK_O:
      key = (k >> 1) / (A.H / A.KVH);
      target = (gen + 1) * (unsigned)A.nrb_max;
      return layer_sync(A, p.l) + A.sm.rdy_attn + key;
    case LA_MK_GU:
      key = k >> 1;
      return layer_sync(A, p.l) + A.sm.rdy_m + key;
    case LA_MK_DOWN:
      key = k;
      return layer_sync(A, p.l) + A.sm.rdy_act + key;
    default:
      key = k >> 1;
      return layer_sync(A, A.L - 1) + A.sm.rdy_h + key;
  }
}

// pieces of stream-K unit tile j (0-based among the split tiles) and this
// CTA's piece index.  With fewer units than CTAs every non-empty range is
// one unit and empty ranges interleave, so pieces are counted in units.
__device__ __forceinline__ int sk_pieces(long U, int kb, long j) {
  const long P = gridDim.x;
  if (U < P) return kb;
  return (int)(la_cta_of((j + 1) * kb - 1, U, P) - la_cta_of(j * kb, U, P) + 1);
}
__device__ __forceinline__ int sk_piece_index(const Ph& p, long j) {
  const long P = gridDim.x;
  if (p.U < P) return (int)(p.u0 - j * p.g.kb);
  return (int)(blockIdx.x - la_cta_of(j * p.g.kb, p.U, P));
}

// ------------------------------------------------- split-K reduction
// Pieces of split tiles are drained to the workspace; the reduction of a
// tile is split into kSlices slices of 32 tokens, spread round-robin over
// ALL CTAs' eight compute warps, each slice summing its pieces in piece order
// with one round of vector loads (deterministic, layout-independent).
// Tiles finished by a single CTA (data-parallel tiles of GU / LM head) take
// their epilogue straight from TMEM instead.

// pieces of feature tile ft of a phase (1: finished by one CTA)
__device__ __forceinline__ int tile_pieces(const LaMegaGeo& g, int ft) {
  if (ft < g.dp) return 1;
  const long U = (long)((g.n_tiles - g.dp) / g.tpc) * g.kb;
  return sk_pieces(U, g.kb, (ft - g.dp) / g.tpc);
}

// epilogue of a single-piece tile applied by the draining CTA itself
__device__ __forceinline__ bool direct_kind(int kind) { return kind == LA_MK_GU || kind == LA_MK_HEAD; }

__device__ __forceinline__ unsigned* arrivals(const LaMegaArgs& A, int kind, int l, int ft) {
  if (kind == LA_MK_HEAD) return A.sync + A.sm.head_cnt + ft;
  return layer_sync(A, l) + A.sm.cnt[kind] + ft;
}

// readiness counter a reduced slice of tile ft of phase (kind, l) bumps
__device__ __forceinline__ unsigned* ready_of(const LaMegaArgs& A, int kind, int l, int ft) {
  unsigned* ls = layer_sync(A, l);
  switch (kind) {
    case LA_MK_QKV: return ls + A.sm.rdy_qkv + ft;
    case LA_MK_O: return ls + A.sm.rdy_m + ft;
    case LA_MK_GU: return ls + A.sm.rdy_act + ft;
    default: return ls + A.sm.rdy_h + ft;
  }
}

// row scale of a deferred RMSNorm: rsqrt(mean(x^2) + eps) of token tok from
// the per-tile partial sums; the 8 threads of a token split the tiles
__device__ __forceinline__ float row_rstd(const LaMegaArgs& A, const float* ss, int tok, int part, bool valid) {
  float s = 0.f;
  if (valid)
    for (int t = part; t < (A.d >> 7); t += 8) s += __ldcg(ss + t * 128 + tok);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  return rsqrtf(s / (float)A.d + A.eps);
}

__device__ __forceinline__ uint4 pack8(const float* v, float scale) {
  return make_uint4(pack_bf16(v[0] * scale, v[1] * scale), pack_bf16(v[2] * scale, v[3] * scale),
                    pack_bf16(v[4] * scale, v[5] * scale), pack_bf16(v[6] * scale, v[7] * scale));
}

// every LM-head tile is folded into the argmax keys: resolve each row's
// argmax (ties -> lowest id), scatter owned rows, reset the keys
__device__ __forceinline__ void head_finish(const LaMegaArgs& A, const FwdPlan* P, int ct) {
  if (ct < LA_MAX_ROWS) {
    const unsigned long long k = atomicExch(A.keys + ct, 0ull);
    if (ct < P->n_rows) {
      const int idx = 0x7fffffff - (int)(uint32_t)(k & 0xffffffffu);
      A.row_amax[ct] = idx;
      if (A.dec && P->own[ct]) A.dec->amax[P->grow[ct]] = idx;
    }
  }
}

// per-token rsqrt(mean(x^2)+eps) into smem for a data-parallel epilogue
// (drain warps, et 0..127)
__device__ __forceinline__ void direct_rstd(const LaMegaArgs& A, const Ph& p, const FwdPlan* P, float* s_rstd,
                                            int et) {
  const float* ss = p.kind == LA_MK_GU ? A.ss_mlp : A.ss_attn;
  if (et < P->n_rows) {
    float s = 0.f;
    for (int t = 0; t < (A.d >> 7); ++t) s += __ldcg(ss + t * 128 + et);
    s_rstd[et] = rsqrtf(s / (float)A.d + A.eps);
  }
  ptx::named_bar_sync(1, 128);
}

// epilogue of a tile computed entirely by this CTA (GU: SwiGLU -> act; LM
// head: logits + argmax), straight from TMEM through a [128 f][33] staging
// tile; drain warps only (et 0..127, f = TMEM lane)
__device__ void direct_epilogue(const LaMegaArgs& A, const Ph& p, const FwdPlan* P, int ft, uint32_t t_base,
                                float* sEpi, const float* s_rstd, int* s_flag, int et, int f) {
  const int n_rows = P->n_rows;
  const int j = et >> 2, q4 = et & 3;
  for (int c0 = 0; c0 < P->n_pad; c0 += 32) {
    float v[32];
    ptx::tmem_ld32(t_base + c0, v);
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) sEpi[f * kEpiLd + jj] = v[jj];
    ptx::named_bar_sync(1, 128);
    const int tok = c0 + j;
    const bool valid = tok < n_rows;
    if (p.kind == LA_MK_GU) {
      if (valid) {
        const float rs = s_rstd[tok];
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int i0 = q4 * 16 + 2 * q;
          const float g0 = sEpi[i0 * kEpiLd + j] * rs, g1 = sEpi[(i0 + 1) * kEpiLd + j] * rs;
          const float u0 = sEpi[(64 + i0) * kEpiLd + j] * rs, u1 = sEpi[(64 + i0 + 1) * kEpiLd + j] * rs;
          w[q] = pack_bf16(g0 / (1.0f + __expf(-g0)) * u0, g1 / (1.0f + __expf(-g1)) * u1);
        }
        const int k0 = ft * 64 + q4 * 16;
        *reinterpret_cast<uint4*>(A.act + la_act_off(tok, k0)) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(A.act + la_act_off(tok, k0 + 8)) = make_uint4(w[4], w[5], w[6], w[7]);
      }
    } else {
      unsigned long long best = 0ull;
      if (valid) {
        const float rs = s_rstd[tok];
#pragma unroll 8
        for (int q = 0; q < 32; ++q) {
          const int fg = ft * 128 + q4 * 32 + q;
          if (fg < A.V) {
            const float lv = sEpi[(q4 * 32 + q) * kEpiLd + j] * rs;
            if (A.logits) A.logits[(size_t)tok * A.V + fg] = lv;
            const unsigned long long key = argmax_key(lv, fg);
            best = key > best ? key : best;
          }
        }
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const unsigned long long key = __shfl_xor_sync(0xffffffffu, best, o);
        best = key > best ? key : best;
      }
      if (valid && q4 == 0 && best) atomicMax(A.keys + tok, best);
    }
    ptx::named_bar_sync(1, 128);
  }
  if (p.kind == LA_MK_GU) fence_proxy_async();
  ptx::named_bar_sync(1, 128);
  if (et == 0) {
    __threadfence();
    *s_flag = 0;
    if (p.kind == LA_MK_GU) {
      atomicAdd(layer_sync(A, p.l) + A.sm.rdy_act + ft, (unsigned)kSlices);
    } else {
      const unsigned total = (unsigned)(p.g.real * kSlices);
      const unsigned old = atomicAdd(A.sync + A.sm.head_done, (unsigned)kSlices);
      if (old + kSlices == total) {
        atomicExch(A.sync + A.sm.head_done, 0u);
        __threadfence();
        *s_flag = 1;
      }
    }
  }
  ptx::named_bar_sync(1, 128);
  if (*s_flag) {
    head_finish(A, P, et);
    ptx::named_bar_sync(1, 128);
  }
}

// all reduction slices of phase p owned by this CTA (256 threads, ct)
__device__ void reduce_phase(const LaMegaArgs& A, const Ph& p, const FwdPlan* P, unsigned gen, unsigned hgen,
                             int* s_flag, int ct) {
  const int n_rows = P->n_rows;
  const int jj = ct >> 3, part = ct & 7;
  unsigned* err = A.sync + A.sm.err;
  const unsigned g1 = (p.kind == LA_MK_HEAD ? hgen : gen) + 1;
  const int total_slices = p.g.real * kSlices;               // LM-head completion count
  const int t0 = direct_kind(p.kind) ? p.g.dp : 0;            // data-parallel tiles finish in the drain
  const int n_slices = (p.g.real - t0) * kSlices;
  for (int sl0 = blockIdx.x; sl0 < n_slices; sl0 += gridDim.x) {
    const int sl = sl0 + t0 * kSlices;
    const int ft = sl / kSlices;
    if (direct_kind(p.kind) && tile_pieces(p.g, ft) == 1) continue;   // finished by its only CTA
    const int tok = (sl % kSlices) * 32 + jj;
    const bool any = (sl % kSlices) * 32 < n_rows;
    const bool valid = tok < n_rows;
    const int nseg = tile_pieces(p.g, ft);
    if (any) {
      if (ct == 0) wait_ge(arrivals(A, p.kind, p.l, ft), g1 * (unsigned)nseg, err);
      ptx::named_bar_sync(2, 256);
    }
    // v[0..7] = features part*8.., v[8..15] = features 64 + part*8..
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.f;
    if (valid && !(A.debug & 2)) {
      const float* base = p.ws + ((size_t)ft * p.g.max_segs * 128 + tok) * 128 + part * 8;
      for (int s0 = 0; s0 < nseg; s0 += 4) {
        float4 r[4][4];
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (s0 + s < nseg) {
            const float4* q = reinterpret_cast<const float4*>(base + (size_t)(s0 + s) * 128 * 128);
            r[s][0] = __ldcg(q); r[s][1] = __ldcg(q + 1); r[s][2] = __ldcg(q + 16); r[s][3] = __ldcg(q + 17);
          }
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (s0 + s < nseg) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              v[4 * c] += r[s][c].x; v[4 * c + 1] += r[s][c].y; v[4 * c + 2] += r[s][c].z; v[4 * c + 3] += r[s][c].w;
            }
          }
      }
    }
    if (p.kind == LA_MK_QKV) {
      const float rs = row_rstd(A, A.ss_attn, tok, part, valid);
      if (valid && ft < p.g.real) {
        const size_t lstride = (size_t)A.slots * A.KVH * 128;
        __nv_bfloat16* dst;
        bool rope = true;
        if (ft < A.H) {
          dst = A.q + ((size_t)tok * A.H + ft) * 128;
        } else if (ft < A.H + A.KVH) {
          dst = A.kc + (size_t)p.l * lstride + ((size_t)P->slot[tok] * A.KVH + (ft - A.H)) * 128;
        } else {
          dst = A.vc + (size_t)p.l * lstride + ((size_t)P->slot[tok] * A.KVH + (ft - A.H - A.KVH)) * 128;
          rope = false;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= rs;
        if (rope) {
          // rotate-half RoPE at the row's absolute position: (x_i, x_{i+64})
          const float* cs = A.rope_cos + (size_t)P->pos[tok] * 64 + part * 8;
          const float* sn = A.rope_sin + (size_t)P->pos[tok] * 64 + part * 8;
          float lo[8], hi[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            lo[i] = v[i] * cs[i] - v[8 + i] * sn[i];
            hi[i] = v[8 + i] * cs[i] + v[i] * sn[i];
          }
          *reinterpret_cast<uint4*>(dst + part * 8) = pack8(lo, 1.f);
          *reinterpret_cast<uint4*>(dst + 64 + part * 8) = pack8(hi, 1.f);
        } else {
          *reinterpret_cast<uint4*>(dst + part * 8) = pack8(v, 1.f);
          *reinterpret_cast<uint4*>(dst + 64 + part * 8) = pack8(v + 8, 1.f);
        }
      }
    } else if (p.kind == LA_MK_O || p.kind == LA_MK_DOWN) {
      // residual add; next GEMM input bf16(x * g); per-tile sum of x^2
      const float* g;
      __nv_bfloat16* hout;
      float* ss;
      if (p.kind == LA_MK_O) {
        g = A.layers[p.l].mlp_norm; hout = A.h_mlp; ss = A.ss_mlp;
      } else {
        g = p.l + 1 < A.L ? A.layers[p.l + 1].attn_norm : A.final_norm;
        hout = A.h_attn; ss = A.ss_attn;
      }
      float sq = 0.f;
      if (valid) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int f0 = ft * 128 + h2 * 64 + part * 8;
          float* xr = A.x + (size_t)tok * A.d + f0;
          const float4 a0 = __ldcg(reinterpret_cast<const float4*>(xr));
          const float4 a1 = __ldcg(reinterpret_cast<const float4*>(xr + 4));
          float* xv = v + 8 * h2;
          xv[0] += a0.x; xv[1] += a0.y; xv[2] += a0.z; xv[3] += a0.w;
          xv[4] += a1.x; xv[5] += a1.y; xv[6] += a1.z; xv[7] += a1.w;
          __stcg(reinterpret_cast<float4*>(xr), make_float4(xv[0], xv[1], xv[2], xv[3]));
          __stcg(reinterpret_cast<float4*>(xr + 4), make_float4(xv[4], xv[5], xv[6], xv[7]));
          const float4 g0 = *reinterpret_cast<const float4*>(g + f0);
          const float4 g1v = *reinterpret_cast<const float4*>(g + f0 + 4);
          const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1v.x, g1v.y, g1v.z, g1v.w};
          float hv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            sq += xv[i] * xv[i];
            hv[i] = xv[i] * gg[i];
          }
          *reinterpret_cast<uint4*>(hout + la_act_off(tok, f0)) = pack8(hv, 1.f);
        }
      }
      sq += __shfl_xor_sync(0xffffffffu, sq, 1);
      sq += __shfl_xor_sync(0xffffffffu, sq, 2);
      sq += __shfl_xor_sync(0xffffffffu, sq, 4);
      if (valid && part == 0) __stcg(ss + ft * 128 + tok, sq);
    } else if (p.kind == LA_MK_GU) {
      const float rs = row_rstd(A, A.ss_mlp, tok, part, valid);
      if (valid) {
        float w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float gt = v[i] * rs, up = v[8 + i] * rs;
          w[i] = gt / (1.0f + __expf(-gt)) * up;
        }
        *reinterpret_cast<uint4*>(A.act + la_act_off(tok, ft * 64 + part * 8)) = pack8(w, 1.f);
      }
    } else {   // LM head: logits = rstd * acc; per-row argmax, ties -> lowest id
      const float rs = row_rstd(A, A.ss_attn, tok, part, valid);
      unsigned long long best = 0ull;
      if (valid) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int fg = ft * 128 + (i < 8 ? part * 8 + i : 64 + part * 8 + i - 8);
          if (fg < A.V) {
            const float lv = v[i] * rs;
            if (A.logits) A.logits[(size_t)tok * A.V + fg] = lv;
            const unsigned long long k = argmax_key(lv, fg);
            best = k > best ? k : best;
          }
        }
      }
#pragma unroll
      for (int o = 1; o <= 4; o <<= 1) {
        const unsigned long long k = __shfl_xor_sync(0xffffffffu, best, o);
        best = k > best ? k : best;
      }
      if (valid && part == 0 && best) atomicMax(A.keys + tok, best);
    }
    // publish: writer-side proxy fence only where a bulk copy reads the
    // result; one release fence per CTA after the barrier (the barrier orders
    // every thread's stores before it, the fence is cumulative)
    if (p.kind == LA_MK_O || p.kind == LA_MK_GU || p.kind == LA_MK_DOWN) fence_proxy_async();
    ptx::named_bar_sync(2, 256);
    if (ct == 0) {
      __threadfence();
      *s_flag = 0;
      if (p.kind == LA_MK_HEAD) {
        const unsigned old = atomicAdd(A.sync + A.sm.head_done, 1u);
        if (old == (unsigned)total_slices - 1) {
          atomicExch(A.sync + A.sm.head_done, 0u);
          __threadfence();
          *s_flag = 1;
        }
      } else {
        atomicAdd(ready_of(A, p.kind, p.l, ft), 1u);
      }
    }
    ptx::named_bar_sync(2, 256);
    if (p.kind == LA_MK_HEAD && *s_flag) {
      head_finish(A, P, ct);
      ptx::named_bar_sync(2, 256);
    }
  }
}

// ------------------------------------------------------------ attention
__device__ __forceinline__ int chunk_keys(int ctx, int S) {
  return ((ctx + S - 1) / S + kKeyTile - 1) / kKeyTile * kKeyTile;
}

// all attention units of layer l owned by this CTA; warps 3..10 (ct 0..255)
__device__ void attention_layer(const LaMegaArgs& A, const FwdPlan* P, int l, unsigned gen, uint8_t* sKV,
                                uint32_t* sMask, int* s_flag, int ct) {
  const int n_rows = P->n_rows, ctx = P->n_prefix;
  const int g = A.H / A.KVH;
  const int nq = n_rows * g;
  const int n_rb = (nq + 127) >> 7;
  const int S = A.attn_S;
  const int per_kvh = n_rb * (S + 1);
  const int n_units = A.KVH * per_kvh;
  const int cw = ct >> 5, lane = ct & 31;
  const size_t kv_ld = (size_t)A.KVH * 128;
  const size_t lstride = (size_t)A.slots * kv_ld;
  const __nv_bfloat16* kc = A.kc + (size_t)l * lstride;
  const __nv_bfloat16* vc = A.vc + (size_t)l * lstride;
  unsigned* ls = layer_sync(A, l);
  unsigned* err = A.sync + A.sm.err;
  const float sl2 = kLog2e / sqrtf(128.0f);
  const int CH = ctx > 0 ? chunk_keys(ctx, S) : 0;

  for (int e = blockIdx.x; e < n_units; e += gridDim.x) {
    const int kvh = e / per_kvh;
    const int rb = (e % per_kvh) / (S + 1);
    const int split = e % (S + 1);
    const int uid = (kvh * A.nrb_max + rb) * (S + 1) + split;
    const bool step_unit = split == S;
    int k_begin, k_end;
    if (step_unit) {
      k_begin = ctx; k_end = ctx + P->n_global;
    } else {
      k_begin = min(ctx, split * CH); k_end = min(ctx, (split + 1) * CH);
    }
    // dependencies: this group's q tiles (and, for the step keys, k / v)
    if (ct == 0) {
      const unsigned tq = (gen + 1) * (unsigned)kSlices;
      for (int hg = 0; hg < g; ++hg) wait_ge(ls + A.sm.rdy_qkv + kvh * g + hg, tq, err);
      if (step_unit) {
        wait_ge(ls + A.sm.rdy_qkv + A.H + kvh, tq, err);
        wait_ge(ls + A.sm.rdy_qkv + A.H + A.KVH + kvh, tq, err);
      }
      __threadfence();
      if (e == blockIdx.x) tr(A, 4 * A.L + 1 + l, 2);
    }
    ptx::named_bar_sync(2, 256);

    const int qrow0 = cw * 16 + (lane >> 2);          // this thread's rows (qrow0, qrow0 + 8)
    const bool warp_active = rb * 128 + cw * 16 < nq;
    if (step_unit) {
      for (int i = ct; i < 128 * 4; i += 256) sMask[i] = 0u;
      ptx::named_bar_sync(2, 256);
      for (int row = cw; row < 128; row += 8) {
        const int qr = rb * 128 + row;
        if (qr >= nq) continue;
        const int r = qr / g;
        const int n = P->chain_n[r];
        for (int jj = lane; jj <= n; jj += 32) {
          const int key = (jj < n ? P->chain[r][jj] : P->slot[r]) - ctx;
          atomicOr(&sMask[row * 4 + (key >> 5)], 1u << (key & 31));
        }
      }
    }
    const int n_tiles = (A.debug & 4) ? 0 : (k_end - k_begin + kKeyTile - 1) / kKeyTile;
    auto load_kv = [&](int t) {
      uint8_t* kb = sKV + (t & 1) * 2 * kKeyTile * 256;
      const int t0 = k_begin + t * kKeyTile;
      for (int i = ct; i < kKeyTile * 16; i += 256) {
        const int row = i >> 4, ch = i & 15, key = t0 + row;
        const bool ok = key < k_end;
        const size_t off = ((size_t)(ok ? key : k_begin) * kv_ld) + kvh * 128 + ch * 8;
        cp_async16(ptx::smem_u32(kb) + swz(row, ch), kc + off, ok);
        cp_async16(ptx::smem_u32(kb + kKeyTile * 256) + swz(row, ch), vc + off, ok);
      }
    };
    if (n_tiles > 0) load_kv(0);
    cp_commit();

    // Q fragments straight from global (m16n8k16 A layout)
    uint32_t qf[8][4];
    {
      const int qa = rb * 128 + qrow0, qb = qa + 8;
      const __nv_bfloat16* pa = nullptr;
      const __nv_bfloat16* pb = nullptr;
      if (qa < nq) pa = A.q + ((size_t)(qa / g) * A.H + kvh * g + qa % g) * 128;
      if (qb < nq) pb = A.q + ((size_t)(qb / g) * A.H + kvh * g + qb % g) * 128;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int col = kk * 16 + (lane & 3) * 2;
        qf[kk][0] = pa ? __ldcg(reinterpret_cast<const unsigned*>(pa + col)) : 0u;
        qf[kk][1] = pb ? __ldcg(reinterpret_cast<const unsigned*>(pb + col)) : 0u;
        qf[kk][2] = pa ? __ldcg(reinterpret_cast<const unsigned*>(pa + col + 8)) : 0u;
        qf[kk][3] = pb ? __ldcg(reinterpret_cast<const unsigned*>(pb + col + 8)) : 0u;
      }
    }
    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int t = 0; t < n_tiles; ++t) {
      if (t + 1 < n_tiles) load_kv(t + 1);
      cp_commit();
      cp_wait<1>();
      ptx::named_bar_sync(2, 256);
      if (warp_active) {
        const uint8_t* sK = sKV + (t & 1) * 2 * kKeyTile * 256;
        const uint8_t* sV = sK + kKeyTile * 256;
        float s[8][4];
#pragma unroll
        for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
          for (int np = 0; np < 4; ++np) {
            const int key = np * 16 + (lane & 7) + (lane >> 4) * 8;
            const int ch = kk * 2 + ((lane >> 3) & 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4(ptx::smem_u32(sK) + swz(key, ch), b0, b1, b2, b3);
            mma16816(s[2 * np], qf[kk], b0, b1);
            mma16816(s[2 * np + 1], qf[kk], b2, b3);
          }
        }
        const int kbase = k_begin + t * kKeyTile;
        float mx0 = m0, mx1 = m1;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const int key = kbase + n * 8 + (lane & 3) * 2 + (e2 & 1);
            bool vis = key < k_end;
            if (step_unit && vis) {
              const int kg = key - ctx, row = qrow0 + (e2 >> 1) * 8;
              vis = (sMask[row * 4 + (kg >> 5)] >> (kg & 31)) & 1u;
            }
            s[n][e2] = vis ? s[n][e2] * sl2 : -INFINITY;
          }
          mx0 = fmaxf(mx0, fmaxf(s[n][0], s[n][1]));
          mx1 = fmaxf(mx1, fmaxf(s[n][2], s[n][3]));
        }
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const float b0 = mx0 == -INFINITY ? 0.f : mx0, b1 = mx1 == -INFINITY ? 0.f : mx1;
        const float al0 = exp2f(m0 - b0), al1 = exp2f(m1 - b1);
        m0 = mx0;
        m1 = mx1;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          s[n][0] = exp2f(s[n][0] - b0);
          s[n][1] = exp2f(s[n][1] - b0);
          s[n][2] = exp2f(s[n][2] - b1);
          s[n][3] = exp2f(s[n][3] - b1);
          rs0 += s[n][0] + s[n][1];
          rs1 += s[n][2] + s[n][3];
        }
        l0 = l0 * al0 + rs0;
        l1 = l1 * al1 + rs1;
#pragma unroll
        for (int dd = 0; dd < 16; ++dd) {
          o[dd][0] *= al0; o[dd][1] *= al0; o[dd][2] *= al1; o[dd][3] *= al1;
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          uint32_t pa[4] = {pack_bf16(s[2 * kk][0], s[2 * kk][1]), pack_bf16(s[2 * kk][2], s[2 * kk][3]),
                            pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                            pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
          for (int dp = 0; dp < 8; ++dp) {
            const int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
            const int ch = dp * 2 + (lane >> 4);
            uint32_t v0, v1, v2, v3;
            ldsm_x4_t(ptx::smem_u32(sV) + swz(key, ch), v0, v1, v2, v3);
            mma16816(o[2 * dp], pa, v0, v1);
            mma16816(o[2 * dp + 1], pa, v2, v3);
          }
        }
      }
      ptx::named_bar_sync(2, 256);
    }
    cp_wait<0>();
    if (ct == 0 && e == blockIdx.x) tr(A, 4 * A.L + 1 + l, 3);
    // partial (unnormalised O, (m, l) in log2 units) of this key chunk
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int row = qrow0 + half * 8;
      if (rb * 128 + row >= nq) continue;
      float* dst = A.attn_ws + ((size_t)uid * 128 + row) * 128;
#pragma unroll
      for (int dd = 0; dd < 16; ++dd) {
        const int col = dd * 8 + (lane & 3) * 2;
        __stcg(reinterpret_cast<float2*>(dst + col), make_float2(o[dd][half * 2], o[dd][half * 2 + 1]));
      }
      if ((lane & 3) == 0)
        __stcg(A.attn_ml + (size_t)uid * 128 + row, make_float2(half ? m1 : m0, half ? l1 : l0));
    }
    ptx::named_bar_sync(2, 256);
    if (ct == 0) {
      __threadfence();
      unsigned* cnt = ls + A.sm.attn_cnt + kvh * A.nrb_max + rb;
      const unsigned old = atomicAdd(cnt, 1u);
      const int last = old == (unsigned)S;
      if (last) {
        atomicExch(cnt, 0u);   // only this CTA touches it again this launch
        __threadfence();
      }
      *s_flag = last;
    }
    ptx::named_bar_sync(2, 256);
    if (*s_flag) {
      // last chunk of (kvh, rb): merge the S+1 partials in chunk order
      const int row = ct >> 1, hd = (ct & 1) * 64;
      const int qr = rb * 128 + row;
      if (qr < nq) {
        float m = -INFINITY, ll = 0.f;
        float acc[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) acc[i] = 0.f;
        for (int sp = 0; sp <= S; ++sp) {
          const int us = (kvh * A.nrb_max + rb) * (S + 1) + sp;
          const float2 ml = __ldcg(A.attn_ml + (size_t)us * 128 + row);
          if (ml.x == -INFINITY) continue;
          const float mn = fmaxf(m, ml.x);
          const float s0 = exp2f(m - mn), s1 = exp2f(ml.x - mn);
          const float4* po = reinterpret_cast<const float4*>(A.attn_ws + ((size_t)us * 128 + row) * 128 + hd);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float4 v = __ldcg(po + i);
            acc[4 * i] = acc[4 * i] * s0 + v.x * s1;
            acc[4 * i + 1] = acc[4 * i + 1] * s0 + v.y * s1;
            acc[4 * i + 2] = acc[4 * i + 2] * s0 + v.z * s1;
            acc[4 * i + 3] = acc[4 * i + 3] * s0 + v.w * s1;
          }
          ll = ll * s0 + ml.y * s1;
          m = mn;
        }
        const float inv = 1.0f / ll;
        const int r = qr / g, head = kvh * g + qr % g;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(A.attn_out + la_act_off(r, head * 128 + hd + 8 * c)) =
              make_uint4(pack_bf16(acc[8 * c] * inv, acc[8 * c + 1] * inv),
                         pack_bf16(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv),
                         pack_bf16(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv),
                         pack_bf16(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv));
      }
      fence_proxy_async();
      ptx::named_bar_sync(2, 256);
      // per-launch total per KV head is nrb_max whatever the row count
      if (ct == 0) {
        __threadfence();
        atomicAdd(ls + A.sm.rdy_attn + kvh, rb == n_rb - 1 ? 1u + (unsigned)(A.nrb_max - n_rb) : 1u);
        tr(A, 4 * A.L + 1 + l, 4);
      }
    }
  }
}

// x := embedding rows; layer-0 GEMM input bf16(x * g); per-tile sums of x^2
__device__ void embed_phase(const LaMegaArgs& A, const FwdPlan* P, int ct) {
  const int n_rows = P->n_rows;
  const int nt = A.d >> 7;
  const float* g = A.layers[0].attn_norm;
  const int span = (n_rows * 16 + 31) & ~31;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    for (int i = ct; i < span; i += 256) {
      const int r = i >> 4, c8 = i & 15;
      const bool valid = r < n_rows;
      const int f0 = t * 128 + c8 * 8;
      float s = 0.f;
      if (valid) {
        const uint4 e = *reinterpret_cast<const uint4*>(A.embed + (size_t)P->ids[r] * A.d + f0);
        const __nv_bfloat162* e2 = reinterpret_cast<const __nv_bfloat162*>(&e);
        float xv[8];
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          const float2 f2 = __bfloat1622float2(e2[i2]);
          xv[2 * i2] = f2.x; xv[2 * i2 + 1] = f2.y;
        }
        float* xr = A.x + (size_t)r * A.d + f0;
        __stcg(reinterpret_cast<float4*>(xr), make_float4(xv[0], xv[1], xv[2], xv[3]));
        __stcg(reinterpret_cast<float4*>(xr + 4), make_float4(xv[4], xv[5], xv[6], xv[7]));
        const float4 g0 = *reinterpret_cast<const float4*>(g + f0);
        const float4 g1 = *reinterpret_cast<const float4*>(g + f0 + 4);
        *reinterpret_cast<uint4*>(A.h_attn + la_act_off(r, f0)) =
            make_uint4(pack_bf16(xv[0] * g0.x, xv[1] * g0.y), pack_bf16(xv[2] * g0.z, xv[3] * g0.w),
                       pack_bf16(xv[4] * g1.x, xv[5] * g1.y), pack_bf16(xv[6] * g1.z, xv[7] * g1.w));
#pragma unroll
        for (int i2 = 0; i2 < 8; ++i2) s += xv[i2] * xv[i2];
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (valid && c8 == 0) __stcg(A.ss_attn + t * 128 + r, s);
    }
    fence_proxy_async();
    ptx::named_bar_sync(2, 256);
    if (ct == 0) {
      __threadfence();
      atomicAdd(A.sync + A.sm.h0 + t, 1u);
    }
  }
}

// ---------------------------------------------------------------- kernel
__global__ void __launch_bounds__(kThreads, 1) la_mega_kernel(const LaMegaArgs A) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024 - (ptx::smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = sm + kOffA;
  uint8_t* sB = sm + kOffB;
  float* sEpi = reinterpret_cast<float*>(sm + kOffEpi);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kOffBar);
  uint64_t* afull = bars;
  uint64_t* aempty = bars + kAStages;
  uint64_t* bfull = bars + 2 * kAStages;
  uint64_t* bempty = bars + 2 * kAStages + kBStages;
  uint64_t* tfull = bars + 2 * kAStages + 2 * kBStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kOffMisc);
  int* s_flag = reinterpret_cast<int*>(sm + kOffMisc + 16);
  volatile int* s_attn_layers = reinterpret_cast<volatile int*>(sm + kOffMisc + 32);   // layers whose attention this CTA finished
  float* s_rstd = reinterpret_cast<float*>(sm + kOffRstd);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nph = 4 * A.L + (A.do_head ? 1 : 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kAStages; ++s) { ptx::mbar_init(&afull[s], 1); ptx::mbar_init(&aempty[s], 1); }
    for (int s = 0; s < kBStages; ++s) { ptx::mbar_init(&bfull[s], 1); ptx::mbar_init(&bempty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&tfull[b], 1); ptx::mbar_init(&tempty[b], 128); }
    *s_attn_layers = 0;
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // weights do not depend on the previous kernel: start streaming them now.
  // Two cursors walk every weight unit of the step: loads into the smem
  // ring and, A.pf_units ahead of them, L2 prefetches.
  const uint64_t pol_w = ptx::policy_evict_first();
  struct Cursor {
    int ph;
    long v, nv;
    Ph p;
  };
  auto cur_init = [&](Cursor& c) {
    c.ph = 0; c.v = 0; c.p = phase_of(A, 0); c.nv = n_virtual(c.p);
  };
  // advance to the next existing unit; false when the step has no more
  auto cur_valid = [&](Cursor& c) -> bool {
    while (c.v >= c.nv) {
      if (++c.ph >= nph) return false;
      c.p = phase_of(A, c.ph); c.v = 0; c.nv = n_virtual(c.p);
    }
    return true;
  };
  Cursor ac, pc;
  int a_it = 0;
  long pf_n = 0;
  auto pf_ahead = [&](long target) {
    while (pf_n < target && cur_valid(pc)) {
      int tu, k;
      unit_of(pc.p, pc.v, tu, k);
      ptx::bulk_prefetch_l2(a_src(pc.p, tu, k), (uint32_t)pc.p.g.tpc * kTile);
      ++pc.v;
      ++pf_n;
    }
  };
  auto a_issue = [&](int s) {
    int tu, k;
    unit_of(ac.p, ac.v, tu, k);
    const uint32_t bytes = (uint32_t)ac.p.g.tpc * kTile;
    ptx::mbar_expect_tx(&afull[s], bytes);
    ptx::bulk_load(sA + s * kAStage, a_src(ac.p, tu, k), bytes, &afull[s], pol_w);
    ++ac.v;
  };
  if (warp == 0 && lane == 0) {
    cur_init(ac);
    cur_init(pc);
    while (a_it < kAStages && cur_valid(ac)) {
      a_issue(a_it);
      ++a_it;
      // the ring's first units are loaded directly: prefetch only beyond them
      if (cur_valid(pc)) { ++pc.v; ++pf_n; }
    }
    pf_ahead((long)a_it + A.pf_units);
  }
  la_pdl_wait();
  const FwdPlan* P = A.plan;
  const int n_rows = P->n_rows;
  unsigned* err = A.sync + A.sm.err;
  const unsigned gen = ld_acquire(A.sync + A.sm.gen);
  const unsigned hgen = ld_acquire(A.sync + A.sm.head_gen);   // launches that ran the LM head
  if (A.timing && threadIdx.x == 0 && n_rows > 0) {
    if (atomicAdd(&A.timing[3], 1ull) == 0ull) A.timing[0] = globaltimer();
  }

  if (n_rows == 0) {
    // nothing to evaluate: retire the prefetched weight tiles and leave
    if (warp == 0 && lane == 0)
      for (int s = 0; s < a_it; ++s) ptx::mbar_wait(&afull[s], 0);
  } else if (warp == 0) {
    // ----------------------------------------------------- weight producer
    if (lane == 0) {
      while (cur_valid(ac)) {
        const int s = a_it % kAStages;
        pf_ahead((long)a_it + 1 + A.pf_units);
        if (a_it >= kAStages) ptx::mbar_wait(&aempty[s], ((a_it / kAStages) - 1) & 1);
        a_issue(s);
        ++a_it;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------- step-row producer
    if (lane == 0) {
      const uint64_t pol_x = ptx::policy_evict_last();
      const uint32_t bbytes = (uint32_t)P->n_pad * 128;
      int it = 0;
      for (int ph = 0; ph < nph; ++ph) {
        const Ph p = phase_of(A, ph);
        if (p.kind == LA_MK_O) {
          // the B ring is lent to this CTA's attention units of layer l
          while (*s_attn_layers <= p.l) __nanosleep(64);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        int dep_key = -1;
        const long nv = n_virtual(p);
        for (long v = 0; v < nv; ++v, ++it) {
          const int s = it % kBStages;
          if (it >= kBStages) ptx::mbar_wait(&bempty[s], ((it / kBStages) - 1) & 1);
          int tu, k;
          unit_of(p, v, tu, k);
          unsigned target;
          int key;
          const unsigned* dep = b_dep(A, p, k, gen, target, key);
          if (key != dep_key) {
            wait_ge(dep, target, err);
            fence_proxy_async();
            if (dep_key < 0) tr(A, ph, 0);
            dep_key = key;
          }
          if (A.debug & 1) {
            ptx::mbar_arrive(&bfull[s]);   // timing experiment: no step-row traffic
          } else {
            ptx::mbar_expect_tx(&bfull[s], bbytes);
            ptx::bulk_load(sB + s * kBStage, p.b + (size_t)k * 8192, bbytes, &bfull[s], pol_x);
          }
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = ptx::umma_idesc_bf16(128, (uint32_t)P->n_pad);
      int it = 0, use[2] = {0, 0}, buf = 0;
      for (int ph = 0; ph < nph; ++ph) {
        const Ph p = phase_of(A, ph);
        const long nv = n_virtual(p);
        long v = 0;
        while (v < nv) {
          const long seg_start = v, seg_end = seg_end_of(p, v);
          if (use[buf] > 0) {
            ptx::mbar_wait(&tempty[buf], (use[buf] - 1) & 1);
            ptx::tc_fence_after();
          }
          const uint32_t d_tmem = tmem + buf * (LA_TPC * 128);
          for (; v < seg_end; ++v, ++it) {
            const int sa = it % kAStages, sb = it % kBStages;
            ptx::mbar_wait(&afull[sa], (uint32_t)(it / kAStages) & 1);
            ptx::mbar_wait(&bfull[sb], (uint32_t)(it / kBStages) & 1);
            ptx::tc_fence_after();
            if (v == 0) tr(A, ph, 1);
            const uint32_t a_addr = ptx::smem_u32(sA + sa * kAStage);
            const uint32_t b_addr = ptx::smem_u32(sB + sb * kBStage);
            for (int tt = 0; tt < p.g.tpc; ++tt)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                ptx::umma_bf16(d_tmem + tt * 128, ptx::umma_desc_sw128(a_addr + tt * kTile + kk * 32),
                               ptx::umma_desc_sw128(b_addr + kk * 32), idesc,
                               (v > seg_start || kk > 0) ? 1u : 0u);
            ptx::umma_commit(&aempty[sa]);
            ptx::umma_commit(&bempty[sb]);
          }
          ptx::umma_commit(&tfull[buf]);
          use[buf]++;
          buf ^= 1;
        }
        if (nv > 0) tr(A, ph, 2);
      }
    }
  } else {
    // ----------------------- warps 3..10: drain / reduce / attention
    const int ct = threadIdx.x - 96;           // 0..255
    const bool epi = warp <= 6;                // warps 3..6 own the TMEM lanes 32*(warp%4)..
    const int f = 32 * (warp & 3) + lane;      // accumulator lane = feature in tile
    embed_phase(A, P, ct);
    int use[2] = {0, 0}, buf = 0;
    for (int ph = 0; ph < nph; ++ph) {
      const Ph p = phase_of(A, ph);
      if (epi) {
        // drain every piece of this CTA: split tiles to the workspace
        // (arrival counted), single-piece GU / LM-head tiles straight through
        // the epilogue
        bool have_rstd = false;
        const long nv = n_virtual(p), ns = p.u1 - p.u0;
        long v = 0;
        while (v < nv) {
          const long seg_end = seg_end_of(p, v);
          int tu, k0;
          unit_of(p, v, tu, k0);
          int seg = 0, nseg = 1;
          if (v < ns) {
            const long j = tu - p.g.dp / p.g.tpc;
            nseg = sk_pieces(p.U, p.g.kb, j);
            seg = sk_piece_index(p, j);
          }
          ptx::mbar_wait(&tfull[buf], use[buf] & 1);
          ptx::tc_fence_after();
          const uint32_t t_row = (uint32_t)(32 * (warp & 3)) << 16;
          if (nseg == 1 && direct_kind(p.kind)) {
            if (!have_rstd) {
              direct_rstd(A, p, P, s_rstd, ct);
              have_rstd = true;
            }
            direct_epilogue(A, p, P, tu, tmem + t_row + buf * (LA_TPC * 128), sEpi, s_rstd, s_flag + 2, ct, f);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[buf]);
          } else {
            for (int tt = 0; tt < p.g.tpc; ++tt) {
              const int ft = tu * p.g.tpc + tt;
              if (ft >= p.g.real) continue;
              const uint32_t t_base = tmem + t_row + buf * (LA_TPC * 128) + tt * 128;
              float* wsp = p.ws + ((size_t)ft * p.g.max_segs + seg) * 128 * 128 + f;
              for (int c0 = 0; c0 < P->n_pad; c0 += 32) {
                float vv[32];
                ptx::tmem_ld32(t_base + c0, vv);
                const int nj = min(32, n_rows - c0);
                if (!(A.debug & 8)) {
#pragma unroll
                  for (int jj = 0; jj < 32; ++jj)
                    if (jj < nj) __stcg(wsp + (size_t)(c0 + jj) * 128, vv[jj]);
                }
              }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[buf]);
            ptx::named_bar_sync(1, 128);
            if (ct == 0) {
              __threadfence();
              for (int tt = 0; tt < p.g.tpc; ++tt) {
                const int ft = tu * p.g.tpc + tt;
                if (ft < p.g.real) atomicAdd(arrivals(A, p.kind, p.l, ft), 1u);
              }
            }
          }
          use[buf]++;
          buf ^= 1;
          v = seg_end;
        }
        if (ct == 0 && nv > 0) tr(A, ph, 3);
      }
      ptx::named_bar_sync(2, 256);
      if (ct == 0) tr(A, ph, 4);
      reduce_phase(A, p, P, gen, hgen, s_flag, ct);
      if (ct == 0) tr(A, ph, 5);
      if (p.kind == LA_MK_QKV) {
        // this CTA's QKV MMAs are complete: the B ring is free for attention
        ptx::named_bar_sync(2, 256);
        if (ct == 0) tr(A, nph + p.l, 0);
        attention_layer(A, P, p.l, gen, sB, reinterpret_cast<uint32_t*>(sEpi), s_flag + 1, ct);
        ptx::named_bar_sync(2, 256);
        if (ct == 0) {
          tr(A, nph + p.l, 1);
          __threadfence_block();
          *s_attn_layers = p.l + 1;
        }
      }
    }
  }

  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0 && n_rows > 0) {
    __threadfence();
    const unsigned done = atomicAdd(A.sync + A.sm.cta_done, 1u);
    if (done == (gen + 1) * gridDim.x - 1) {
      if (A.timing) {
        A.timing[1] += globaltimer() - A.timing[0];
        A.timing[2] += 1;
        A.timing[3] = 0;
      }
      __threadfence();
      if (A.do_head) atomicAdd(A.sync + A.sm.head_gen, 1u);
      atomicAdd(A.sync + A.sm.gen, 1u);
    }
  }
}

}  // namespace

size_t la_mega_smem_bytes() { return kSmemBytes; }
int la_mega_threads() { return kThreads; }

cudaError_t la_mega_launch(const LaMegaArgs& a, int grid, cudaStream_t st, bool pdl) {
  static std::atomic<unsigned> attr{0};
  cudaError_t e = la_smem_attr_once(attr, la_mega_kernel, (int)kSmemBytes);
  if (e != cudaSuccess) return e;
  return la_launch(la_mega_kernel, dim3(grid), dim3(kThreads), kSmemBytes, st, pdl, a);
}

LA_TL_DEFINE_SETTER(mega)
