// Step attention of one decoder layer (reference models.py:250-260 with the
// visibility sets of layout.py:139-170): flash attention + chunk merge in ONE
// launch (q / K / V come from la_qkv_epi_kernel).
//
// Work unit = (KV head, block of 128 query rows, key chunk).  The confirmed
// prefix (cache slots [0, ctx)) is cut into S chunks whose boundaries depend
// on ctx only, so every lookahead-parallel shard -- and the plain greedy step
// -- sums a row's keys in the same order; unit S is the step block (slots
// ctx .. ctx+n_global) under the paper's structured mask, generated per row
// from the plan's chains (a 128-bit visibility set, never an M x M matrix).
//
//  * one CTA of 8 warps covers 128 query rows (16 per warp, mma.sync bf16,
//    fp32 online softmax) so each K/V tile is read from HBM once; all tiles
//    of a chunk are issued up front into a 5-deep cp.async ring.
//  * the last chunk of (KV head, row block) to finish merges the chunk
//    partials in chunk order and writes the O-projection input (packed rows).
#include <cuda_bf16.h>

#include "la_attn.cuh"
#include "la_common.cuh"
#include "la_gemm.cuh"
#include "la_reduce_dev.cuh"
#include "la_ptx.cuh"

namespace {

constexpr int kKeyTile = 64;
constexpr int kStages = 5;                           // K/V tiles in flight
constexpr int kTileBytes = 2 * kKeyTile * 256;       // K + V of 64 keys
constexpr float kLog2e = 1.4426950408889634f;
// tensor-core path (tcgen05): a chunk of <= kTcTiles key tiles in one pass.
// smem: Q [2 dim blocks][128 rows][128 B] | K, later P [kTcTiles][16 KB] |
// V [kTcTiles][2 dim blocks][64 keys][128 B]; TMEM: S tiles at 64 columns each,
// O at columns 384..511.
constexpr int kTcTiles = 6;
constexpr int kTcQ = 0, kTcK = 32768, kTcV = kTcK + kTcTiles * 16384;
constexpr int kTcSmem = kTcV + kTcTiles * 16384;                   // 224 KB
constexpr int kMaskOff = kTcSmem > kStages * kTileBytes ? kTcSmem : kStages * kTileBytes;
constexpr int kMaskOffMma = kStages * kTileBytes;   // mma.sync-only launches
// cluster mode: 4-tile ring | pushed partials [(S+1) * rows_per <= 136][128] fp32 |
// their (m, l) | mask
constexpr int kClStages = 4;
constexpr int kClPush = kClStages * kTileBytes;
constexpr int kClPushRows = 136;
constexpr int kClPushML = kClPush + kClPushRows * 128 * 4;
constexpr int kClMaskOff = kClPushML + kClPushRows * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 256 + ((chunk ^ (row & 7)) << 4));
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
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ int chunk_keys(int ctx, int S) {
  return ((ctx + S - 1) / S + kKeyTile - 1) / kKeyTile * kKeyTile;
}
// bounded mbarrier wait (debug safety: a stuck tensor-core stage records its
// id in trace slot 7 instead of hanging the GPU)
__device__ __forceinline__ void mbar_wait_bounded(const LaAttnFusedArgs& a, uint64_t* bar, uint32_t parity, int id) {
  for (unsigned n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))), "r"(parity)
        : "memory");
    if (ok) return;
    if (n > (1u << 22)) {
      if (a.trace) a.trace[blockIdx.x * 8 + 7] = 1000 + id;
      return;
    }
  }
}

__device__ __forceinline__ void stamp(const LaAttnFusedArgs& a, int k) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    *reinterpret_cast<volatile unsigned long long*>(a.trace + blockIdx.x * 8 + k) = t;
  }
}
// stamp from the first softmax warp (tensor-core path)
__device__ __forceinline__ void stamp_w4(const LaAttnFusedArgs& a, int k) {
  if (a.trace && threadIdx.x == 128) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    *reinterpret_cast<volatile unsigned long long*>(a.trace + blockIdx.x * 8 + k) = t;
  }
}
// A query row's visible step keys as a 128-bit set (bit k = slot ctx + k): its
// chain and itself.  Chain entries are read 16 at a time with every load of a
// batch in flight together -- one L2 round trip for the lookahead rows' chains
// (<= W + N - 2 keys) instead of one dependent load per key (2.8 us of the step
// unit's start at 13B).  Entries past chain_n are read (the row holds
// LA_MAX_CHAIN) but never used.
__device__ __forceinline__ void mask_add(uint32_t (&w)[4], int key) {
#pragma unroll
  for (int q = 0; q < 4; ++q) w[q] |= (key >> 5) == q ? 1u << (key & 31) : 0u;
}
__device__ __forceinline__ uint4 row_step_mask(const FwdPlan* P, int r, int ctx) {
  const int* ch = P->chain[r];
  int k[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) k[u] = ch[u];
  const int n = P->chain_n[r];
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  mask_add(w, P->slot[r] - ctx);
#pragma unroll
  for (int u = 0; u < 16; ++u)
    if (u < n) mask_add(w, k[u] - ctx);
  for (int j0 = 16; j0 < n; j0 += 16) {
#pragma unroll
    for (int u = 0; u < 16; ++u) k[u] = ch[j0 + u];
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (j0 + u < n) mask_add(w, k[u] - ctx);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
static_assert(LA_MAX_CHAIN % 16 == 0, "chain rows are read in batches of 16");
// per-warp progress marks (debug): trace slot 6 holds one byte per warp
__device__ __forceinline__ void wmark(const LaAttnFusedArgs& a, int v) {
  if (a.trace && (a.dbg & 4) && (threadIdx.x & 31) == 0) {
    reinterpret_cast<volatile uint8_t*>(a.trace + blockIdx.x * 8 + 6)[threadIdx.x >> 5] = (uint8_t)v;
    __threadfence_system();
  }
}

}  // namespace

size_t la_attn_fused_smem(bool tc, bool cluster) {
  return (size_t)(tc ? kMaskOff : cluster ? kClMaskOff : kMaskOffMma) + LA_MAX_ROWS * 4 * 4 + 64;
}

// ---------------------------------------------------------------------------
// Tensor-core chunk unit: S = Q K^T (tcgen05, M = 128 query rows, N = 64 keys
// per tile, fp32 in TMEM) -> one-pass masked softmax by warps 4-7 (one TMEM
// lane = one query row), P (bf16) written over the K tiles -> O = P V
// (tcgen05, V as the MN-major B operand straight from its [key][dim] smem
// image) -> unnormalised O and (max, sum) in log2 units, the same partial
// format as the mma.sync path.
__device__ void attn_tc_unit(const LaAttnFusedArgs& a, const FwdPlan* P, uint8_t* smem, const uint32_t* sMask,
                             uint64_t* bars, uint32_t* tmem_slot, int kvh, int rb, int g, int nq, int ctx,
                             int k_begin, int k_end, int n_tiles, bool step_unit, float* part_o, float2* part_ml) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* sQ = smem + kTcQ;
  uint8_t* sK = smem + kTcK;
  uint8_t* sV = smem + kTcV;
  uint64_t* s_done = bars;
  uint64_t* o_done = bars + 1;
  if (tid == 0) {
    ptx::mbar_init(s_done, 1);
    ptx::mbar_init(o_done, 1);
    ptx::fence_barrier_init();
  }
  wmark(a, 1);
  if (warp == 0) ptx::tmem_alloc<512>(tmem_slot);
  wmark(a, 2);
  // ---- loads: Q rows (zero beyond the block), the chunk's K and V rows
  const size_t kv_ld = (size_t)a.KVH * 128;
  for (int i = tid; i < 128 * 16; i += 256) {
    const int row = i >> 4, c = i & 15;
    const int qr = rb * 128 + row;
    const bool ok = qr < nq;
    const __nv_bfloat16* src = ok ? a.q + ((size_t)(qr / g) * a.H + kvh * g + qr % g) * 128 + c * 8 : a.q;
    cp_async16(smem_u32(sQ + (c >> 3) * 16384 + row * 128) + (((c & 7) ^ (row & 7)) << 4), src, ok);
  }
  for (int i = tid; i < n_tiles * 64 * 16; i += 256) {
    const int t = i >> 10, row = (i >> 4) & 63, c = i & 15;
    const int key = k_begin + t * 64 + row;
    const bool ok = key < k_end;
    const size_t off = (size_t)(ok ? key : k_begin) * kv_ld + kvh * 128 + c * 8;
    const uint32_t o = t * 16384 + (c >> 3) * 8192 + row * 128 + (((c & 7) ^ (row & 7)) << 4);
    cp_async16(smem_u32(sK) + o, a.kc + off, ok);
    cp_async16(smem_u32(sV) + o, a.vc + off, ok);
  }
  cp_commit();
  cp_wait<0>();
  wmark(a, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> tensor core
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  stamp(a, 2);
  wmark(a, 4);

  // ---- S = Q K^T, one 64-column TMEM block per key tile
  if (warp == 0 && lane == 0) {
    const uint32_t idesc = ptx::umma_idesc_bf16(128, 64);
    for (int t = 0; t < ((a.dbg & 2) ? 0 : n_tiles); ++t)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        ptx::umma_bf16(tmem + t * 64,
                       ptx::umma_desc_sw128(smem_u32(sQ) + (kk >> 2) * 16384 + (kk & 3) * 32),
                       ptx::umma_desc_sw128(smem_u32(sK) + t * 16384 + (kk >> 2) * 8192 + (kk & 3) * 32),
                       idesc, kk > 0 ? 1u : 0u);
    ptx::umma_commit(s_done);
    stamp(a, 3);
  }

  // ---- softmax: all 8 warps; TMEM lane = query row (lane quadrant = warp % 4),
  // warps w and w+4 take the two halves of the row's columns and exchange the
  // row max / sum through shared memory
  const int row = (warp & 3) * 32 + lane;
  const int half = warp >> 2;
  const int ncol = n_tiles * 32;                 // columns per half (multiple of 32)
  const int cbeg = half * ncol;
  float* sRed = reinterpret_cast<float*>(smem + kTcQ);   // Q is dead once the S MMAs completed
  const uint32_t t_row = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const float sl2 = a.scale * kLog2e;
  const int nvalid = k_end - k_begin;            // columns beyond are masked
  uint32_t mw[4] = {~0u, ~0u, ~0u, ~0u};
  if (step_unit) {
    const uint4 w = *reinterpret_cast<const uint4*>(sMask + row * 4);
    mw[0] = w.x; mw[1] = w.y; mw[2] = w.z; mw[3] = w.w;
  }
  auto vis_bits = [&](int c0) -> uint32_t {
    const uint32_t r = c0 + 32 <= nvalid ? ~0u : (c0 >= nvalid ? 0u : ((1u << (nvalid - c0)) - 1u));
    return step_unit ? (r & mw[c0 >> 5]) : r;
  };
  mbar_wait_bounded(a, s_done, 0, 1);
  ptx::tc_fence_after();
  float m = -INFINITY;
  for (int c0 = cbeg; c0 < cbeg + ncol; c0 += 32) {
    float v[32];
    ptx::tmem_ld32(t_row + c0, v);
    const uint32_t vis = vis_bits(c0);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if ((vis >> j) & 1u) m = fmaxf(m, v[j]);
  }
  m *= sl2;                                       // positive scale: commutes with max
  sRed[half * 128 + row] = m;                     // (S MMAs done: Q smem is free)
  __syncthreads();
  m = fmaxf(sRed[row], sRed[128 + row]);
  const float mb = m == -INFINITY ? 0.f : m;
  float l = 0.f;
  for (int c0 = cbeg; c0 < cbeg + ncol; c0 += 32) {
    float v[32];
    ptx::tmem_ld32(t_row + c0, v);
    const uint32_t vis = vis_bits(c0);
    uint32_t pk[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const float p0 = ((vis >> j) & 1u) ? exp2f(fmaf(v[j], sl2, -mb)) : 0.f;
      const float p1 = ((vis >> (j + 1)) & 1u) ? exp2f(fmaf(v[j + 1], sl2, -mb)) : 0.f;
      l += p0 + p1;
      pk[j >> 1] = pack_bf16(p0, p1);
    }
    // P tile c0/64 overwrites K tile c0/64 (its S MMAs are complete)
    uint8_t* prow = sK + (c0 >> 6) * 16384 + row * 128;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int chunk = ((c0 & 63) >> 3) + q;
      *reinterpret_cast<uint4*>(prow + ((chunk ^ (row & 7)) << 4)) =
          make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    }
  }
  sRed[256 + half * 128 + row] = l;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // P -> tensor core
  ptx::tc_fence_before();
  __syncthreads();
  l = sRed[256 + row] + sRed[256 + 128 + row];
  stamp_w4(a, 7);
  // ---- O = P V (V: MN-major B operand, 64-dim blocks 8 KB apart, 8-key groups 1 KB apart)
  if (warp == 0 && lane == 0) {
    ptx::tc_fence_after();
    const uint32_t idesc = ptx::umma_idesc_bf16_bmn(128, 128);
    for (int t = 0; t < ((a.dbg & 1) ? 0 : n_tiles); ++t)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        ptx::umma_bf16(tmem + 384, ptx::umma_desc_sw128(smem_u32(sK) + t * 16384 + kk * 32),
                       ptx::umma_desc_sw128_mn(smem_u32(sV) + t * 16384 + kk * 2048, 8192, 1024), idesc,
                       (t > 0 || kk > 0) ? 1u : 0u);
    ptx::umma_commit(o_done);
    stamp(a, 5);
  }
  mbar_wait_bounded(a, o_done, 0, 2);
  ptx::tc_fence_after();
  {
    // tcgen05.ld is warp-collective (.sync.aligned): every lane loads, only the
    // block's valid rows store; the two warps of a quadrant split O's columns
    const bool valid = rb * 128 + row < nq;
    float4* dst = reinterpret_cast<float4*>(part_o + (size_t)row * 128);
    for (int c0 = half * 64; c0 < half * 64 + 64; c0 += 32) {
      float v[32];
      ptx::tmem_ld32(t_row + 384 + c0, v);
      if (valid) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          __stcg(dst + (c0 >> 2) + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
      }
    }
    if (valid && half == 0) __stcg(part_ml + row, make_float2(m, l));
  }
  ptx::tc_fence_before();
  wmark(a, 10);
  __syncthreads();
  wmark(a, 11);
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  wmark(a, 12);
}

// Before the dependency wait: pull unit e's prefix K/V rows into L2.  Only a
// cache hint -- if the plan or cache is not final yet the lines are merely
// refetched after the wait -- so it is always safe.  Off by default
// (LA_ATTN_KV_PF=1): one serialised bulk prefetch per 256-B row costs more
// than it hides once chunks are long (13B, 3.5K keys: attention 60 -> 51 us
// per layer without it; 7B 512-1K keys: no change).
__device__ __forceinline__ void attn_prefetch_kv(const LaAttnFusedArgs& a, int e) {
  const FwdPlan* P = a.plan;
  const int S = a.S;
  const int split = e % (S + 1);
  const int ctx = P->n_prefix;
  if (a.kv_pf && split < S && P->n_rows > 0 && ctx > 0) {
    const int kvh = e / (a.nrb_max * (S + 1));
    const int CH = chunk_keys(ctx, S);
    const int k0 = min(ctx, split * CH), k1 = min(ctx, (split + 1) * CH);
    const size_t kv_ld = (size_t)a.KVH * 128;
    for (int i = threadIdx.x; i < 2 * (k1 - k0); i += blockDim.x) {
      const int key = k0 + (i >> 1);
      const __nv_bfloat16* src = ((i & 1) ? a.vc : a.kc) + (size_t)key * kv_ld + kvh * 128;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], 256;" ::"l"(reinterpret_cast<uint64_t>(src)) : "memory");
    }
  }
}

// Cluster-mode merge: rows [r0, r1) of this CTA's share, combining the S+1
// chunk partials held in the cluster's shared memories (rank = chunk) in chunk
// order -- the same arithmetic as the global-memory merge.
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
__device__ void attn_merge_cluster(const LaAttnFusedArgs& a, uint8_t* smem, int rb, int g, int nq, int kvh,
                                   int S, int split) {
  const int tid = threadIdx.x;
  const float* sP = reinterpret_cast<const float*>(smem + kClPush);
  const float2* sM = reinterpret_cast<const float2*>(smem + kClPushML);
  const int nqb = min(128, nq - rb * 128);
  const int rows_per = (nqb + S) / (S + 1);
  const int r0 = split * rows_per, r1 = min(nqb, r0 + rows_per);
  for (int row = r0 + (tid >> 3); row < r1; row += 32) {
    const int lr = row - r0;
    const int qr = rb * 128 + row;
    const int hd = (tid & 7) * 16;
    float m = -INFINITY, ll = 0.f;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    for (int sp = 0; sp <= S; ++sp) {
      const int slot = sp * rows_per + lr;
      const float2 ml = sM[slot];
      if (ml.x == -INFINITY) continue;
      const float4* po = reinterpret_cast<const float4*>(sP + (size_t)slot * 128 + hd);
      const float4 v0 = po[0], v1 = po[1], v2 = po[2], v3 = po[3];
      const float vv[16] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w,
                            v2.x, v2.y, v2.z, v2.w, v3.x, v3.y, v3.z, v3.w};
      const float mn = fmaxf(m, ml.x);
      const float s0 = exp2f(m - mn), s1 = exp2f(ml.x - mn);
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = acc[i] * s0 + vv[i] * s1;
      ll = ll * s0 + ml.y * s1;
      m = mn;
    }
    const float inv = 1.0f / ll;
    const int r = qr / g, head = kvh * g + qr % g;
#pragma unroll
    for (int c = 0; c < 2; ++c)
      *reinterpret_cast<uint4*>(a.out + la_act_off(r, head * 128 + hd + 8 * c)) =
          make_uint4(pack_bf16(acc[8 * c] * inv, acc[8 * c + 1] * inv),
                     pack_bf16(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv),
                     pack_bf16(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv),
                     pack_bf16(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv));
  }
}

// Chunk arrival + merge of a (KV head, row block) group after every chunk
// CTA wrote its partial to global memory: spread (every chunk CTA merges a
// share of the rows once all arrived) or last-arriver (one CTA merges all).
__device__ __forceinline__ void attn_merge_rows(const LaAttnFusedArgs& a, size_t base, int count, int r0, int r1,
                                                int rb, int g, int kvh);
__device__ __forceinline__ void attn_arrive_merge(const LaAttnFusedArgs& a, int* sFlag, size_t grp, int S, int split,
                                  int rb, int g, int nq, int kvh, bool spread) {
  const int tid = threadIdx.x;
  __syncthreads();
  // arrival of this chunk.  Counters only grow: an active group gains exactly
  // S+1 per launch, so the group's target is the next multiple of S+1.
  if (tid == 0) {
    __threadfence();
    const unsigned old = atomicAdd(a.cnt + grp, 1u);
    const unsigned target = (old / (unsigned)(S + 1) + 1) * (unsigned)(S + 1);
    if (spread) {
      // every chunk CTA of the group is resident (grid <= SMs, 1 CTA / SM):
      // wait for the others, then merge this chunk's share of the rows
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.cnt + grp) : "memory");
        if ((int)(v - target) < 0) __nanosleep(64);
      } while ((int)(v - target) < 0);
      *sFlag = 1;
    } else {
      *sFlag = old + 1 == target;   // the last chunk merges every row
      if (*sFlag) __threadfence();
    }
  }
  __syncthreads();
  stamp(a, 5);
  if (!*sFlag) return;

  // ---- merge the S+1 chunk partials of this group in chunk order: rows
  // [r0, r1) of the group's valid rows
  const int nqb = min(128, nq - rb * 128);
  const int rows_per = spread ? (nqb + S) / (S + 1) : nqb;
  const int r0 = spread ? split * rows_per : 0;
  const int r1 = min(nqb, r0 + rows_per);
  attn_merge_rows(a, grp * (S + 1), S + 1, r0, r1, rb, g, kvh);
}

// Merge partial slots [base, base + count) in slot order into the attention
// output for rows [r0, r1) of row block rb, 8 threads per row x 16 dims
__device__ __forceinline__ void attn_merge_rows(const LaAttnFusedArgs& a, size_t base, int count, int r0, int r1,
                                                int rb, int g, int kvh) {
  const int tid = threadIdx.x;
  for (int row = r0 + (tid >> 3); row < r1; row += 32) {
    const int qr = rb * 128 + row;
    const int hd = (tid & 7) * 16;
    float m = -INFINITY, ll = 0.f;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    // partials in batches of 4 with every load of a batch in flight together
    // (a dependent L2 round trip per partial otherwise); same combine order
    for (int sp0 = 0; sp0 < count; sp0 += 4) {
      float2 mlv[4];
      float4 pv[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int sp = sp0 + j;
        if (sp < count) {
          const size_t us = base + sp;
          mlv[j] = __ldcg(a.part_ml + us * 128 + row);
          const float4* po = reinterpret_cast<const float4*>(a.part_o + (us * 128 + row) * 128 + hd);
#pragma unroll
          for (int q = 0; q < 4; ++q) pv[j][q] = __ldcg(po + q);
        } else {
          mlv[j] = make_float2(-INFINITY, 0.f);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 ml = mlv[j];
        if (ml.x == -INFINITY) continue;
        const float mn = fmaxf(m, ml.x);
        const float s0 = exp2f(m - mn), s1 = exp2f(ml.x - mn);
        const float vv[16] = {pv[j][0].x, pv[j][0].y, pv[j][0].z, pv[j][0].w,
                              pv[j][1].x, pv[j][1].y, pv[j][1].z, pv[j][1].w,
                              pv[j][2].x, pv[j][2].y, pv[j][2].z, pv[j][2].w,
                              pv[j][3].x, pv[j][3].y, pv[j][3].z, pv[j][3].w};
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = acc[i] * s0 + vv[i] * s1;
        ll = ll * s0 + ml.y * s1;
        m = mn;
      }
    }
    const float inv = 1.0f / ll;
    const int r = qr / g, head = kvh * g + qr % g;
#pragma unroll
    for (int c = 0; c < 2; ++c)
      *reinterpret_cast<uint4*>(a.out + la_act_off(r, head * 128 + hd + 8 * c)) =
          make_uint4(pack_bf16(acc[8 * c] * inv, acc[8 * c + 1] * inv),
                     pack_bf16(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv),
                     pack_bf16(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv),
                     pack_bf16(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv));
  }
}

// K/V tile t of [k_begin, k_end) into ring slot t % STAGES (cp.async, rows past
// k_end zero-filled)
template <int STAGES>
__device__ __forceinline__ void attn_load_kv(const LaAttnFusedArgs& a, uint8_t* sKV, int t, int k_begin,
                                             int k_end, int kvh) {
  uint8_t* kb = sKV + (t % STAGES) * kTileBytes;
  const size_t kv_ld = (size_t)a.KVH * 128;
  const int t0 = k_begin + t * kKeyTile;
  for (int i = threadIdx.x; i < kKeyTile * 16; i += 256) {
    const int row = i >> 4, ch = i & 15, key = t0 + row;
    const bool ok = key < k_end;
    const size_t off = ((size_t)(ok ? key : k_begin) * kv_ld) + kvh * 128 + ch * 8;
    cp_async16(smem_u32(kb) + swz(row, ch), a.kc + off, ok);
    cp_async16(smem_u32(kb + kKeyTile * 256) + swz(row, ch), a.vc + off, ok);
  }
}

// Before the dependency wait (graph-loop decode only, a.spec_ctx set): start the
// first STAGES-1 prefix tiles of unit e for the decode state's ctx.  ctx and the
// prefix K/V were final when this loop iteration began (written by K10 / the KV
// commit of the previous step); the unit checks the guess against its plan after
// the wait and reloads on a mismatch.  Returns the guessed ctx, or -1 (no issue).
template <int STAGES>
__device__ __forceinline__ int attn_spec_issue(const LaAttnFusedArgs& a, uint8_t* smem, int e) {
  const int S = a.S;
  const int split = e % (S + 1);
  if (split == S || (e / (S + 1)) % a.nrb_max != 0) return -1;
  const int ctx = *reinterpret_cast<const volatile int*>(a.spec_ctx);
  const int kvh = e / (a.nrb_max * (S + 1));
  const int CH = chunk_keys(ctx, S);
  const int k_begin = min(ctx, split * CH), k_end = min(ctx, (split + 1) * CH);
  const int n_tiles = (k_end - k_begin + kKeyTile - 1) / kKeyTile;
#pragma unroll 1
  for (int t = 0; t < STAGES - 1; ++t) {
    if (t < n_tiles) attn_load_kv<STAGES>(a, smem, t, k_begin, k_end, kvh);
    cp_commit();
  }
  return ctx;
}

// One attention unit e = (KV head, row block, key chunk) after the dependency
// wait, on a K/V ring of STAGES tiles at smem (plus the mask at mask_off).
// spec >= 0: attn_spec_issue already started the first tiles for ctx == spec.
template <int STAGES, bool CLUSTER = false>
__device__ void attn_unit(const LaAttnFusedArgs& a, uint8_t* smem, int e, int spec = -1) {
  stamp(a, 1);
  const FwdPlan* P = a.plan;
  const int n_rows = P->n_rows, ctx = P->n_prefix;
  // a wrong guess (or nothing to do): drain the speculative copies first
  const bool spec_hit = spec >= 0 && spec == ctx && n_rows > 0;
  if (spec >= 0 && !spec_hit) cp_wait<0>();
  if (n_rows == 0) return;
  const int g = a.H / a.KVH;
  const int nq = n_rows * g;
  const int n_rb = (nq + 127) >> 7;
  const int S = a.S;
  const int kvh = e / (a.nrb_max * (S + 1));
  const int rb = (e / (S + 1)) % a.nrb_max;
  const int split = e % (S + 1);
  const bool active = rb < n_rb;
  // co-residency of a group's chunk CTAs: guaranteed when the whole grid fits
  // the SMs, or when the active units do (inactive CTAs exit at once)
  const bool spread = a.spread_merge || (a.sms > 0 && a.KVH * n_rb * (S + 1) <= a.sms);
  const bool step_unit = split == S;
  int k_begin, k_end;
  if (step_unit) {
    k_begin = ctx;
    k_end = ctx + P->n_global;
  } else {
    const int CH = chunk_keys(ctx, S);
    k_begin = min(ctx, split * CH);
    k_end = min(ctx, (split + 1) * CH);
  }

  uint8_t* sKV = smem;                                                   // [STAGES][K | V]
  uint32_t* sMask = reinterpret_cast<uint32_t*>(smem + (a.tc ? kMaskOff : CLUSTER ? kClMaskOff : STAGES * kTileBytes));   // [128][4]
  int* sFlag = reinterpret_cast<int*>(sMask + LA_MAX_ROWS * 4);
  uint64_t* sBars = reinterpret_cast<uint64_t*>(sFlag + 4);           // tensor-core path
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(sBars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t kv_ld = (size_t)a.KVH * 128;
  const int n_tiles = (k_end - k_begin + kKeyTile - 1) / kKeyTile;
  // tensor-core path when the chunk fits TMEM (<= 6 key tiles) and smem is
  // 1024-B aligned (SW128 atoms); chunking depends on ctx only, so the path
  // choice -- and every row's summation order -- is the same for every shard
  const bool tc = a.tc && n_tiles <= kTcTiles && (smem_u32(smem) & 1023u) == 0u;

  auto load_kv = [&](int t) {
    uint8_t* kb = sKV + (t % STAGES) * kTileBytes;
    const int t0 = k_begin + t * kKeyTile;
    for (int i = tid; i < kKeyTile * 16; i += 256) {
      const int row = i >> 4, ch = i & 15, key = t0 + row;
      const bool ok = key < k_end;
      const size_t off = ((size_t)(ok ? key : k_begin) * kv_ld) + kvh * 128 + ch * 8;
      cp_async16(smem_u32(kb) + swz(row, ch), a.kc + off, ok);
      cp_async16(smem_u32(kb + kKeyTile * 256) + swz(row, ch), a.vc + off, ok);
    }
  };
  // prefix keys are cached K/V of earlier steps: start streaming them now
  // (before the QKV epilogue), the step block's keys only after it
  auto issue_first = [&]() {
#pragma unroll 1
    for (int t = 0; t < STAGES - 1; ++t) {
      if (t < n_tiles) load_kv(t);
      cp_commit();
    }
  };
  // ---- q fragments straight from global (m16n8k16 A layout); issued before
  // the K/V ring so their L2 latency overlaps the cp.async issue
  const int qrow0 = warp * 16 + (lane >> 2);
  uint32_t qf[8][4];
  auto load_q = [&]() {
    const int qa = rb * 128 + qrow0, qb = qa + 8;
    const __nv_bfloat16* pa = qa < nq ? a.q + ((size_t)(qa / g) * a.H + kvh * g + qa % g) * 128 : nullptr;
    const __nv_bfloat16* pb = qb < nq ? a.q + ((size_t)(qb / g) * a.H + kvh * g + qb % g) * 128 : nullptr;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int col = kk * 16 + (lane & 3) * 2;
      qf[kk][0] = pa ? __ldcg(reinterpret_cast<const unsigned*>(pa + col)) : 0u;
      qf[kk][1] = pb ? __ldcg(reinterpret_cast<const unsigned*>(pb + col)) : 0u;
      qf[kk][2] = pa ? __ldcg(reinterpret_cast<const unsigned*>(pa + col + 8)) : 0u;
      qf[kk][3] = pb ? __ldcg(reinterpret_cast<const unsigned*>(pb + col + 8)) : 0u;
    }
  };
  if (active && !tc && !a.fuse_qkv) load_q();
  if (active && !step_unit && !tc && !spec_hit) issue_first();
  if (a.fuse_qkv) {
    // QKV split-K epilogue (la_qkv_fix) spread over every CTA of the grid,
    // then a grid barrier: all CTAs are resident (grid <= SMs, 1 CTA / SM)
    const int T = a.H + 2 * a.KVH;
    const long total = (long)T * n_rows * 16;
    for (long idx = (long)blockIdx.x * 256 + tid; idx < total; idx += (long)gridDim.x * 256)
      la_qkv_fix(a.qkv, P, (int)(idx / ((long)n_rows * 16)), (int)((idx >> 4) % n_rows));
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const unsigned old = atomicAdd(a.gbar, 1u);
      const unsigned target = (old / gridDim.x + 1) * gridDim.x;
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.gbar) : "memory");
        if ((int)(v - target) < 0) __nanosleep(32);
      } while ((int)(v - target) < 0);
    }
    __syncthreads();
  }
  if (!active) return;
  const size_t grp = (size_t)kvh * a.nrb_max + rb;
  if (step_unit) {
    // the step block's K/V (written by the QKV epilogue before the wait) stream
    // in while the mask is built
    if (!tc && !a.fuse_qkv) issue_first();
    // structured mask: a query row sees its chain's step keys and itself;
    // one thread per row builds its 128-bit set in registers (independent loads)
    if (tid < LA_MAX_ROWS) {
      const int qr = rb * 128 + tid;
      *reinterpret_cast<uint4*>(sMask + tid * 4) =
          qr < nq ? row_step_mask(P, qr / g, ctx) : make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
  }

  if (tc) {
    attn_tc_unit(a, P, smem, sMask, sBars, sTmem, kvh, rb, g, nq, ctx, k_begin, k_end, n_tiles, step_unit,
                 a.part_o + (grp * (S + 1) + split) * 128 * 128, a.part_ml + (grp * (S + 1) + split) * 128);
  } else {
    if (step_unit && a.fuse_qkv) issue_first();

    if (a.fuse_qkv) load_q();   // q is produced by the fused epilogue above

    float o[16][4];
  #pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    const float sl2 = a.scale * kLog2e;
    stamp(a, 2);
    const bool warp_active = rb * 128 + warp * 16 < nq;

    for (int t = 0; t < n_tiles; ++t) {
      if (t + STAGES - 1 < n_tiles) load_kv(t + STAGES - 1);
      cp_commit();
      cp_wait<STAGES - 1>();
      __syncthreads();
      if (t == 0) stamp(a, 3);
      if (warp_active) {
        const uint8_t* sK = sKV + (t % STAGES) * kTileBytes;
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
            ldsm_x4(smem_u32(sK) + swz(key, ch), b0, b1, b2, b3);
            mma16816(s[2 * np], qf[kk], b0, b1);
            mma16816(s[2 * np + 1], qf[kk], b2, b3);
          }
        }
        // 64-key visibility of this thread's two rows: the key range, and for
        // the step block the rows' structured-mask words; pre-shifted by the
        // lane's column so the per-element bit index is a constant
        const int kbase = k_begin + t * kKeyTile;
        const int nvalid = min(kKeyTile, k_end - kbase);
        unsigned long long vm0 = nvalid >= 64 ? ~0ull : ((1ull << nvalid) - 1ull), vm1 = vm0;
        if (step_unit) {
          const uint32_t* w0 = sMask + qrow0 * 4 + 2 * t;
          const uint32_t* w1 = sMask + (qrow0 + 8) * 4 + 2 * t;
          vm0 &= ((unsigned long long)w0[1] << 32) | w0[0];
          vm1 &= ((unsigned long long)w1[1] << 32) | w1[0];
        }
        vm0 >>= (lane & 3) * 2;
        vm1 >>= (lane & 3) * 2;
        float mx0 = m0, mx1 = m1;
  #pragma unroll
        for (int n = 0; n < 8; ++n) {
  #pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const unsigned long long vm = (e2 >> 1) ? vm1 : vm0;
            const bool vis = (vm >> (n * 8 + (e2 & 1))) & 1ull;
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
            ldsm_x4_t(smem_u32(sV) + swz(key, ch), v0, v1, v2, v3);
            mma16816(o[2 * dp], pa, v0, v1);
            mma16816(o[2 * dp + 1], pa, v2, v3);
          }
        }
      }
      __syncthreads();
    }
    cp_wait<0>();
    stamp(a, 4);

    // ---- chunk partial: unnormalised O and (m, l) in log2 units
  #pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    // cluster mode: push each row's partial straight into the smem of the
    // chunk CTA that merges it (rank row / rows_per), slot [chunk][local row]
    const int nqb_ = min(128, nq - rb * 128);
    const int rows_per_ = (nqb_ + S) / (S + 1);
  #pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int row = qrow0 + half * 8;
      if (rb * 128 + row >= nq) continue;
      if constexpr (CLUSTER) {
        const unsigned owner = (unsigned)(row / rows_per_);
        const int slot = split * rows_per_ + (row - (int)owner * rows_per_);
        const uint32_t dst = dsmem_addr(smem + kClPush + (size_t)slot * 512, owner);
  #pragma unroll
        for (int dd = 0; dd < 16; ++dd) {
          const int col = dd * 8 + (lane & 3) * 2;
          asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};"
                       :: "r"(dst + col * 4), "f"(o[dd][half * 2]), "f"(o[dd][half * 2 + 1]) : "memory");
        }
        if ((lane & 3) == 0) {
          const float2 ml = make_float2(half ? m1 : m0, half ? l1 : l0);
          asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};"
                       :: "r"(dsmem_addr(smem + kClPushML + slot * 8, owner)), "f"(ml.x), "f"(ml.y) : "memory");
        }
        continue;
      }
      float* dst = a.part_o + ((grp * (S + 1) + split) * 128 + row) * 128;
  #pragma unroll
      for (int dd = 0; dd < 16; ++dd) {
        const int col = dd * 8 + (lane & 3) * 2;
        __stcg(reinterpret_cast<float2*>(dst + col), make_float2(o[dd][half * 2], o[dd][half * 2 + 1]));
      }
      if ((lane & 3) == 0)
        __stcg(a.part_ml + (grp * (S + 1) + split) * 128 + row, make_float2(half ? m1 : m0, half ? l1 : l0));
    }
  }
  if constexpr (CLUSTER) {
    // every chunk CTA of the group is in this cluster: one barrier makes the
    // pushed partials visible; each CTA then merges its rows from local smem
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    stamp(a, 5);
    attn_merge_cluster(a, smem, rb, g, nq, kvh, S, split);
    stamp(a, 6);
    return;
  }
  attn_arrive_merge(a, sFlag, grp, S, split, rb, g, nq, kvh, spread);
  stamp(a, 6);
}

// grid = KVH * nrb_max * (S + 1) units, block = 256 (8 warps x 16 query rows)
__global__ void __launch_bounds__(256, 1) la_attn_fused_kernel(LaAttnFusedArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  stamp(a, 0);
  la_pdl_trigger();
  la_l2_prefetch_gemm(a.pf);
  attn_prefetch_kv(a, blockIdx.x);
  const int spec = a.spec_ctx && !a.tc && !a.fuse_qkv ? attn_spec_issue<kStages>(a, smem, blockIdx.x) : -1;
  la_pdl_wait();
  attn_unit<kStages>(a, smem, blockIdx.x, spec);
  if (a.dbg & 8) {   // timing experiment: 5 us of extra attention time per CTA
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); } while (t - t0 < 5000ull);
  }
}

// LA_ATTN_CLUSTER=1 variant: launched as clusters of S+1 CTAs (one per
// (KV head, row block)), partials pushed into the merging CTA's smem
__global__ void __launch_bounds__(256, 1) la_attn_cluster_kernel(LaAttnFusedArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  la_pdl_trigger();
  attn_prefetch_kv(a, blockIdx.x);
  la_pdl_wait();
  attn_unit<kClStages, true>(a, smem, blockIdx.x);
}

// ---------------------------------------------------------------------------
// Key-split variant (LA_ATTN_KSPLIT=1).  A chunk's key tiles are split by
// parity: every row's chunk partial is (online softmax over the even tiles)
// combined with (online softmax over the odd tiles), in that order.  Row
// blocks of <= 64 rows run the two parities at once on the two warp groups
// (one warp of each pair even tiles, the other odd; 2 tiles per ring slot) --
// the idle half of the CTA joins the long serial tile chain; larger blocks stream the
// tiles even-first then odd on all 8 warps and park the even state in smem
// at the switch.  A row's arithmetic is the same in both modes (and for every
// row count), so the mode is a per-CTA choice.
namespace {
constexpr int kKsPairSlots = 3;                                  // concurrent: 3 x 2 tiles
constexpr int kKsSeqSlots = 4;                                   // sequential: 4 tiles + stash
constexpr int kKsStashOff = kKsSeqSlots * kTileBytes;            // sequential stash (conc: offset 0)
constexpr int kKsStash = 68;                                     // o[16][4], m0, m1, l0, l1 per thread
constexpr int kKsMaskOff = kKsStashOff + 256 * kKsStash * 4;
static_assert(kKsMaskOff >= 2 * kKsPairSlots * kTileBytes, "pair ring overlaps the mask");
constexpr int kKsSmem = kKsMaskOff + LA_MAX_ROWS * 4 * 4 + 128;
constexpr int kKsSmemTma = kKsSmem + 1024;                      // 1024-B aligned ring (SW128 boxes)
}  // namespace

// TMA: each 64-key tile lands as 4 SW128 boxes [K d0-63 | K d64-127 | V d0-63 |
// V d64-127] of [64 keys][128 B]; cp.async: [K | V] rows of 256 B (swz)
template <bool TMA>
__device__ __forceinline__ uint32_t ks_swz(int row, int ch) {
  if constexpr (TMA) return (uint32_t)((ch >> 3) * 8192 + row * 128 + (((ch & 7) ^ (row & 7)) << 4));
  else return swz(row, ch);
}

// one 64-key tile of QK^T -> masked online softmax -> PV for a warp's 16 rows
template <bool TMA>
__device__ __forceinline__ void ks_tile(const uint8_t* sK, const uint32_t (&qf)[8][4], float (&o)[16][4],
                                        float& m0, float& m1, float& l0, float& l1, int lane, int nvalid,
                                        const uint32_t* w0, const uint32_t* w1, float sl2) {
  const uint8_t* sV = sK + kKeyTile * 256;   // both layouts: V at +16 KB
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
      ldsm_x4(smem_u32(sK) + ks_swz<TMA>(key, ch), b0, b1, b2, b3);
      mma16816(s[2 * np], qf[kk], b0, b1);
      mma16816(s[2 * np + 1], qf[kk], b2, b3);
    }
  }
  unsigned long long vm0 = nvalid >= 64 ? ~0ull : ((1ull << nvalid) - 1ull), vm1 = vm0;
  if (w0) {
    vm0 &= ((unsigned long long)w0[1] << 32) | w0[0];
    vm1 &= ((unsigned long long)w1[1] << 32) | w1[0];
  }
  vm0 >>= (lane & 3) * 2;
  vm1 >>= (lane & 3) * 2;
  float mx0 = m0, mx1 = m1;
#pragma unroll
  for (int n = 0; n < 8; ++n) {
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      const unsigned long long vm = (e2 >> 1) ? vm1 : vm0;
      const bool vis = (vm >> (n * 8 + (e2 & 1))) & 1ull;
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
                      pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
    for (int dp = 0; dp < 8; ++dp) {
      const int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      const int ch = dp * 2 + (lane >> 4);
      uint32_t v0, v1, v2, v3;
      ldsm_x4_t(smem_u32(sV) + ks_swz<TMA>(key, ch), v0, v1, v2, v3);
      mma16816(o[2 * dp], pa, v0, v1);
      mma16816(o[2 * dp + 1], pa, v2, v3);
    }
  }
}

// park / restore a thread's softmax state ([element][thread] words)
__device__ __forceinline__ void ks_stash(float* st, int stride, const float (&o)[16][4], float m0, float m1,
                                         float l0, float l1) {
#pragma unroll
  for (int dd = 0; dd < 16; ++dd)
#pragma unroll
    for (int c = 0; c < 4; ++c) st[(dd * 4 + c) * stride] = o[dd][c];
  st[64 * stride] = m0;
  st[65 * stride] = m1;
  st[66 * stride] = l0;
  st[67 * stride] = l1;
}

// state = even-tile state combined with odd-tile state -- always in that
// order and with explicit roundings, whichever of the two sits in registers
__device__ __forceinline__ void ks_combine(float (&o)[16][4], float& m0, float& m1, float& l0, float& l1,
                                           const float* st, int stride, bool regs_odd) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float ms = st[(64 + h) * stride], ls = st[(66 + h) * stride];
    const float mr = h ? m1 : m0, lr = h ? l1 : l0;
    const float me = regs_odd ? ms : mr, mo = regs_odd ? mr : ms;
    const float le = regs_odd ? ls : lr, lo = regs_odd ? lr : ls;
    const float mn = fmaxf(me, mo);
    const float b = mn == -INFINITY ? 0.f : mn;
    const float se = exp2f(me - b), so = exp2f(mo - b);
    const float ln = __fmaf_rn(le, se, __fmul_rn(lo, so));
#pragma unroll
    for (int dd = 0; dd < 16; ++dd)
#pragma unroll
      for (int c = 2 * h; c < 2 * h + 2; ++c) {
        const float xs = st[(dd * 4 + c) * stride], xr = o[dd][c];
        const float xe = regs_odd ? xs : xr, xo = regs_odd ? xr : xs;
        o[dd][c] = __fmaf_rn(xe, se, __fmul_rn(xo, so));
      }
    if (h) { m1 = mn; l1 = ln; } else { m0 = mn; l0 = ln; }
  }
}

// One key segment of a (KV head, row block): prefix keys [k_begin, k_end) then,
// for the step unit, the step block [ctx, ctx + n_global) under the lookahead
// mask; its partial (o, m, l) goes to partial slot `pslot`.  reinit: a second
// segment of the same CTA (flat mapping) re-arms the TMA barriers first.
template <bool TMA, bool FLAT>
__device__ void ks_segment(const LaAttnFusedArgs& a, uint8_t* smem, const FwdPlan* P, int ctx, int nq, int g,
                           int kvh, int rb, int k_begin, int k_end, bool step_unit, size_t pslot, bool reinit) {
  const int n_pre = (k_end - k_begin + kKeyTile - 1) / kKeyTile;
  const int s_end = ctx + P->n_global;
  const int nqb = min(128, nq - rb * 128);
  const bool conc = nqb <= 64;

  uint8_t* sKV = smem;
  uint32_t* sMask = reinterpret_cast<uint32_t*>(smem + kKsMaskOff);   // [128][4]
  int* sFlag = reinterpret_cast<int*>(sMask + LA_MAX_ROWS * 4);
  uint64_t* sBar = reinterpret_cast<uint64_t*>(sFlag + 4);            // TMA: one per tile slot
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t kv_ld = (size_t)a.KVH * 128;
  const int n_tiles = n_pre + (step_unit ? (P->n_global + kKeyTile - 1) / kKeyTile : 0);
  const int ne = (n_tiles + 1) >> 1;                 // even tiles
  auto tile_key0 = [&](int t) { return t < n_pre ? k_begin + t * kKeyTile : ctx + (t - n_pre) * kKeyTile; };
  auto tile_end = [&](int t) { return t < n_pre ? k_end : s_end; };
  // concurrent: blocks of <= 32 rows pair warps (2k, 2k+1) on a 16-row slice so
  // the active warps spread over all four SM sub-partitions (warp % 4; 13B
  // greedy step -4.5 %); 33-64 rows use warps w and w + 4 (measured faster there)
  const bool narrow = nqb <= 32;
  const int par = conc ? (narrow ? warp & 1 : warp >> 2) : 0;
  const int wrow = conc ? (narrow ? warp >> 1 : warp & 3) : warp;
  const int n_items = conc ? ne : n_tiles;

  const uint64_t pol = TMA ? ptx::policy_evict_first() : 0ull;
  auto load_tile = [&](int t, uint8_t* kb) {
    const int t0 = tile_key0(t), te = tile_end(t);
    if constexpr (TMA) {
      // keys past k_end load real (finite) cache rows; the mask drops them
      if (tid == 0) {
        uint64_t* bar = sBar + (kb - sKV) / kTileBytes;
        ptx::mbar_expect_tx(bar, kTileBytes);
        const int row = a.kv_row0 + t0;
        ptx::tma_load_2d(kb, a.kmap, bar, kvh * 128, row, pol);
        ptx::tma_load_2d(kb + 8192, a.kmap, bar, kvh * 128 + 64, row, pol);
        ptx::tma_load_2d(kb + 16384, a.vmap, bar, kvh * 128, row, pol);
        ptx::tma_load_2d(kb + 24576, a.vmap, bar, kvh * 128 + 64, row, pol);
      }
      return;
    }
    for (int i = tid; i < kKeyTile * 16; i += 256) {
      const int row = i >> 4, ch = i & 15, key = t0 + row;
      const bool ok = key < te;
      const size_t off = ((size_t)(ok ? key : t0) * kv_ld) + kvh * 128 + ch * 8;
      cp_async16(smem_u32(kb) + swz(row, ch), a.kc + off, ok);
      cp_async16(smem_u32(kb + kKeyTile * 256) + swz(row, ch), a.vc + off, ok);
    }
  };
  // item: concurrent = tiles (2i, 2i+1) in pair slot i % 3; sequential = the
  // i-th tile of the order 0, 2, 4, ..., 1, 3, ... in slot i % 4
  auto load_item = [&](int it) {
    if (conc) {
      uint8_t* kb = sKV + (it % kKsPairSlots) * 2 * kTileBytes;
      if (2 * it < n_tiles) load_tile(2 * it, kb);
      if (2 * it + 1 < n_tiles) load_tile(2 * it + 1, kb + kTileBytes);
    } else {
      load_tile(it < ne ? 2 * it : 2 * (it - ne) + 1, sKV + (it % kKsSeqSlots) * kTileBytes);
    }
  };
  const int depth = conc ? kKsPairSlots - 1 : kKsSeqSlots - 1;
  auto issue_first = [&]() {
#pragma unroll 1
    for (int it = 0; it < depth; ++it) {
      if (it < n_items) load_item(it);
      cp_commit();
    }
  };
  const int qrow0 = wrow * 16 + (lane >> 2);
  uint32_t qf[8][4];
  {
    const int qa = rb * 128 + qrow0, qb = qa + 8;
    const __nv_bfloat16* pa = qa < nq ? a.q + ((size_t)(qa / g) * a.H + kvh * g + qa % g) * 128 : nullptr;
    const __nv_bfloat16* pb = qb < nq ? a.q + ((size_t)(qb / g) * a.H + kvh * g + qb % g) * 128 : nullptr;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int col = kk * 16 + (lane & 3) * 2;
      qf[kk][0] = pa ? __ldcg(reinterpret_cast<const unsigned*>(pa + col)) : 0u;
      qf[kk][1] = pb ? __ldcg(reinterpret_cast<const unsigned*>(pb + col)) : 0u;
      qf[kk][2] = pa ? __ldcg(reinterpret_cast<const unsigned*>(pa + col + 8)) : 0u;
      qf[kk][3] = pb ? __ldcg(reinterpret_cast<const unsigned*>(pb + col + 8)) : 0u;
    }
  }
  if (FLAT && reinit) __syncthreads();   // the previous segment's stash reads are done
  if (TMA && tid == 0) {
    for (int i = 0; i < 2 * kKsPairSlots; ++i) {
      if (FLAT && reinit) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(sBar + i)) : "memory");
      ptx::mbar_init(sBar + i, 1);
    }
    ptx::fence_barrier_init();
  }
  // every tile of this unit is final after the dependency wait (the step
  // block's K / V too): start the ring now, the step unit's mask meanwhile
  issue_first();
  if (!step_unit && TMA) __syncthreads();   // barrier inits visible before any wait
  if (step_unit) {
    if (tid < LA_MAX_ROWS) {
      const int qr = rb * 128 + tid;
      *reinterpret_cast<uint4*>(sMask + tid * 4) =
          qr < nq ? row_step_mask(P, qr / g, ctx) : make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
  }

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = a.scale * kLog2e;
  const bool warp_active = rb * 128 + wrow * 16 < nq;
  float* seq_st = reinterpret_cast<float*>(smem + kKsStashOff) + tid;
  stamp(a, 2);
  for (int it = 0; it < n_items; ++it) {
    if (it + depth < n_items) load_item(it + depth);
    cp_commit();
    if constexpr (!TMA) {
      if (conc) cp_wait<kKsPairSlots - 1>(); else cp_wait<kKsSeqSlots - 1>();
      __syncthreads();
    }
    if (it == 0) stamp(a, 3);
    int t, slot;
    uint32_t phase;
    if (conc) {
      t = 2 * it + par;
      slot = (it % kKsPairSlots) * 2 + par;
      phase = (it / kKsPairSlots) & 1;
    } else {
      t = it < ne ? 2 * it : 2 * (it - ne) + 1;
      slot = it % kKsSeqSlots;
      phase = (it / kKsSeqSlots) & 1;
    }
    const uint8_t* sK = sKV + slot * kTileBytes;
    if (TMA && t < n_tiles) ptx::mbar_wait(sBar + slot, phase);
    if (!conc) {
      if (it == ne) {   // even tiles done: park their state, start the odd ones
        ks_stash(seq_st, 256, o, m0, m1, l0, l1);
#pragma unroll
        for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
        m0 = m1 = -INFINITY;
        l0 = l1 = 0.f;
      }
    }
    if (warp_active && t < n_tiles) {
      const int nvalid = min(kKeyTile, tile_end(t) - tile_key0(t));
      const bool masked = t >= n_pre;   // a step-block tile: the structured mask applies
      const uint32_t* w0 = masked ? sMask + qrow0 * 4 + 2 * (t - n_pre) : nullptr;
      const uint32_t* w1 = masked ? sMask + (qrow0 + 8) * 4 + 2 * (t - n_pre) : nullptr;
      ks_tile<TMA>(sK, qf, o, m0, m1, l0, l1, lane, nvalid, w0, w1, sl2);
    }
    __syncthreads();
  }
  cp_wait<0>();
  stamp(a, 4);
  if (conc) {
    // odd group parks its state in the drained ring; the even group combines
    float* st = reinterpret_cast<float*>(smem) + wrow * 32 + lane;
    if (par) ks_stash(st, 128, o, m0, m1, l0, l1);
    __syncthreads();
    if (!par) ks_combine(o, m0, m1, l0, l1, st, 128, false);
  } else {
    if (n_items <= ne) {   // no odd tile: the registers hold the even state
      ks_stash(seq_st, 256, o, m0, m1, l0, l1);
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
    }
    ks_combine(o, m0, m1, l0, l1, seq_st, 256, true);
  }
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }
  if (!par) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int row = qrow0 + half * 8;
      if (rb * 128 + row >= nq) continue;
      float* dst = a.part_o + (pslot * 128 + row) * 128;
#pragma unroll
      for (int dd = 0; dd < 16; ++dd) {
        const int col = dd * 8 + (lane & 3) * 2;
        __stcg(reinterpret_cast<float2*>(dst + col), make_float2(o[dd][half * 2], o[dd][half * 2 + 1]));
      }
      if ((lane & 3) == 0)
        __stcg(a.part_ml + pslot * 128 + row, make_float2(half ? m1 : m0, half ? l1 : l0));
    }
  }
}


// Flat mapping (a.flat): the prefix tiles of all KV heads, head-major, are cut
// into gridDim.x (or fewer, >= 1 tile each) contiguous ranges, one per CTA --
// every SM streams about the same number of tiles whatever KVH (13B: 40 heads
// x 3 chunk units left 28 SMs idle).  A range spanning two heads is two
// segments; the CTA holding a head's last prefix tile also takes its step
// block.  The cut depends on ctx, KVH and the grid only, so every row of a
// step -- and the same row in a greedy step -- sees the same key partition;
// the head's partials merge in range order.  All CTAs are co-resident (grid <=
// SMs, one CTA per SM): each waits for its heads' segments, merges its share
// of their rows, and the head's last merger re-zeroes the head's counters.
template <bool TMA>
__device__ void attn_flat_ks(const LaAttnFusedArgs& a, uint8_t* smem_raw) {
  stamp(a, 1);
  const FwdPlan* P = a.plan;
  const int n_rows = P->n_rows, ctx = P->n_prefix;
  if (n_rows == 0) return;
  const int g = a.H / a.KVH;
  const int nq = min(128, n_rows * g);   // one row block (flat needs nrb_max == 1)
  const long T = max(1, (ctx + kKeyTile - 1) / kKeyTile);   // a virtual tile when ctx == 0
  const long total = (long)a.KVH * T;
  const long G = min((long)gridDim.x, total);
  const int e = blockIdx.x;
  if (e >= G) return;
  auto owner = [&](long x) { return (int)(((x + 1) * G - 1) / total); };   // the CTA holding tile x
  const long lo = e * total / G, hi = (e + 1) * total / G;
  uint8_t* smem = TMA ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) : smem_raw;
  const int tid = threadIdx.x;
  int hs[2], ps[2], ns[2], nseg = 0;
  for (long x = lo; x < hi && nseg < 2;) {
    const int h = (int)(x / T);
    const long hend = min(hi, (h + 1) * T);
    const int f = owner(h * T);
    const int kb = (int)(x - h * T) * kKeyTile, ke = (int)(hend - h * T) * kKeyTile;
    ks_segment<TMA, true>(a, smem, P, ctx, nq, g, h, 0, min(ctx, kb), min(ctx, ke), hend == (h + 1) * T,
                    (size_t)h * a.flat_maxp + (e - f), nseg > 0);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(a.fcnt + h, 1u);
    }
    hs[nseg] = h;
    ps[nseg] = e - f;
    ns[nseg] = owner((h + 1) * T - 1) - f + 1;
    ++nseg;
    x = hend;
  }
  for (int i = 0; i < nseg; ++i) {
    const int h = hs[i], n = ns[i];
    if (tid == 0) {
      unsigned v, spins = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.fcnt + h) : "memory");
        if (v < (unsigned)n) {
          __nanosleep(64);
          if (++spins > (1u << 26)) __trap();
        }
      } while (v < (unsigned)n);
      if (atomicAdd(a.fdone + h, 1u) + 1 == (unsigned)n) {   // every merger of h is past its wait
        a.fcnt[h] = 0u;
        a.fdone[h] = 0u;
      }
    }
    __syncthreads();
    if (i == 0) stamp(a, 5);
    const int rows_per = (nq + n - 1) / n;
    const int r0 = ps[i] * rows_per;
    attn_merge_rows(a, (size_t)h * a.flat_maxp, n, r0, min(nq, r0 + rows_per), 0, g, h);
  }
  stamp(a, 6);
}

template <bool TMA>
__device__ void attn_unit_ks(const LaAttnFusedArgs& a, uint8_t* smem_raw, int e) {
  stamp(a, 1);
  const FwdPlan* P = a.plan;
  const int n_rows = P->n_rows, ctx = P->n_prefix;
  if (n_rows == 0) return;
  const int g = a.H / a.KVH;
  const int nq = n_rows * g;
  const int n_rb = (nq + 127) >> 7;
  const int S = a.S;
  const int kvh = e / (a.nrb_max * (S + 1));
  const int rb = (e / (S + 1)) % a.nrb_max;
  const int split = e % (S + 1);
  if (rb >= n_rb) return;
  const bool spread = a.spread_merge || (a.sms > 0 && a.KVH * n_rb * (S + 1) <= a.sms);
  const bool step_unit = split == S;
  // key tiles of this unit: [k_begin, k_end) of the prefix (n_pre tiles), then
  // -- the step-block unit -- the step block [ctx, ctx + n_global).  fold_step:
  // the prefix is cut into S + 1 chunks and the last unit takes chunk S as well
  // as the step block (no unit holds one lone tile); otherwise S chunks and the
  // step block alone.  Chunking depends on ctx only either way.
  int k_begin = ctx, k_end = ctx;
  if (!step_unit || a.fold_step) {
    const int nch = a.fold_step ? S + 1 : S;
    const int CH = chunk_keys(ctx, nch);
    k_begin = min(ctx, split * CH);
    k_end = min(ctx, (split + 1) * CH);
  }
  // 1024-B alignment for the SW128 TMA boxes by pointer + offset (an integer
  // round trip hides the shared address space: generic LD/ST for every access)
  uint8_t* smem = TMA ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) : smem_raw;
  int* sFlag = reinterpret_cast<int*>(smem + kKsMaskOff + LA_MAX_ROWS * 16);
  const size_t grp = (size_t)kvh * a.nrb_max + rb;
  ks_segment<TMA, false>(a, smem, P, ctx, nq, g, kvh, rb, k_begin, k_end, step_unit, grp * (S + 1) + split, false);
  attn_arrive_merge(a, sFlag, grp, S, split, rb, g, nq, kvh, spread);
  stamp(a, 6);
}

// FLAT: the flat mapping (a separate instantiation: its second segment and
// per-head merge cost the default kernel 20 registers and ~1-2 % when inlined)
template <bool TMA, bool FLAT>
__global__ void __launch_bounds__(256, 1) la_attn_ks_kernel(LaAttnFusedArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  stamp(a, 0);
  la_pdl_trigger();
  la_l2_prefetch_gemm(a.pf);
  attn_prefetch_kv(a, blockIdx.x);
  if (TMA && threadIdx.x == 0) {
    ptx::tma_prefetch_desc(a.kmap);
    ptx::tma_prefetch_desc(a.vmap);
  }
  la_pdl_wait();
  if constexpr (FLAT)
    attn_flat_ks<TMA>(a, smem);
  else
    attn_unit_ks<TMA>(a, smem, blockIdx.x);
}

cudaError_t la_attn_fused_launch(const LaAttnFusedArgs& a, int grid, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = la_attn_fused_smem(a.tc != 0, a.cluster != 0);
  const bool ks = a.ksplit && !a.tc && !a.cluster && !a.fuse_qkv;
  if (ks) cfg.dynamicSmemBytes = a.ksplit == 2 ? kKsSmemTma : kKsSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (a.cluster) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = a.S + 1;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  if (a.cluster) {
    static std::atomic<unsigned> attr{0};
    cudaError_t e = la_smem_attr_once(attr, la_attn_cluster_kernel, (int)la_attn_fused_smem(false, true));
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, la_attn_cluster_kernel, a);
  }
  if (ks) {
    static std::atomic<unsigned> attr_cp{0}, attr_tma{0}, attr_flat{0};
    if (a.ksplit == 2 && a.flat) {
      cudaError_t e = la_smem_attr_once(attr_flat, la_attn_ks_kernel<true, true>, kKsSmemTma);
      if (e != cudaSuccess) return e;
      return cudaLaunchKernelEx(&cfg, la_attn_ks_kernel<true, true>, a);
    }
    if (a.ksplit == 2) {
      cudaError_t e = la_smem_attr_once(attr_tma, la_attn_ks_kernel<true, false>, kKsSmemTma);
      if (e != cudaSuccess) return e;
      return cudaLaunchKernelEx(&cfg, la_attn_ks_kernel<true, false>, a);
    }
    cudaError_t e = la_smem_attr_once(attr_cp, la_attn_ks_kernel<false, false>, kKsSmem);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, la_attn_ks_kernel<false, false>, a);
  }
  return cudaLaunchKernelEx(&cfg, la_attn_fused_kernel, a);
}

// ---------------------------------------------------------------------------
// Attention + O projection, one persistent launch (see la_attn.cuh).
namespace {
constexpr int kAoStages = 2;   // attention K/V ring in the fused kernel
constexpr int kAoAttnBytes = kAoStages * kTileBytes + LA_MAX_ROWS * 4 * 4 + 64;
constexpr int kAoGemmOff = (kAoAttnBytes + 1023) / 1024 * 1024;
constexpr int kAoTile = 128 * 128;          // one 128 x 64 bf16 weight tile
constexpr int kAoB = 128 * 128;             // <= 128 step rows x 64 bf16
constexpr unsigned kAoSpin = 1u << 26;

__device__ __forceinline__ unsigned ao_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
}  // namespace

size_t la_attn_o_smem(int nst) {
  return 1024 + kAoGemmOff + (size_t)nst * (LA_TPC * kAoTile + kAoB) + 8 * (2 * nst + 4) + 16;
}

__global__ void __launch_bounds__(256, 1) la_attn_o_kernel(LaAttnOArgs x) {
  extern __shared__ uint8_t ao_raw[];
  uint8_t* smem = ao_raw + ((1024 - (smem_u32(ao_raw) & 1023)) & 1023);
  const LaGemmArgs& g = x.g;
  const LaAttnFusedArgs& a = x.at;
  const int nst = x.nst;
  constexpr uint32_t a_bytes = LA_TPC * kAoTile;
  uint8_t* sA = smem + kAoGemmOff;
  uint8_t* sB = sA + nst * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + nst * kAoB);
  uint64_t* empty = full + nst;
  uint64_t* tfull = empty + nst;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { ptx::mbar_init(&tfull[b], 1); ptx::mbar_init(&tempty[b], 128); }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // O stream-K range of this CTA (identical to the standalone O GEMM's)
  const int kb = g.kb;
  const long U = (long)(g.n_tiles / LA_TPC) * kb;
  const long Pn = gridDim.x;
  const long u_begin = (long)blockIdx.x * U / Pn, u_end = (long)(blockIdx.x + 1) * U / Pn;
  const int n_pre = (int)min((long)nst, u_end - u_begin);
  la_pdl_trigger();
  if (x.g.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); x.g.trace[blockIdx.x * 8 + 0] = t_; }
  uint64_t pol_w = 0;
  if (threadIdx.x == 0) {
    pol_w = ptx::policy_evict_first();
    for (int i = 0; i < n_pre; ++i) {
      ptx::mbar_expect_tx_noarrive(&full[i], a_bytes);
      ptx::bulk_load(sA + i * a_bytes, g.a + (size_t)(u_begin + i) * (a_bytes / 2), a_bytes, &full[i], pol_w);
    }
    // the units beyond the ring go to L2 meanwhile (read right after attention)
    if (g.l2pf)
      for (long u = u_begin + n_pre; u < u_end; ++u)
        ptx::bulk_prefetch_l2(g.a + (size_t)u * (a_bytes / 2), a_bytes);
  }
  const int n_att = a.KVH * a.nrb_max * (a.S + 1);
  if ((int)blockIdx.x < n_att) attn_prefetch_kv(a, blockIdx.x);
  la_pdl_wait();
  const FwdPlan* P = g.plan;
  const int n_rows = P->n_rows, n_pad = P->n_pad;

  // ---- attention phase: this CTA's unit, then publish its KV head
  if ((int)blockIdx.x < n_att) {
    attn_unit<kAoStages>(a, smem, blockIdx.x);
    asm volatile("fence.proxy.async.global;" ::: "memory");   // the O bulk copies read a.out
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(x.head_done + blockIdx.x / (a.nrb_max * (a.S + 1)), 1u);
    }
  }
  __syncthreads();

  if (x.g.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); x.g.trace[blockIdx.x * 8 + 1] = t_; }
  // ---- O projection phase (split-K pieces, as la_gemm_kernel<LA_EPI_PARTIAL>)
  const unsigned target = (unsigned)(a.nrb_max * (a.S + 1));
  const int feats_per_kvh = (a.H / a.KVH) * 128;
  if (n_rows == 0) {
    if (threadIdx.x == 0)
      for (int i = 0; i < n_pre; ++i) {
        ptx::mbar_arrive(&full[i]);
        ptx::mbar_wait(&full[i], 0);
      }
  } else if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_x = ptx::policy_evict_last();
      const uint32_t bbytes = (uint32_t)n_pad * 128;
      int ready = -1;
      long it = 0;
      for (long u = u_begin; u < u_end; ++u, ++it) {
        const int k = (int)(u % kb);
        const int s = (int)(it % nst);
        const uint32_t r = (uint32_t)(it / nst);
        const int kvh = k * 64 / feats_per_kvh;
        if (kvh != ready) {
          unsigned n = 0;
          while ((int)(ao_ld_acquire(x.head_done + kvh) - target) < 0) {
            if (++n > kAoSpin) { atomicExch(x.err, 1u); break; }
            __nanosleep(64);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          if (ready < 0 && x.g.trace) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); x.g.trace[blockIdx.x * 8 + 2] = t_; }
          ready = kvh;
        }
        if (it < n_pre) {
          ptx::mbar_expect_tx(&full[s], bbytes);
        } else {
          ptx::mbar_wait(&empty[s], (r - 1) & 1);
          ptx::mbar_expect_tx(&full[s], a_bytes + bbytes);
          ptx::bulk_load(sA + s * a_bytes, g.a + (size_t)u * (a_bytes / 2), a_bytes, &full[s], pol_w);
        }
        ptx::bulk_load(sB + s * kAoB, g.b + (size_t)k * (kAoB / 2), bbytes, &full[s], pol_x);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::umma_idesc_bf16(128, (uint32_t)n_pad);
      long it = 0, u = u_begin;
      int use[2] = {0, 0}, buf = 0;
      while (u < u_end) {
        const int tile = (int)(u / kb);
        const long seg_start = u, seg_end = min(u_end, (long)(tile + 1) * kb);
        if (use[buf] > 0) {
          ptx::mbar_wait(&tempty[buf], (use[buf] - 1) & 1);
          ptx::tc_fence_after();
        }
        const uint32_t d_tmem = tmem + buf * (LA_TPC * 128);
        for (; u < seg_end; ++u, ++it) {
          const int s = (int)(it % nst);
          ptx::mbar_wait(&full[s], (uint32_t)(it / nst) & 1);
          ptx::tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * a_bytes), b_addr = smem_u32(sB + s * kAoB);
          for (int tt = 0; tt < LA_TPC; ++tt)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              ptx::umma_bf16(d_tmem + tt * 128, ptx::umma_desc_sw128(a_addr + tt * kAoTile + kk * 32),
                             ptx::umma_desc_sw128(b_addr + kk * 32), idesc,
                             (u > seg_start || kk > 0) ? 1u : 0u);
          ptx::umma_commit(&empty[s]);
        }
        ptx::umma_commit(&tfull[buf]);
        use[buf]++;
        buf ^= 1;
      }
    }
  } else if (warp < 6) {
    const int row_base = 32 * (warp & 3);
    const int f = row_base + lane;
    int use[2] = {0, 0}, buf = 0;
    long u = u_begin;
    while (u < u_end) {
      const int tile = (int)(u / kb);
      const long seg_end = min(u_end, (long)(tile + 1) * kb);
      const long c_first = la_cta_of((long)tile * kb, U, Pn);
      const int seg = (int)(blockIdx.x - c_first);
      ptx::mbar_wait(&tfull[buf], use[buf] & 1);
      ptx::tc_fence_after();
      for (int tt = 0; tt < LA_TPC; ++tt) {
        const uint32_t t_base = tmem + ((uint32_t)row_base << 16) + buf * (LA_TPC * 128) + tt * 128;
        float* wsp = g.ws + ((size_t)(tile * LA_TPC + tt) * g.max_segs + seg) * 128 * 128 + f;
        for (int c0 = 0; c0 < n_pad; c0 += 32) {
          float v[32];
          ptx::tmem_ld32(t_base + c0, v);
          const int nj = min(32, n_rows - c0);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            if (jj < nj) __stcg(wsp + (size_t)(c0 + jj) * 128, v[jj]);
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[buf]);
      use[buf]++;
      buf ^= 1;
      u = seg_end;
    }
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  if (x.g.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); x.g.trace[blockIdx.x * 8 + 3] = t_; }
  if (threadIdx.x == 0) {
    // the last CTA out resets the per-head counters for the next launch
    __threadfence();
    if (atomicAdd(x.exit_cnt, 1u) == gridDim.x - 1) {
      for (int h = 0; h < a.KVH; ++h) x.head_done[h] = 0u;
      *x.exit_cnt = 0u;
      __threadfence();
    }
  }
}

cudaError_t la_attn_o_launch(const LaAttnOArgs& x, int grid, cudaStream_t st, bool pdl) {
  static std::atomic<unsigned> attr{0};
  const size_t smem = la_attn_o_smem(x.nst);   // nst is fixed per process (LA_O_STAGES)
  cudaError_t e = la_smem_attr_once(attr, la_attn_o_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  return la_launch(la_attn_o_kernel, dim3(grid), dim3(256), smem, st, pdl, x);
}

LA_TL_DEFINE_SETTER(attnf)
