// Attention of the step rows (reference models.py:250-260 with the visibility
// sets of layout.py:139-170), as two kernels:
//
//  1. la_attn_chunks_kernel -- flash attention over <= NC key chunks x KV
//     heads x 128-query-row blocks (GQA groups share the K/V tile), mma.sync
//     bf16 QK^T and PV with an online softmax and a double-buffered cp.async K/V
//     pipeline.  The confirmed prefix (cache slots [0, ctx)) is dense -- every
//     step row sees it; the last chunk continues into the step block (slots
//     ctx + global row) under the paper's structured mask, GENERATED
//     in-kernel from the plan's per-row chains (a 128-bit visibility set per
//     query row, never an M x M matrix in memory).  One chunk per 128 prefix
//     keys (at most NC): short contexts finish in one pass and write the
//     output directly.
//  2. la_attn_merge_kernel -- for multi-chunk contexts, merges the chunk
//     partials in chunk order and writes the normalised output (packed LA
//     rows, the O-projection input).
//
// Layout independence: prefix chunking depends only on ctx, and step keys
// sit at their GLOBAL row position with masked entries exactly zero, so a
// row's result is bit-identical in every lookahead-parallel shard.
#include <cuda_bf16.h>

#include "la_attn.cuh"
#include "la_common.cuh"
#include "la_gemm.cuh"

namespace {

constexpr int kKeyTile = 64;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// [rows][128] bf16 tile, 16-byte chunks XOR-swizzled by (row & 7)
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 256 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
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

// Prefix split: one chunk per >= kMinChunk keys (at most NC).  Depends on
// ctx only, so every shard of a step chunks the prefix identically.  The
// last chunk also owns the step block, so short contexts need ONE pass.
__device__ __forceinline__ int n_chunks_of(int ctx, int NC, int min_chunk) {
  return max(1, min(NC, (ctx + min_chunk - 1) / min_chunk));
}
__device__ __forceinline__ int chunk_keys(int ctx, int nch) {
  return ((ctx + nch - 1) / nch + kKeyTile - 1) / kKeyTile * kKeyTile;
}

}  // namespace

constexpr int kStages = 2;    // K/V tile pipeline depth (2 CTAs per SM)

size_t la_attn_prefix_smem(int qrows) { return qrows * 256 + kStages * 2 * kKeyTile * 256 + qrows * 4 * 4; }

// grid = (KVH, NC, row blocks of kQRows flattened (row, head-in-group)
// queries); kQRows / 16 warps
template <int kQRows>
__global__ void __launch_bounds__(kQRows * 2) la_attn_chunks_kernel(LaAttnArgs a) {
  LA_PDL_ENTRY_PF(a.pf);
  const FwdPlan* P = a.plan;
  const int n_rows = P->n_rows, ctx = P->n_prefix;
  if (n_rows == 0) return;
  const int g = a.H / a.KVH;
  const int kvh = blockIdx.x, c = blockIdx.y, rb = blockIdx.z;
  const int nq = n_rows * g;
  if (rb * kQRows >= nq) return;
  const int nch = n_chunks_of(ctx, a.NC, a.min_chunk);
  if (c >= nch) return;
  const bool last = c == nch - 1;           // also owns the masked step block
  const int CH = ctx > 0 ? chunk_keys(ctx, nch) : 0;
  const int k_begin = min(ctx, c * CH);
  const int k_end = last ? ctx + P->n_global : min(ctx, (c + 1) * CH);

  extern __shared__ __align__(128) uint8_t attn_smem[];
  uint8_t* sQ = attn_smem;
  uint8_t* sKV = sQ + kQRows * 256;                              // [kStages][K, V]
  uint32_t* sMask = reinterpret_cast<uint32_t*>(sKV + kStages * 2 * kKeyTile * 256);  // [kQRows][4]
  const int nthr = blockDim.x, nwarp = nthr >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t kv_ld = (size_t)a.KVH * 128;

  // ---- Q tile (128 query rows x 128 dims)
  for (int i = tid; i < kQRows * 16; i += nthr) {
    int row = i >> 4, ch = i & 15, qr = rb * kQRows + row;
    const __nv_bfloat16* src = a.q;
    bool ok = qr < nq;
    if (ok) {
      int r = qr / g, h = kvh * g + qr % g;
      src = a.q + ((size_t)r * a.H + h) * 128 + ch * 8;
    }
    cp_async16(smem_u32(sQ) + swz(row, ch), src, ok);
  }
  if (last) {
    // structured mask: a query row sees its chain's step keys and itself
    for (int i = tid; i < kQRows * 4; i += nthr) sMask[i] = 0u;
    __syncthreads();
    for (int row = warp; row < kQRows; row += nwarp) {
      const int qr = rb * kQRows + row;
      if (qr >= nq) continue;
      const int r = qr / g;
      const int n = P->chain_n[r];
      for (int j = lane; j <= n; j += 32) {
        const int key = (j < n ? P->chain[r][j] : P->slot[r]) - ctx;
        atomicOr(&sMask[row * 4 + (key >> 5)], 1u << (key & 31));
      }
    }
  }
  // keys [k_begin, k_end) are cache slots [k_begin, k_end): the prefix slots
  // and, for the last chunk, the step slots ctx + global row right after them
  const int n_tiles = (k_end - k_begin + kKeyTile - 1) / kKeyTile;
  auto load_kv = [&](int t) {
    uint8_t* kb = sKV + (t % kStages) * 2 * kKeyTile * 256;
    const int t0 = k_begin + t * kKeyTile;
    for (int i = tid; i < kKeyTile * 16; i += nthr) {
      int row = i >> 4, ch = i & 15, key = t0 + row;
      bool ok = key < k_end;
      size_t off = ((size_t)(ok ? key : k_begin) * kv_ld) + kvh * 128 + ch * 8;
      cp_async16(smem_u32(kb) + swz(row, ch), a.kc + off, ok);
      cp_async16(smem_u32(kb + kKeyTile * 256) + swz(row, ch), a.vc + off, ok);
    }
  };
#pragma unroll
  for (int t = 0; t < kStages - 1; ++t) {
    if (t < n_tiles) load_kv(t);
    cp_commit();
  }

  uint32_t qf[8][4];
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = a.scale * kLog2e;
  const int qrow0 = warp * 16 + (lane >> 2);   // this thread's two query rows in the tile

  for (int t = 0; t < n_tiles; ++t) {
    if (t + kStages - 1 < n_tiles) load_kv(t + kStages - 1);
    cp_commit();
    cp_wait<kStages - 1>();
    __syncthreads();
    const uint8_t* sK = sKV + (t % kStages) * 2 * kKeyTile * 256;
    const uint8_t* sV = sK + kKeyTile * 256;
    if (t == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        int row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        int ch = kk * 2 + (lane >> 4);
        ldsm_x4(smem_u32(sQ) + swz(row, ch), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    // S = Q K^T (16 rows x 64 keys per warp)
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        int key = np * 16 + (lane & 7) + (lane >> 4) * 8;
        int ch = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_u32(sK) + swz(key, ch), b0, b1, b2, b3);
        mma16816(s[2 * np], qf[kk], b0, b1);
        mma16816(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // mask (range end; structured mask on step keys), scale into log2 units
    const int kbase = k_begin + t * kKeyTile;
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kbase + n * 8 + (lane & 3) * 2 + (e & 1);
        bool vis = key < k_end;
        if (vis && key >= ctx) {
          const int kg = key - ctx, row = qrow0 + (e >> 1) * 8;
          vis = (sMask[row * 4 + (kg >> 5)] >> (kg & 31)) & 1u;
        }
        s[n][e] = vis ? s[n][e] * sl2 : -INFINITY;
      }
      mx0 = fmaxf(mx0, fmaxf(s[n][0], s[n][1]));
      mx1 = fmaxf(mx1, fmaxf(s[n][2], s[n][3]));
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    // rows with nothing visible yet keep (m, l, o) = (-inf, 0, 0)
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
    for (int d = 0; d < 16; ++d) {
      o[d][0] *= al0; o[d][1] *= al0; o[d][2] *= al1; o[d][3] *= al1;
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4] = {pack_bf16(s[2 * kk][0], s[2 * kk][1]), pack_bf16(s[2 * kk][2], s[2 * kk][3]),
                        pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                        pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        int ch = dp * 2 + (lane >> 4);
        uint32_t v0, v1, v2, v3;
        ldsm_x4_t(smem_u32(sV) + swz(key, ch), v0, v1, v2, v3);
        mma16816(o[2 * dp], pa, v0, v1);
        mma16816(o[2 * dp + 1], pa, v2, v3);
      }
    }
    __syncthreads();
  }
  // row sums across the 4 lanes of a row
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    int qr = rb * kQRows + qrow0 + half * 8;
    if (qr >= nq) continue;
    int r = qr / g, h = kvh * g + qr % g;
    if (nch == 1) {
      // single pass: normalise and write the O-projection input directly
      const float inv = 1.0f / (half ? l1 : l0);
#pragma unroll
      for (int d = 0; d < 16; ++d) {
        int col = d * 8 + (lane & 3) * 2;
        *reinterpret_cast<uint32_t*>(a.out + la_act_off(r, h * 128 + col)) =
            pack_bf16(o[d][half * 2] * inv, o[d][half * 2 + 1] * inv);
      }
      continue;
    }
    // unnormalised partial O and (m, l) in log2 units
    size_t base = ((size_t)c * LA_MAX_ROWS + r) * a.H + h;
    float* dst = a.part_o + base * 128;
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      int col = d * 8 + (lane & 3) * 2;
      *reinterpret_cast<float2*>(dst + col) =
          make_float2(o[d][half * 2 + 0], o[d][half * 2 + 1]);
    }
    if ((lane & 3) == 0) a.part_ml[base] = make_float2(half ? m1 : m0, half ? l1 : l0);
  }
}

// grid = rows, block = 32 x min(H, 16): warp per (row, head); merges the
// active prefix chunks in chunk order, then the step chunk, and writes the
// normalised bf16 output into the packed O-projection input.
__global__ void __launch_bounds__(512) la_attn_merge_kernel(LaAttnArgs a) {
  LA_PDL_ENTRY();
  const FwdPlan* P = a.plan;
  const int r = blockIdx.x;
  if (r >= P->n_rows) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int n_chunks = n_chunks_of(P->n_prefix, a.NC, a.min_chunk);
  if (n_chunks == 1) return;   // the chunk kernel already wrote the output
  for (int h = warp; h < a.H; h += nw) {
    float2 ml[8];
    float4 po[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < n_chunks) {
        const size_t base = ((size_t)i * LA_MAX_ROWS + r) * a.H + h;
        ml[i] = a.part_ml[base];
        po[i] = reinterpret_cast<const float4*>(a.part_o + base * 128)[lane];
      }
    }
    float m = -INFINITY, l = 0.f, o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < n_chunks) {
        const float mn = fmaxf(m, ml[i].x);
        const float s0 = exp2f(m - mn), s1 = exp2f(ml[i].x - mn);
        o0 = o0 * s0 + po[i].x * s1;
        o1 = o1 * s0 + po[i].y * s1;
        o2 = o2 * s0 + po[i].z * s1;
        o3 = o3 * s0 + po[i].w * s1;
        l = l * s0 + ml[i].y * s1;
        m = mn;
      }
    const float inv = 1.0f / l;
    __nv_bfloat16* dst = a.out + la_act_off(r, h * 128 + lane * 4);   // packed LA rows
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(o0 * inv, o1 * inv),
                                                pack_bf16(o2 * inv, o3 * inv));
  }
}

template __global__ void la_attn_chunks_kernel<64>(LaAttnArgs a);
template __global__ void la_attn_chunks_kernel<128>(LaAttnArgs a);

LA_TL_DEFINE_SETTER(attn)
