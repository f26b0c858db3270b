// Step-row attention kernels (la_attn.cu).
#pragma once
#include <cuda_bf16.h>

#include "la_common.cuh"
#include "la_gemm.cuh"
#include "la_reduce.cuh"

struct LaAttnArgs {
  LaPrefetch pf;                 // next GEMM's weights -> L2 (optional)
  const FwdPlan* plan;
  const __nv_bfloat16* q;        // [LA_MAX_ROWS][H][128] (RoPE applied)
  const __nv_bfloat16 *kc, *vc;  // layer base, [slots][KVH][128]
  float* part_o;                 // [NC+1][LA_MAX_ROWS][H][128] (chunk NC = step block)
  float2* part_ml;               // [NC+1][LA_MAX_ROWS][H]  (max, sum) in log2 units
  __nv_bfloat16* out;            // packed LA rows [H*128/64][128][64] (la_act_off)
  int H, KVH, NC;
  int min_chunk;                 // prefix keys per chunk at least (chunks = min(NC, ctx/min))
  float scale;                   // 1/sqrt(head_dim)
};

template <int kQRows>
__global__ void la_attn_chunks_kernel(LaAttnArgs a);
__global__ void la_attn_merge_kernel(LaAttnArgs a);
size_t la_attn_prefix_smem(int qrows);

// Attention + chunk merge in one launch (la_attn_fused.cu)
struct LaAttnFusedArgs {
  LaPrefetch pf;                 // O-projection weights -> L2 while attention runs
  const FwdPlan* plan;
  const __nv_bfloat16* q;        // [LA_MAX_ROWS][H][128] (RoPE applied)
  const __nv_bfloat16 *kc, *vc;  // layer base, [slots][KVH][128]
  float* part_o;                 // [KVH][nrb_max][S+1][128][128] chunk partials
  float2* part_ml;               // [KVH][nrb_max][S+1][128] (max, sum) in log2 units
  unsigned* cnt;                 // [KVH][nrb_max] chunk arrivals (monotonic; +S+1 per launch)
  __nv_bfloat16* out;            // packed LA rows (la_act_off), the O-projection input
  int H, KVH, S, nrb_max;
  float scale;
  int spread_merge;              // grid <= SMs: every chunk CTA merges a share of the rows
  int sms;                       // > 0: also spread-merge any launch whose ACTIVE units (row
                                 // blocks in use x KVH x (S+1)) fit on this many SMs
  int fuse_qkv;                  // grid <= SMs: the QKV epilogue runs here first (grid barrier)
  int tc;                        // tcgen05 QK^T / PV for chunks of <= 6 key tiles
  int cluster;                   // launched as clusters of S+1 CTAs = one (KV head, row block):
                                 // chunk partials stay in smem and merge over DSMEM
  int dbg;                       // LA_ATTN_DBG experiments: 1 skip PV MMAs, 2 skip QK^T MMAs
  int ksplit;                    // key tiles split by parity over the two warp groups (LA_ATTN_KSPLIT;
                                 // 2: K/V tiles by TMA through kmap / vmap)
  const CUtensorMap* kmap;       // whole K / V cache as [layers * slots][KVH * 128], SW128 boxes
  const CUtensorMap* vmap;       //   of [64 keys][64 dims] (device memory)
  int kv_row0;                   // this layer's first row in the maps (layer * slots)
  const int* spec_ctx;           // graph-loop decode: the decode state's ctx, read before the
                                 // dependency wait to start the first prefix tiles early
  int kv_pf;                     // bulk-prefetch the unit's prefix K/V into L2 before the
                                 // dependency wait (LA_ATTN_KV_PF=1; measured slower, off)
  LaQkvEpi qkv;                  // its arguments
  unsigned* gbar;                // grid-barrier counter (monotonic; + grid per launch)
  unsigned long long* trace;     // optional [grid][8] globaltimer stamps (LA_ATTN_TRACE=1)
  int fold_step;                 // key-split kernel: S + 1 prefix chunks, the last with the step block
  int flat;                      // key-split kernel, one row block: the KVH x prefix-tile space cut
                                 // evenly over the grid (every SM), a head's step block with the CTA
                                 // holding its last prefix tile; partials [KVH][flat_maxp]
  int flat_maxp;                 // partial slots per KV head (>= CTAs meeting one head)
  unsigned* fcnt;                // [KVH] segment arrivals, re-zeroed by the head's last merger
  unsigned* fdone;               // [KVH] mergers past their wait
};

__global__ void la_attn_fused_kernel(LaAttnFusedArgs a);
cudaError_t la_attn_fused_launch(const LaAttnFusedArgs& a, int grid, cudaStream_t st, bool pdl);
size_t la_attn_fused_smem(bool tc, bool cluster = false);

// Attention + O projection in ONE persistent launch (LA_ATTN_O=1, experimental):
// every CTA streams its first O-weight units into its smem ring at launch, runs
// its attention unit (if any), publishes per-KV-head completion, then runs its
// O stream-K units -- each waiting only for the heads its k-range reads.  The
// O pieces land exactly where the standalone O GEMM puts them.
struct LaAttnOArgs {
  LaAttnFusedArgs at;     // attention (mma.sync path)
  LaGemmArgs g;           // the O projection (split-K pieces, tpc = LA_TPC)
  unsigned* head_done;    // [KVH] attention units finished this launch (reset by the last CTA)
  unsigned* exit_cnt;     // CTAs finished this launch
  unsigned* err;          // spin timeout (dependency never satisfied)
  int nst;                // O-weight ring stages
};
size_t la_attn_o_smem(int nst);
cudaError_t la_attn_o_launch(const LaAttnOArgs& x, int grid, cudaStream_t st, bool pdl);

