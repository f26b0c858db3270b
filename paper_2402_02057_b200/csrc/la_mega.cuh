// Persistent whole-forward kernel of the bf16 lookahead step (declarations).
//
// One launch evaluates every decoder layer (+ the LM head and the per-row
// argmax) for the <= 128 rows of the current FwdPlan.  One CTA per SM, warp
// specialised:
//   warp 0      weight producer: streams the packed weight tiles of EVERY
//               projection of the step, in order, into a 4-stage smem ring.
//               Weights never depend on activations, so it runs ahead across
//               layer boundaries and keeps HBM busy while the rest of the CTA
//               waits on dependencies.
//   warp 1      activation producer: bulk-loads the step-row k-block a unit
//               needs once the producing tile's readiness flag is set.
//   warp 2      TMEM owner + single-thread tcgen05 MMA issuer.
//   warps 3-6   TMEM drain: stream-K partials, and the split-K fix-up +
//               fused epilogue by the LAST-ARRIVING CTA of each tile
//               (RoPE + KV write, residual + RMSNorm statistics, SwiGLU,
//               logits argmax); it publishes the tile's readiness flag.
//   warps 3-10  attention units (mma.sync flash attention over a key chunk
//               of one KV head, structured mask generated in-kernel) and the
//               embedding gather.
// Dependencies are per tile / per KV head (global counters with acquire /
// release), never grid-wide barriers.  RMSNorm is applied "deferred": the
// GEMM input is bf16(x * g) and the consuming fix-up scales its accumulator
// by the row's rsqrt(mean(x^2) + eps), whose per-tile partial sums the
// producing fix-ups publish -- so no kernel needs a whole row before the
// next projection may start.
#pragma once
#include <cuda_bf16.h>

#include "la_common.cuh"
#include "la_gemm.cuh"

enum LaMegaKind { LA_MK_QKV = 0, LA_MK_O = 1, LA_MK_GU = 2, LA_MK_DOWN = 3, LA_MK_HEAD = 4 };

struct LaMegaGeo {
  int n_tiles;    // processed 128-row tiles (multiple of tpc)
  int real;       // tiles that carry real weights (the rest are zero padding)
  int tpc;        // tiles per stream-K unit
  int kb;         // K / 64
  int max_segs;   // workspace segments per tile
  int dp;         // data-parallel tiles [0, dp): one whole tile per CTA (0 or gridDim.x; needs tpc == 1)
};

struct LaMegaLayer {
  const __nv_bfloat16 *wqkv, *wo, *wgu, *wd;   // packed LA tiles
  const float *attn_norm, *mlp_norm;
};

// offsets (in uint32 words) into the sync area; per-layer blocks repeat
struct LaMegaSyncMap {
  int layer_stride;
  int cnt[4];        // per kind: [n_tiles] pieces drained per feature tile
  int rdy_qkv;       // [qkv tiles]
  int attn_cnt;      // [KVH * nrb_max] attention-unit arrivals
  int rdy_attn;      // [KVH]
  int rdy_m;         // [d / 128] mlp-input tiles
  int rdy_act;       // [gu tiles]
  int rdy_h;         // [d / 128] next layer's attention-input tiles
  int h0;            // global: [d / 128] layer-0 input tiles (embedding)
  int head_cnt;      // global: [head tiles] pieces drained
  int head_done;     // global: reduced LM-head slices (reset by the last)
  int head_gen;      // global: launches that ran the LM head
  int cta_done;      // global: CTAs finished
  int gen;           // global: completed launches
  int err;           // global: spin timeout (dependency never satisfied)
  int total;
};

struct LaMegaArgs {
  const FwdPlan* plan;
  DevDecode* dec;                     // argmax scatter target (null: none)
  const LaMegaLayer* layers;          // [L] (device)
  int L, d, H, KVH, ffn, V, slots;
  float eps;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* lm_head;
  const float* final_norm;
  LaMegaGeo geo[5];
  float* ws[5];                       // stream-K partials per kind
  float* x;                           // [128][d] residual stream (fp32)
  __nv_bfloat16 *h_attn, *h_mlp, *attn_out, *act;   // packed GEMM inputs
  float *ss_attn, *ss_mlp;            // [d/128][128] per-tile sums of x^2
  __nv_bfloat16* q;                   // [128][H][128]
  __nv_bfloat16 *kc, *vc;             // cache base, layer stride slots*KVH*128
  const float *rope_cos, *rope_sin;   // [slots][64]
  float* attn_ws;                     // [units][128][128] partial O
  float2* attn_ml;                    // [units][128] (m, l) in log2 units
  int attn_S;                         // prefix key splits (+1 step-key unit)
  int nrb_max;                        // query-row blocks per KV head at 128 rows
  unsigned long long* keys;           // [128] argmax keys
  int* row_amax;                      // [128]
  float* logits;                      // [128][V] dump or null
  unsigned* sync;
  LaMegaSyncMap sm;
  int do_head;
  int pf_units;
  int debug;   // timing experiments (LA_MEGA_DEBUG): 1 no step-row loads, 2 no reduce loads,
               // 4 no attention keys, 8 no partial stores -- results are garbage                       // weight units prefetched to L2 beyond the smem ring
  unsigned long long* timing;         // [0] start, [1] sum ns, [2] launches, [3] started, [4] finished
  // optional timeline [gridDim][trace_slots = 4L + 1 + L][8] globaltimer stamps
  // (LA_MEGA_TRACE=1): per GEMM phase {B dep satisfied, first MMA, last MMA,
  // drain done, reduce start, reduce end}; per layer attention {start, end,
  // first unit's deps met, first unit's keys done, merge done}
  unsigned long long* trace;
  int trace_slots;
};

size_t la_mega_smem_bytes();
int la_mega_threads();
cudaError_t la_mega_launch(const LaMegaArgs& a, int grid, cudaStream_t st, bool pdl);
