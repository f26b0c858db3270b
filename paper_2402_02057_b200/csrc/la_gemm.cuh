// Small-M weight-streaming GEMM on tcgen05 (declarations).
//
//   Y[tok][f] = sum_k X[tok][k] * Wt[f][k]      (X: step rows, Wt: weights [out][in])
//
// Swap-AB: the weight tile is the MMA "A" operand (M = 128 output features),
// the <= 128 step rows are "B" (N = n_pad tokens), the accumulator lives in
// TMEM as 128 lanes (features) x n_pad fp32 columns.  Work is split stream-K
// over (feature tile, 64-wide k block) units across one persistent CTA per SM
// so every SM streams weights for the whole launch; partial tiles are reduced
// deterministically (fixed segment order) by the last-arriving CTA.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "la_common.cuh"

enum LaGemmEpi {
  LA_EPI_QKV = 0,     // RoPE(q, k); q -> Q buffer, k/v -> KV cache slot
  LA_EPI_RESID = 1,   // x[tok][f] += y
  LA_EPI_SWIGLU = 2,  // tile = 64 gate + 64 up rows -> act = silu(g) * u
  LA_EPI_LOGITS = 3,  // per-tile (max, argmax) per token (+ optional fp32 logits dump)
};

struct LaGemmArgs {
  int n_tiles;   // 128-row feature tiles
  int kb;        // K / 64
  int a_mode;    // 0 single map; 1 q/k/v maps (tile boundaries t0, t1); 2 gate/up halves
  int t0, t1;
  int max_segs;  // workspace segments per tile
  const FwdPlan* plan;
  float* ws;     // [n_tiles][max_segs][128 tok][128 f] fp32 partials
  int* counters; // [n_tiles] arrival counters (left zeroed)
  // LA_EPI_QKV
  __nv_bfloat16* q_out;          // [128][H*128]
  __nv_bfloat16 *kc, *vc;        // layer base, [slots][KVH*128]
  const float *rope_cos, *rope_sin;  // [slots][64]
  int H, KVH;
  // LA_EPI_RESID
  float* x;
  int x_ld;
  // LA_EPI_SWIGLU
  __nv_bfloat16* act;
  int act_ld;
  // LA_EPI_LOGITS
  float2* pmax;                  // [n_tiles][128] (max, index-as-float-bits)
  float* logits;                 // [128][V] or null
  int V;
  // launch timing (device globaltimer): [0] first-CTA start, [1] sum ns,
  // [2] launches, [3] started CTAs, [4] finished CTAs; null = off
  unsigned long long* timing;
};

// Host-side descriptor of one GEMM (tensor maps + args), built once per
// engine and launched into the step graph.
struct LaGemm {
  CUtensorMap a0, a1, a2, b;
  LaGemmArgs args;
  int epi;
  int grid;
};

// Encode a [rows][K] bf16 row-major matrix as a TMA map with a
// box of (64 K elements) x box_rows rows, 128-byte swizzle.
int la_make_tmap(CUtensorMap* map, const void* base, int rows, int K, int box_rows);
int la_gemm_launch(const LaGemm& g, cudaStream_t st);
int la_gemm_workspace_segs(int n_tiles, int kb, int grid);
int la_sm_count();
