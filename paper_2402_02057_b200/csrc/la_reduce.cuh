// Parameter blocks of the split-K reduce / epilogue kernels (la_reduce.cu).
#pragma once
#include <cuda_bf16.h>

#include "la_common.cuh"

// stream-K geometry of the producing GEMM
struct LaSplit {
  int n_tiles, kb, grid, max_segs, tpc;
};

struct LaQkvEpi {
  LaPrefetch pf;                 // next GEMM's weights -> L2 (optional)
  const FwdPlan* plan;
  const float* ws;
  LaSplit sp;
  __nv_bfloat16* q_out;          // [128][H][128]
  __nv_bfloat16 *kc, *vc;        // layer base [slots][KVH][128]
  const float *rope_cos, *rope_sin;
  int H, KVH;
  LaRowNorm nrm;                 // deferred RMSNorm of the projection input
  const int* ready = nullptr;   // producing GEMM's per-unit-tile piece counters (la_gemm.cuh)
  int* runs = nullptr;          // [grid] this kernel's launches so far, one slot per CTA
};

struct LaResidNorm {
  LaPrefetch pf;                 // next GEMM's weights -> L2 (optional)
  const FwdPlan* plan;
  const float* ws;               // null: no partials to add
  LaSplit sp;
  const __nv_bfloat16* embed;    // non-null: x := embedding row (start of the step)
  float* x;                      // [128][d] fp32 residual stream
  const float* g;                // RMSNorm gain
  __nv_bfloat16* h;              // packed LA rows (la_act_off): bf16(x * g)
  int d;
  float eps;
  float* ss;                     // [d/128][128] per-tile sums of x^2 (LaRowNorm.ss)
  const int* ready = nullptr;   // producing GEMM's per-unit-tile piece counters (la_gemm.cuh)
  int* runs = nullptr;          // [grid] this kernel's launches so far, one slot per CTA
};

struct LaSwigluEpi {
  LaPrefetch pf;                 // next GEMM's weights -> L2 (optional)
  const FwdPlan* plan;
  const float* ws;
  LaSplit sp;
  __nv_bfloat16* act;            // packed LA rows (la_act_off)
  int act_ld;
  LaRowNorm nrm;
  const int* ready = nullptr;   // producing GEMM's per-unit-tile piece counters (la_gemm.cuh)
  int* runs = nullptr;          // [grid] this kernel's launches so far, one slot per CTA
};

struct LaLogitsEpi {
  const FwdPlan* plan;
  const float* ws;
  LaSplit sp;
  unsigned long long* keys;      // [128] per-row (value, -index) atomicMax keys
  float* logits;                 // [128][V] or null
  int V;
  LaRowNorm nrm;
  const int* ready = nullptr;   // producing GEMM's per-unit-tile piece counters (la_gemm.cuh)
  int* runs = nullptr;          // [grid] this kernel's launches so far, one slot per CTA
};

__global__ void la_qkv_epi_kernel(LaQkvEpi e);
__global__ void la_resid_norm_kernel(LaResidNorm e);
__global__ void la_swiglu_epi_kernel(LaSwigluEpi e);
__global__ void la_logits_epi_kernel(LaLogitsEpi e);
__global__ void la_argmax_finish_kernel(const FwdPlan* P, unsigned long long* keys, int* row_amax,
                                        DevDecode* dp);
