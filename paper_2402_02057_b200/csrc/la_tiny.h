// Parameter blocks of the fp32 single-CTA decode megakernel (la_tiny.cu).
#pragma once
#include "la_common.cuh"

#define TINY_ARCH_GPT 0     // reference TinyTransformer (models.py:189-271)
#define TINY_ARCH_LLAMA 1   // RMSNorm / RoPE / SwiGLU / GQA, fp32
#define TINY_MAX_LAYERS 8
#ifndef TINY_THREADS
#define TINY_THREADS 512    // threads of the single-CTA kernels (<= 1024; 512 leaves 128 registers a thread)
#endif
#define TINY_MAX_HD 16      // head_dim bound of the fp32 path (attention keeps a row of q, k, v, o in registers)

struct TinyLayer {
  const float *wq, *wk, *wv, *wo;     // [out][in]
  const float *w1, *b1, *w2, *b2;     // GPT: ReLU MLP; Llama: w1 = gate, w2 = down
  const float *wu;                    // Llama: up
  const float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
  // transposed copies ([in][out], made at setup) read by the kernels: a warp's
  // 32 consecutive outputs load 32 consecutive floats (one L1 wavefront)
  const float *wqkvT;                 // [d][qd + 2 kvd]  (q | k | v columns)
  const float *woT, *w1T, *wuT, *w2T; // [qd][d], [d][ff], [d][ff], [ff][d]
};

struct TinyModel {
  int arch, V, d, L, H, KVH, hd, ff;
  float eps;
  int slots;                          // KV capacity (tokens)
  const float* embed;                 // [V][d]
  const float* pos_tab;               // GPT: [slots][d] sinusoid (fp64 on host -> fp32)
  const float *rope_cos, *rope_sin;   // Llama: [slots][hd/2]
  const float *lnf_g, *lnf_b;
  const float* unembed;               // [V][d]
  const float* unembedT;              // [d][V] (transposed copy)
  TinyLayer layers[TINY_MAX_LAYERS];
  float *kcache, *vcache;             // [L][slots][KVH*hd]
};

struct TinyScratch {
  float *x, *h, *q, *att, *ff;        // [LA_MAX_ROWS][...] (global; shared memory when smem)
  int smem;                           // 1: the kernels keep x / h / q / att / ff in dynamic smem;
                                      // 2: and la_tiny_decode its step plan
  int* row_amax;                      // [LA_MAX_ROWS]
};
// dynamic shared memory the kernels need for the activations (0: keep them global)
size_t la_tiny_smem_bytes(const TinyModel& m, int* mode);
int la_tiny_set_smem(size_t bytes);

__global__ void la_tiny_prefill(TinyModel m, TinyScratch s, FwdPlan* P, const int* tokens, int n);
__global__ void la_tiny_decode(TinyModel m, TinyScratch s, FwdPlan* P, DevDecode* dp,
                               float* logits);
__global__ void la_tiny_forward(TinyModel m, TinyScratch s, FwdPlan* P, float* logits);
__global__ void la_tiny_step_forward(TinyModel m, TinyScratch s, FwdPlan* P, DevDecode* dp,
                                     float* logits);
__global__ void la_tiny_step_finish(DevDecode* dp);
// profiling: enable (and zero) the per-phase cycle counters of la_tiny_decode,
// or read them (out != null: 8 values, see la_tiny.cu)
int la_tiny_prof(bool enable, unsigned long long* out);
// out[c][col_off + r] = in[r][c] for in [rows][cols], out rows of out_ld floats
__global__ void la_tiny_transpose(const float* in, int rows, int cols, float* out, int out_ld, int col_off);
