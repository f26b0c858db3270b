// Parameter blocks of the fp32 single-CTA decode megakernel (la_tiny.cu).
#pragma once
#include "la_common.cuh"

#define TINY_ARCH_GPT 0     // reference TinyTransformer (models.py:189-271)
#define TINY_ARCH_LLAMA 1   // RMSNorm / RoPE / SwiGLU / GQA, fp32
#define TINY_MAX_LAYERS 8

struct TinyLayer {
  const float *wq, *wk, *wv, *wo;     // [out][in]
  const float *w1, *b1, *w2, *b2;     // GPT: ReLU MLP; Llama: w1 = gate, w2 = down
  const float *wu;                    // Llama: up
  const float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
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
  TinyLayer layers[TINY_MAX_LAYERS];
  float *kcache, *vcache;             // [L][slots][KVH*hd]
};

struct TinyScratch {
  float *x, *h, *q, *att, *ff;        // [LA_MAX_ROWS][...]
  float* scores;                      // [LA_MAX_ROWS*H][max_keys]
  int max_keys;
  int* row_amax;                      // [LA_MAX_ROWS]
};

__global__ void la_tiny_prefill(TinyModel m, TinyScratch s, FwdPlan* P, const int* tokens, int n);
__global__ void la_tiny_decode(TinyModel m, TinyScratch s, FwdPlan* P, DevDecode* dp,
                               float* logits);
__global__ void la_tiny_forward(TinyModel m, TinyScratch s, FwdPlan* P, float* logits);
__global__ void la_tiny_step_forward(TinyModel m, TinyScratch s, FwdPlan* P, DevDecode* dp,
                                     float* logits);
__global__ void la_tiny_step_finish(DevDecode* dp);
