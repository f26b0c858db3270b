// bf16 Llama-2-shaped multi-kernel path (BASELINE configs 2-5).
//
// One lookahead step = K1 build -> embed+norm -> L x {QKV GEMM (+RoPE, K/V
// to cache) -> prefix attention -> chain attention -> O GEMM (+residual) ->
// norm -> gate/up GEMM (+SwiGLU) -> down GEMM (+residual) -> norm} -> LM-head
// GEMM (+per-tile argmax) -> argmax reduce -> K10 finish -> KV commit.
// The step is captured once into a CUDA graph whose body runs inside a
// device-side WHILE conditional node until the decode's done flag is set, so
// a whole decode is ONE graph launch with no host round trip.
#include <algorithm>
#include <cmath>
#include <vector>

#include "la_attn.cuh"
#include "la_engine.h"
#include "la_gemm.cuh"
#include "la_kernels.h"

#define CK(x) LA_CUDA_CHECK(x)
#define RET_IF(x)               \
  do {                          \
    int _r = (x);               \
    if (_r != LA_OK) return _r; \
  } while (0)

struct LlamaLayerW {
  const __nv_bfloat16 *wq, *wk, *wv, *wo, *wg, *wu, *wd;
  const float *attn_norm, *mlp_norm;
};

struct LlamaPath {
  int d = 0, L = 0, H = 0, KVH = 0, ffn = 0, V = 0, NC = 1;
  float eps = 1e-5f;
  const __nv_bfloat16 *embed = nullptr, *lm_head = nullptr;
  const float* final_norm = nullptr;
  std::vector<LlamaLayerW> lw;
  float* x = nullptr;
  __nv_bfloat16 *h = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr;
  float* ws = nullptr;
  int* counters = nullptr;
  float2* pmax = nullptr;
  float* part_o = nullptr;
  float2* part_ml = nullptr;
  float *rope_cos = nullptr, *rope_sin = nullptr;
  int* row_amax = nullptr;
  unsigned long long* timing = nullptr;   // [4 epilogue kinds][8]
  float* logits = nullptr;   // device dump target (parity hook), else null
  std::vector<LaGemm> qkv, o, gu, down;
  LaGemm head{};
  int head_tiles = 0;
  int kernels_per_step = 0;
  cudaStream_t cap = nullptr;
  cudaGraphExec_t loop_exec = nullptr;   // while(!done) { step }
  cudaGraphExec_t fwd_exec = nullptr;    // K1 + forward + owned argmax (LP)
  cudaGraph_t loop_graph = nullptr, fwd_graph = nullptr;
};

// ------------------------------------------------------------- kernels
namespace {

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// RMSNorm of one row (fp32 residual -> bf16 GEMM input); grid = rows
__global__ void __launch_bounds__(256) la_rmsnorm_kernel(const FwdPlan* P, const float* x,
                                                        const float* g, __nv_bfloat16* h, int d,
                                                        float eps, const __nv_bfloat16* embed) {
  const int r = blockIdx.x;
  if (r >= P->n_rows) return;
  __shared__ float red[8];
  float* xr = const_cast<float*>(x) + (size_t)r * d;
  if (embed) {   // first norm of the step: x = embedding row (reference models.py:247)
    const __nv_bfloat16* er = embed + (size_t)P->ids[r] * d;
    for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
      uint4 u = *reinterpret_cast<const uint4*>(er + i);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 f = __bfloat1622float2(b[k]);
        xr[i + 2 * k] = f.x;
        xr[i + 2 * k + 1] = f.y;
      }
    }
    __syncthreads();
  }
  float ss = 0.f;
  for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(xr + i);
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  const float inv = rsqrtf(block_sum(ss, red) / d + eps);
  __nv_bfloat16* hr = h + (size_t)r * d;
  for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(xr + i);
    float4 gg = *reinterpret_cast<const float4*>(g + i);
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x * inv * gg.x, v.y * inv * gg.y);
    __nv_bfloat162 b = __floats2bfloat162_rn(v.z * inv * gg.z, v.w * inv * gg.w);
    *reinterpret_cast<__nv_bfloat162*>(hr + i) = a;
    *reinterpret_cast<__nv_bfloat162*>(hr + i + 2) = b;
  }
}

// per-row argmax over the LM-head tiles (lowest index on ties), then the
// owned rows go to the decode state's global-row table
__global__ void la_argmax_reduce_kernel(const FwdPlan* P, const float2* pmax, int n_tiles,
                                        int* row_amax, DevDecode* dp) {
  const int r = threadIdx.x;
  if (r >= P->n_rows) return;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = 0; t < n_tiles; ++t) {
    float2 v = pmax[(size_t)t * 128 + r];
    int idx = __float_as_int(v.y);
    if (v.x > best || (v.x == best && idx < bi)) { best = v.x; bi = idx; }
  }
  row_amax[r] = bi;
  if (dp && P->own[r]) dp->amax[P->grow[r]] = bi;
}

// prefill plan: causal chain over tokens[start, start+R)
__global__ void la_plan_chain_kernel(FwdPlan* P, const int* tokens, int start, int R) {
  if (threadIdx.x == 0) {
    P->n_rows = R; P->n_pad = (R + 15) & ~15; P->n_prefix = start; P->want_logits = 0;
  }
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    P->ids[r] = tokens[start + r];
    P->pos[r] = start + r;
    P->slot[r] = start + r;
    P->grow[r] = r;
    P->own[r] = 1;
    P->chain_n[r] = r;
    for (int j = 0; j < r; ++j) P->chain[r][j] = start + j;
  }
}

__global__ void la_set_cond_kernel(cudaGraphConditionalHandle h, const DevDecode* d) {
  cudaGraphSetConditional(h, d->done ? 0u : 1u);
}

}  // namespace

// ------------------------------------------------------------ host setup
static int build_gemm(LaGemm& g, int epi, int a_mode, const void* a0, int rows0, const void* a1,
                      int rows1, const void* a2, int rows2, int box, const void* b, int K,
                      int n_tiles) {
  memset(&g, 0, sizeof(g));
  RET_IF(la_make_tmap(&g.a0, a0, rows0, K, box));
  RET_IF(la_make_tmap(&g.a1, a1 ? a1 : a0, a1 ? rows1 : rows0, K, box));
  RET_IF(la_make_tmap(&g.a2, a2 ? a2 : a0, a2 ? rows2 : rows0, K, box));
  RET_IF(la_make_tmap(&g.b, b, LA_MAX_ROWS, K, 16));
  g.epi = epi;
  g.args.n_tiles = n_tiles;
  g.args.kb = K / 64;
  g.args.a_mode = a_mode;
  long U = (long)n_tiles * g.args.kb;
  g.grid = (int)std::min<long>(la_sm_count(), U);
  g.args.max_segs = la_gemm_workspace_segs(n_tiles, g.args.kb, g.grid);
  return LA_OK;
}

template <typename T>
static int lalloc(la_engine* e, T** p, size_t n) {
  void* q = nullptr;
  CK(cudaMalloc(&q, std::max<size_t>(n * sizeof(T), 16)));
  CK(cudaMemset(q, 0, std::max<size_t>(n * sizeof(T), 16)));
  e->owned.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return LA_OK;
}

int llama_create(la_engine* e) {
  const la_model_desc& D = e->desc;
  if (D.head_dim != 128) { la_set_error("bf16 path needs head_dim == 128"); return LA_ERR_UNSUPPORTED; }
  if (D.dim % 128 || D.ffn % 64) { la_set_error("bf16 path needs dim %% 128 == 0 and ffn %% 64 == 0"); return LA_ERR_UNSUPPORTED; }
  auto* p = new LlamaPath();
  e->llama = p;
  p->d = D.dim; p->L = D.layers; p->H = D.heads; p->KVH = D.kv_heads; p->ffn = D.ffn;
  p->V = D.vocab; p->eps = D.norm_eps;
  auto B = [&](int i) { return reinterpret_cast<const __nv_bfloat16*>(e->w[i]); };
  auto F = [&](int i) { return reinterpret_cast<const float*>(e->w[i]); };
  p->embed = B(0); p->lm_head = B(1); p->final_norm = F(2);
  for (int l = 0; l < D.layers; ++l) {
    int b = 3 + 9 * l;
    p->lw.push_back({B(b), B(b + 1), B(b + 2), B(b + 3), B(b + 4), B(b + 5), B(b + 6), F(b + 7), F(b + 8)});
  }
  const int R = LA_MAX_ROWS, qd = D.heads * 128;
  RET_IF(lalloc(e, &p->x, (size_t)R * D.dim));
  RET_IF(lalloc(e, &p->h, (size_t)R * D.dim));
  RET_IF(lalloc(e, &p->q, (size_t)R * qd));
  RET_IF(lalloc(e, &p->attn, (size_t)R * qd));
  RET_IF(lalloc(e, &p->act, (size_t)R * D.ffn));
  RET_IF(lalloc(e, &p->row_amax, R));
  // prefix-attention split: ~2 CTAs per SM at full rows
  const int g = D.heads / D.kv_heads;
  const int rblocks = (R * g + 63) / 64;
  p->NC = std::max(1, std::min(16, (2 * la_sm_count() + D.kv_heads * rblocks - 1) / (D.kv_heads * rblocks)));
  RET_IF(lalloc(e, &p->part_o, (size_t)p->NC * R * D.heads * 128));
  RET_IF(lalloc(e, &p->part_ml, (size_t)p->NC * R * D.heads));
  // RoPE tables (float64 on the host, stored fp32)
  {
    std::vector<float> c((size_t)e->slots * 64), s((size_t)e->slots * 64);
    for (int pos = 0; pos < e->slots; ++pos)
      for (int i = 0; i < 64; ++i) {
        double inv = 1.0 / std::pow((double)D.rope_theta, (2.0 * i) / 128.0);
        c[(size_t)pos * 64 + i] = (float)std::cos(pos * inv);
        s[(size_t)pos * 64 + i] = (float)std::sin(pos * inv);
      }
    RET_IF(lalloc(e, &p->rope_cos, c.size()));
    RET_IF(lalloc(e, &p->rope_sin, s.size()));
    CK(cudaMemcpy(p->rope_cos, c.data(), c.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p->rope_sin, s.data(), s.size() * 4, cudaMemcpyHostToDevice));
  }
  // GEMM descriptors
  const int d = D.dim, KVH = D.kv_heads, H = D.heads;
  p->qkv.resize(D.layers); p->o.resize(D.layers); p->gu.resize(D.layers); p->down.resize(D.layers);
  size_t ws_need = 0;
  int max_tiles = 0;
  auto track = [&](const LaGemm& gg) {
    ws_need = std::max(ws_need, (size_t)gg.args.n_tiles * gg.args.max_segs * 128 * 128);
    max_tiles = std::max(max_tiles, gg.args.n_tiles);
  };
  __nv_bfloat16* kc = reinterpret_cast<__nv_bfloat16*>(e->kc);
  __nv_bfloat16* vc = reinterpret_cast<__nv_bfloat16*>(e->vc);
  for (int l = 0; l < D.layers; ++l) {
    const LlamaLayerW& w = p->lw[l];
    LaGemm& a = p->qkv[l];
    RET_IF(build_gemm(a, LA_EPI_QKV, 1, w.wq, H * 128, w.wk, KVH * 128, w.wv, KVH * 128, 128, p->h, d, H + 2 * KVH));
    a.args.t0 = H; a.args.t1 = H + KVH;
    a.args.q_out = p->q;
    a.args.kc = kc + (size_t)l * e->slots * KVH * 128;
    a.args.vc = vc + (size_t)l * e->slots * KVH * 128;
    a.args.rope_cos = p->rope_cos; a.args.rope_sin = p->rope_sin;
    a.args.H = H; a.args.KVH = KVH;
    track(a);
    LaGemm& ob = p->o[l];
    RET_IF(build_gemm(ob, LA_EPI_RESID, 0, w.wo, d, nullptr, 0, nullptr, 0, 128, p->attn, H * 128, d / 128));
    ob.args.x = p->x; ob.args.x_ld = d;
    track(ob);
    LaGemm& gu = p->gu[l];
    RET_IF(build_gemm(gu, LA_EPI_SWIGLU, 2, w.wg, D.ffn, w.wu, D.ffn, nullptr, 0, 64, p->h, d, D.ffn / 64));
    gu.args.act = p->act; gu.args.act_ld = D.ffn;
    track(gu);
    LaGemm& dn = p->down[l];
    RET_IF(build_gemm(dn, LA_EPI_RESID, 0, w.wd, d, nullptr, 0, nullptr, 0, 128, p->act, D.ffn, d / 128));
    dn.args.x = p->x; dn.args.x_ld = d;
    track(dn);
  }
  p->head_tiles = (D.vocab + 127) / 128;
  RET_IF(build_gemm(p->head, LA_EPI_LOGITS, 0, p->lm_head, D.vocab, nullptr, 0, nullptr, 0, 128, p->h, d, p->head_tiles));
  track(p->head);
  RET_IF(lalloc(e, &p->pmax, (size_t)p->head_tiles * 128));
  p->head.args.pmax = p->pmax;
  p->head.args.V = D.vocab;
  RET_IF(lalloc(e, &p->ws, ws_need));
  RET_IF(lalloc(e, &p->counters, max_tiles + 1));
  RET_IF(lalloc(e, &p->timing, 32));
  auto fin = [&](LaGemm& gg) {
    gg.args.plan = e->d_plan; gg.args.ws = p->ws; gg.args.counters = p->counters;
    gg.args.timing = p->timing + 8 * gg.epi;
  };
  for (int l = 0; l < D.layers; ++l) { fin(p->qkv[l]); fin(p->o[l]); fin(p->gu[l]); fin(p->down[l]); }
  fin(p->head);
  CK(cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking));
  cudaError_t ce = cudaFuncSetAttribute(la_attn_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)la_attn_prefix_smem());
  if (ce != cudaSuccess) { la_set_error("attn smem attr: %s", cudaGetErrorString(ce)); return LA_ERR_CUDA; }
  return LA_OK;
}

void llama_destroy(la_engine* e) {
  LlamaPath* p = e->llama;
  if (!p) return;
  if (p->loop_exec) cudaGraphExecDestroy(p->loop_exec);
  if (p->fwd_exec) cudaGraphExecDestroy(p->fwd_exec);
  if (p->loop_graph) cudaGraphDestroy(p->loop_graph);
  if (p->fwd_graph) cudaGraphDestroy(p->fwd_graph);
  if (p->cap) cudaStreamDestroy(p->cap);
  delete p;
  e->llama = nullptr;
}

// ------------------------------------------------------------- forward
static int launch_attn(la_engine* e, int l, cudaStream_t st) {
  LlamaPath* p = e->llama;
  LaAttnArgs a;
  a.plan = e->d_plan;
  a.q = p->q;
  const size_t lstride = (size_t)e->slots * p->KVH * 128;
  a.kc = reinterpret_cast<const __nv_bfloat16*>(e->kc) + l * lstride;
  a.vc = reinterpret_cast<const __nv_bfloat16*>(e->vc) + l * lstride;
  a.part_o = p->part_o;
  a.part_ml = p->part_ml;
  a.out = p->attn;
  a.H = p->H; a.KVH = p->KVH; a.NC = p->NC;
  a.scale = 1.0f / sqrtf(128.0f);
  const int g = p->H / p->KVH;
  dim3 grid(p->KVH, p->NC, (LA_MAX_ROWS * g + 63) / 64);
  la_attn_prefix_kernel<<<grid, 128, la_attn_prefix_smem(), st>>>(a);
  la_attn_chain_kernel<<<LA_MAX_ROWS, 512, 0, st>>>(a);
  CK(cudaGetLastError());
  return LA_OK;
}

// all decoder layers on the rows of e->d_plan; leaves h = final-norm(x)
static int forward_layers(la_engine* e, cudaStream_t st, int* nk) {
  LlamaPath* p = e->llama;
  la_rmsnorm_kernel<<<LA_MAX_ROWS, 256, 0, st>>>(e->d_plan, p->x, p->lw[0].attn_norm, p->h, p->d,
                                                 p->eps, p->embed);
  CK(cudaGetLastError());
  int n = 1;
  for (int l = 0; l < p->L; ++l) {
    RET_IF(la_gemm_launch(p->qkv[l], st));
    RET_IF(launch_attn(e, l, st));
    RET_IF(la_gemm_launch(p->o[l], st));
    la_rmsnorm_kernel<<<LA_MAX_ROWS, 256, 0, st>>>(e->d_plan, p->x, p->lw[l].mlp_norm, p->h, p->d,
                                                   p->eps, nullptr);
    RET_IF(la_gemm_launch(p->gu[l], st));
    RET_IF(la_gemm_launch(p->down[l], st));
    const float* next = (l + 1 < p->L) ? p->lw[l + 1].attn_norm : p->final_norm;
    la_rmsnorm_kernel<<<LA_MAX_ROWS, 256, 0, st>>>(e->d_plan, p->x, next, p->h, p->d, p->eps, nullptr);
    CK(cudaGetLastError());
    n += 8;
  }
  *nk += n;
  return LA_OK;
}

static int forward_head(la_engine* e, cudaStream_t st, bool scatter, int* nk) {
  LlamaPath* p = e->llama;
  p->head.args.logits = p->logits;
  RET_IF(la_gemm_launch(p->head, st));
  la_argmax_reduce_kernel<<<1, 128, 0, st>>>(e->d_plan, p->pmax, p->head_tiles, p->row_amax,
                                            scatter ? e->d_dec : nullptr);
  CK(cudaGetLastError());
  *nk += 2;
  return LA_OK;
}

int llama_prefill(la_engine* e, const int* d_tokens, int n, cudaStream_t st) {
  for (int start = 0; start < n; start += LA_MAX_ROWS) {
    int R = std::min(LA_MAX_ROWS, n - start);
    la_plan_chain_kernel<<<1, 128, 0, st>>>(e->d_plan, d_tokens, start, R);
    CK(cudaGetLastError());
    int nk = 0;
    RET_IF(forward_layers(e, st, &nk));
  }
  return LA_OK;
}

int llama_forward_plan(la_engine* e, float* d_logits, cudaStream_t st) {
  LlamaPath* p = e->llama;
  p->logits = d_logits;
  int nk = 0;
  int rc = forward_layers(e, st, &nk);
  if (rc == LA_OK) rc = forward_head(e, st, false, &nk);
  p->logits = nullptr;
  p->head.args.logits = nullptr;
  return rc;
}

// one step's kernels: K1 -> forward -> argmax (-> K10 -> commit)
static int record_step(la_engine* e, cudaStream_t st, bool finish, int* nk) {
  LlamaPath* p = e->llama;
  la_step_build_kernel<<<1, 256, 0, st>>>(e->d_dec, e->d_plan);
  CK(cudaGetLastError());
  *nk += 1;
  RET_IF(forward_layers(e, st, nk));
  RET_IF(forward_head(e, st, true, nk));
  if (finish) {
    la_step_finish_kernel<<<1, 256, 0, st>>>(e->d_dec);
    la_kv_commit_kernel<<<std::max(1, std::min(148, p->L * e->row_bytes / 16 / 256)), 256, 0, st>>>(
        e->d_dec, (uint8_t*)e->kc, (uint8_t*)e->vc, p->L, e->slots, e->row_bytes);
    CK(cudaGetLastError());
    *nk += 2;
  }
  return LA_OK;
}

static int build_loop_graph(la_engine* e) {
  LlamaPath* p = e->llama;
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle handle;
  CK(cudaGraphConditionalHandleCreate(&handle, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(p->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  int nk = 0;
  int rc = record_step(e, p->cap, true, &nk);
  la_set_cond_kernel<<<1, 1, 0, p->cap>>>(handle, e->d_dec);
  cudaGraph_t captured;
  cudaError_t ce = cudaStreamEndCapture(p->cap, &captured);
  if (rc != LA_OK) { cudaGraphDestroy(g); return rc; }
  if (ce != cudaSuccess) { cudaGraphDestroy(g); la_set_error("step capture: %s", cudaGetErrorString(ce)); return LA_ERR_CUDA; }
  p->kernels_per_step = nk + 1;
  ce = cudaGraphInstantiate(&p->loop_exec, g, 0);
  if (ce != cudaSuccess) { cudaGraphDestroy(g); la_set_error("graph instantiate: %s", cudaGetErrorString(ce)); return LA_ERR_CUDA; }
  p->loop_graph = g;
  return LA_OK;
}

int llama_decode_loop(la_engine* e, cudaStream_t st, int* launches) {
  LlamaPath* p = e->llama;
  if (!p->loop_exec) RET_IF(build_loop_graph(e));
  CK(cudaGraphLaunch(p->loop_exec, st));
  // kernels launched = per-step kernels x steps; the host learns the step
  // count only at readback, so report it there (engine->h_dec is refreshed)
  *launches = -p->kernels_per_step;
  return LA_OK;
}

int llama_step_forward(la_engine* e, cudaStream_t st) {
  LlamaPath* p = e->llama;
  if (!p->fwd_exec) {
    CK(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeRelaxed));
    int nk = 0;
    int rc = record_step(e, p->cap, false, &nk);
    cudaGraph_t g;
    cudaError_t ce = cudaStreamEndCapture(p->cap, &g);
    if (rc != LA_OK) return rc;
    if (ce != cudaSuccess) { la_set_error("fwd capture: %s", cudaGetErrorString(ce)); return LA_ERR_CUDA; }
    ce = cudaGraphInstantiate(&p->fwd_exec, g, 0);
    if (ce != cudaSuccess) { la_set_error("fwd instantiate: %s", cudaGetErrorString(ce)); return LA_ERR_CUDA; }
    p->fwd_graph = g;
  }
  CK(cudaGraphLaunch(p->fwd_exec, st));
  return LA_OK;
}

// ------------------------------------------------------- GEMM timing ABI
extern "C" int32_t la_gemm_timing_reset(la_engine* e) {
  if (!e || !e->llama) { la_set_error("no bf16 path on this engine"); return LA_ERR_INVALID_CONFIG; }
  CK(cudaSetDevice(e->device));
  CK(cudaMemset(e->llama->timing, 0, 32 * sizeof(unsigned long long)));
  return LA_OK;
}

extern "C" int32_t la_gemm_timing_read(la_engine* e, double* out16) {
  if (!e || !e->llama || !out16) { la_set_error("no bf16 path on this engine"); return LA_ERR_INVALID_CONFIG; }
  CK(cudaSetDevice(e->device));
  unsigned long long t[32];
  CK(cudaMemcpy(t, e->llama->timing, sizeof(t), cudaMemcpyDeviceToHost));
  for (int k = 0; k < 4; ++k) {
    out16[4 * k + 0] = (double)t[8 * k + 1];   // summed ns
    out16[4 * k + 1] = (double)t[8 * k + 2];   // launches
    out16[4 * k + 2] = 0.0;
    out16[4 * k + 3] = 0.0;
  }
  return LA_OK;
}
