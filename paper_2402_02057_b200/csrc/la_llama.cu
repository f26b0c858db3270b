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
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>


#include "la_attn.cuh"
#include "la_engine.h"
#include "la_gemm.cuh"
#include "la_mega.cuh"
#include "la_kernels.h"
#include "la_reduce.cuh"

#define CK(x) LA_CUDA_CHECK(x)
#define RET_IF(x)               \
  do {                          \
    int _r = (x);               \
    if (_r != LA_OK) return _r; \
  } while (0)

struct LlamaLayerW {
  const __nv_bfloat16 *wqkv, *wo, *wgu, *wd;   // packed LA tiles (la_gemm.cuh)
  const float *attn_norm, *mlp_norm;
};

struct LlamaPath {
  int d = 0, L = 0, H = 0, KVH = 0, ffn = 0, V = 0, NC = 1;
  float eps = 1e-5f;
  const __nv_bfloat16 *embed = nullptr, *lm_head = nullptr;
  const float* final_norm = nullptr;
  std::vector<LlamaLayerW> lw;
  float* x = nullptr;
  float* ss = nullptr;                    // [d/128][128] per-tile sums of x^2 (deferred RMSNorm)
  LaRowNorm nrm{};
  __nv_bfloat16 *h = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr;
  float* ws = nullptr;
  unsigned long long* keys = nullptr;     // [128] argmax keys
  float* part_o = nullptr;
  float2* part_ml = nullptr;
  float *rope_cos = nullptr, *rope_sin = nullptr;
  int* row_amax = nullptr;
  unsigned long long* timing = nullptr;   // [4 GEMM kinds][8]
  unsigned long long* trace = nullptr;    // [5 GEMM kinds][256 CTAs][8] (LA_GEMM_TRACE=1)
  unsigned long long* utrace = nullptr;   // [5][256][32] unit arrival times (LA_GEMM_TRACE=2)
  float* logits = nullptr;                // device dump target (parity hook), else null
  std::vector<LaGemm> qkv, o, gu, down;
  // dual-chunk prefill (LA_PREFILL_PAIR, default on): one-tile-per-unit configs
  // of the four projections (B = two 128-row prompt chunks per weight stage)
  // and the second chunk's activations
  int prefill_group = 1;                  // prompt chunks per weight pass (LA_PREFILL_GROUP, <= 4)
  std::vector<LaGemm> qkv1, o1, gu1, down1;
  struct ChunkBufs {                      // chunks 1..3 of a group (chunk 0 uses the step buffers)
    FwdPlan* plan = nullptr;
    float *x = nullptr, *ss = nullptr, *ws = nullptr;
    __nv_bfloat16 *h = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr;
  } cx[3];
  LaGemm head{};
  int head_tiles = 0;
  int kernels_per_step = 0;
  int loop_key = 0;                       // sampler shape the loop graph was built for
  bool spec_kv = false;                   // recording the WHILE-graph body: attention may read
                                          // the decode ctx + prefix K/V before its PDL wait
  bool pdl = true;                        // programmatic dependent launch (LA_PDL=0: off)
  bool fused = false;                     // GEMM-fused epilogues (LA_FUSED_EPI=1)
  int attn_rows = 64;                     // query rows per attention CTA (LA_ATTN_ROWS)
  int attn_min_chunk = 128;               // LA_ATTN_MIN_CHUNK
  bool attn_fused = true;                 // fused QKV fix-up + attention + merge (LA_ATTN_FUSED=0: 3 kernels)
  LaAttnFusedArgs af{};                   // its static arguments
  bool attn_o = false;                    // attention + O projection in one launch (LA_ATTN_O=1)
  bool head_fused = false;                // LM head epilogue inside its GEMM (LA_HEAD_FUSED=1)
  unsigned *ao_head = nullptr, *ao_exit = nullptr, *ao_err = nullptr;
  int skip = 0;                           // LA_SKIP: debug mask of per-layer launches to omit (timing only)
  bool mega = false;                      // persistent whole-forward kernel (LA_MEGA=1; experimental)
  LaMegaArgs ma{};
  // per-tile readiness (default; LA_TILE_READY=0: grid waits): the epilogue
  // kernels poll their tile's piece counter instead of waiting for the whole
  // GEMM grid (3 % per 7B lookahead step)
  bool tile_ready = false;
  std::vector<int*> runs_qkv, runs_o, runs_gu, runs_down;   // per layer: [epilogue grid] launch counts
  int* runs_head = nullptr;
  // every readiness counter / launch-count array: zeroed together (stream-
  // ordered) when a forward was left half-launched, so GEMMs and epilogues
  // never run out of lockstep (ready_dirty: a forward started and did not finish)
  std::vector<std::pair<void*, size_t>> readiness;
  bool ready_dirty = false;
  cudaStream_t cap = nullptr;
  cudaGraphExec_t loop_exec = nullptr;   // while(!done) { step }
  cudaGraphExec_t fwd_exec = nullptr;    // K1 + forward + owned argmax (LP)
  cudaGraph_t loop_graph = nullptr, fwd_graph = nullptr;
};

// ------------------------------------------------------------- kernels
namespace {

// prefill plan: causal chain over tokens[start, start+R)
__global__ void la_plan_chain_kernel(FwdPlan* P, const int* tokens, int start, int R) {
  LA_PDL_ENTRY();
  if (threadIdx.x == 0) {
    P->n_rows = R; P->n_pad = (R + 15) & ~15; P->n_prefix = start; P->n_global = R;
    P->want_logits = 0;
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
  LA_PDL_ENTRY();
  cudaGraphSetConditional(h, d->done ? 0u : 1u);
}

}  // namespace

// ------------------------------------------------------------ host setup
// tpc: tiles per stream-K unit.  Two tiles share one step-row load (half the
// L2 traffic of the activations); one tile halves the split-K partial volume
// of the narrow projections (O, down: only d/128 tiles for 148 SMs).
static int build_gemm(LaGemm& g, const void* a_packed, int n_tiles, const void* b, int K, int tpc,
                      int epi = LA_EPI_PARTIAL, int max_grid = 0) {
  memset(&g, 0, sizeof(g));
  g.epi = epi;
  n_tiles = (n_tiles + LA_TPC - 1) / LA_TPC * LA_TPC;   // packed buffers carry zero tiles
  g.args.a = reinterpret_cast<const __nv_bfloat16*>(a_packed);
  g.args.b = reinterpret_cast<const __nv_bfloat16*>(b);
  g.args.n_tiles = n_tiles;
  g.args.tpc = tpc;
  g.args.kb = K / 64;
  long U = (long)(n_tiles / tpc) * g.args.kb;
  g.grid = (int)std::min<long>(max_grid > 0 ? std::min(max_grid, la_sm_count()) : la_sm_count(), U);
  g.args.max_segs = la_gemm_workspace_segs(n_tiles, g.args.kb, g.grid, tpc);
  return LA_OK;
}

// L2 prefetch of a GEMM's first `frac` weight units per CTA (la_common.cuh)
static LaPrefetch prefetch_of(const LaGemm& g, float frac) {
  // opt-in (LA_L2_PREFETCH=<scale>): measured slower on B200 so far
  static const float scale = getenv("LA_L2_PREFETCH") ? (float)atof(getenv("LA_L2_PREFETCH")) : 0.0f;
  return LaPrefetch{g.args.a, g.args.n_tiles, g.args.kb, g.args.tpc, g.grid, frac * scale};
}

// fraction of a GEMM's weights that fits the HBM time of the kernels before it
static float pf_frac(const LaGemm& g, double bytes_budget) {
  double w = (double)g.args.n_tiles * g.args.kb * 16384.0;
  return (float)std::min(1.0, bytes_budget / w);
}

static LaSplit split_of(const LaGemm& g) {
  return LaSplit{g.args.n_tiles, g.args.kb, g.grid, g.args.max_segs, g.args.tpc};
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

static void tl_install(la_engine* e);   // LA_TIMELINE profiling hook (below)

void* g_attn_trace_host = nullptr;   // LA_ATTN_TRACE=2 debug buffer (host view)

// ------------------------------------------------ persistent forward kernel
static int mega_create(la_engine* e) {
  LlamaPath* p = e->llama;
  LaMegaArgs& a = p->ma;
  memset(&a, 0, sizeof(a));
  const int P = la_sm_count();
  a.L = p->L; a.d = p->d; a.H = p->H; a.KVH = p->KVH; a.ffn = p->ffn; a.V = p->V;
  a.slots = e->slots; a.eps = p->eps;
  a.embed = p->embed; a.lm_head = p->lm_head; a.final_norm = p->final_norm;
  // decomposition per projection: the step-row operand is cheap to re-read
  // (L2), split-K partials are not, so one tile per unit everywhere; wide
  // projections (gate/up, LM head: >= one tile per SM) give every CTA one
  // whole tile (epilogue straight from TMEM) and split only the remainder
  const bool use_dp = !(getenv("LA_MEGA_DP") && atoi(getenv("LA_MEGA_DP")) == 0);
  auto geo = [&](int real, int tpc, int K, bool dp) {
    LaMegaGeo g;
    g.real = real; g.tpc = tpc;
    g.n_tiles = (real + tpc - 1) / tpc * tpc;
    g.kb = K / 64;
    g.dp = (dp && tpc == 1 && real >= P) ? P : 0;
    g.max_segs = g.n_tiles > g.dp ? la_gemm_workspace_segs(g.n_tiles - g.dp, g.kb, P, tpc) : 1;
    return g;
  };
  a.geo[LA_MK_QKV] = geo(p->H + 2 * p->KVH, 1, p->d, false);
  a.geo[LA_MK_O] = geo(p->d / 128, 1, p->H * 128, false);
  a.geo[LA_MK_GU] = geo(p->ffn / 64, 1, p->d, use_dp);
  a.geo[LA_MK_DOWN] = geo(p->d / 128, 1, p->ffn, false);
  a.geo[LA_MK_HEAD] = geo(p->head_tiles, 1, p->d, use_dp);
  for (int k = 0; k < 5; ++k)
    RET_IF(lalloc(e, &a.ws[k], (size_t)a.geo[k].n_tiles * a.geo[k].max_segs * 128 * 128));
  a.x = p->x; a.h_attn = p->h; a.attn_out = p->attn; a.act = p->act; a.q = p->q;
  RET_IF(lalloc(e, &a.h_mlp, (size_t)LA_MAX_ROWS * p->d));
  RET_IF(lalloc(e, &a.ss_attn, (size_t)p->d));
  RET_IF(lalloc(e, &a.ss_mlp, (size_t)p->d));
  a.kc = reinterpret_cast<__nv_bfloat16*>(e->kc);
  a.vc = reinterpret_cast<__nv_bfloat16*>(e->vc);
  a.rope_cos = p->rope_cos; a.rope_sin = p->rope_sin;
  // attention units: (KV head, 128-query-row block, key chunk); the prefix
  // split count depends on the model only (LP shards chunk identically)
  const int g = p->H / p->KVH;
  a.nrb_max = (LA_MAX_ROWS * g + 127) / 128;
  int units = std::max(2, std::min(9, P / (p->KVH * a.nrb_max)));
  if (getenv("LA_MEGA_SPLITS")) units = std::max(2, std::min(16, atoi(getenv("LA_MEGA_SPLITS")) + 1));
  a.attn_S = units - 1;
  const size_t n_units = (size_t)p->KVH * a.nrb_max * units;
  RET_IF(lalloc(e, &a.attn_ws, n_units * 128 * 128));
  RET_IF(lalloc(e, &a.attn_ml, n_units * 128));
  a.keys = p->keys; a.row_amax = p->row_amax;
  // sync area
  LaMegaSyncMap& m = a.sm;
  int off = 0;
  for (int k = 0; k < 4; ++k) { m.cnt[k] = off; off += a.geo[k].n_tiles; }
  m.rdy_qkv = off; off += a.geo[LA_MK_QKV].n_tiles;
  m.attn_cnt = off; off += p->KVH * a.nrb_max;
  m.rdy_attn = off; off += p->KVH;
  m.rdy_m = off; off += p->d / 128;
  m.rdy_act = off; off += a.geo[LA_MK_GU].n_tiles;
  m.rdy_h = off; off += p->d / 128;
  m.layer_stride = (off + 31) & ~31;
  off = m.layer_stride * p->L;
  m.h0 = off; off += p->d / 128;
  m.head_cnt = off; off += a.geo[LA_MK_HEAD].n_tiles;
  m.head_done = off++;
  m.head_gen = off++;
  m.cta_done = off++;
  m.gen = off++;
  m.err = off++;
  m.total = off;
  RET_IF(lalloc(e, &a.sync, (size_t)m.total));
  CK(cudaMemset(a.sync, 0, (size_t)m.total * sizeof(unsigned)));
  std::vector<LaMegaLayer> lw(p->L);
  for (int l = 0; l < p->L; ++l)
    lw[l] = LaMegaLayer{p->lw[l].wqkv, p->lw[l].wo, p->lw[l].wgu, p->lw[l].wd, p->lw[l].attn_norm,
                        p->lw[l].mlp_norm};
  LaMegaLayer* dl = nullptr;
  RET_IF(lalloc(e, &dl, (size_t)p->L));
  CK(cudaMemcpy(dl, lw.data(), lw.size() * sizeof(LaMegaLayer), cudaMemcpyHostToDevice));
  a.layers = dl;
  a.timing = p->timing + 32;
  a.debug = getenv("LA_MEGA_DEBUG") ? atoi(getenv("LA_MEGA_DEBUG")) : 0;
  a.pf_units = getenv("LA_MEGA_PF") ? std::max(0, atoi(getenv("LA_MEGA_PF"))) : 8;
  if (getenv("LA_MEGA_TRACE")) {
    a.trace_slots = 4 * p->L + 1 + p->L;
    RET_IF(lalloc(e, &a.trace, (size_t)P * a.trace_slots * 8));
  }
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
    int b = 3 + 6 * l;
    p->lw.push_back({B(b), B(b + 1), B(b + 2), B(b + 3), F(b + 4), F(b + 5)});
  }
  const int R = LA_MAX_ROWS, qd = D.heads * 128;
  RET_IF(lalloc(e, &p->x, (size_t)R * D.dim));
  RET_IF(lalloc(e, &p->ss, (size_t)D.dim));
  p->nrm = LaRowNorm{p->ss, D.dim / 128, 1.0f / (float)D.dim, D.norm_eps};
  RET_IF(lalloc(e, &p->h, (size_t)R * D.dim));
  RET_IF(lalloc(e, &p->q, (size_t)R * qd));
  RET_IF(lalloc(e, &p->attn, (size_t)R * qd));
  RET_IF(lalloc(e, &p->act, (size_t)R * D.ffn));
  RET_IF(lalloc(e, &p->row_amax, R));
  // prefix-attention split: ~2 CTAs per SM at full rows
  const int g = D.heads / D.kv_heads;
  p->attn_rows = getenv("LA_ATTN_ROWS") && atoi(getenv("LA_ATTN_ROWS")) == 128 ? 128 : 64;
  p->attn_min_chunk = getenv("LA_ATTN_MIN_CHUNK") ? std::max(64, atoi(getenv("LA_ATTN_MIN_CHUNK"))) : 128;
  const int rblocks = (R * g + p->attn_rows - 1) / p->attn_rows;
  // at most one chunk per 128 prefix keys (la_attn.cu); cap at ~2 CTAs/SM
  p->NC = std::max(1, std::min(8, (2 * la_sm_count() + D.kv_heads * rblocks - 1) / (D.kv_heads * rblocks)));
  if (getenv("LA_ATTN_NC")) p->NC = std::max(1, std::min(8, atoi(getenv("LA_ATTN_NC"))));
  RET_IF(lalloc(e, &p->part_o, (size_t)(p->NC + 1) * R * D.heads * 128));
  RET_IF(lalloc(e, &p->part_ml, (size_t)(p->NC + 1) * R * D.heads));
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
  __nv_bfloat16* kc = reinterpret_cast<__nv_bfloat16*>(e->kc);
  __nv_bfloat16* vc = reinterpret_cast<__nv_bfloat16*>(e->vc);
  p->qkv.resize(D.layers); p->o.resize(D.layers); p->gu.resize(D.layers); p->down.resize(D.layers);
  const int narrow_tpc = getenv("LA_NARROW_TPC") ? atoi(getenv("LA_NARROW_TPC")) : LA_TPC;   // measured: 2 > 1
  // stream-K fix-up + epilogue inside the GEMM (LA_FUSED_EPI=1) or in the
  // separate reduce kernels spread over the GPU (default: measured faster)
  const bool fused = getenv("LA_FUSED_EPI") && atoi(getenv("LA_FUSED_EPI"));
  p->fused = fused;
  // split-K fix-up + epilogue inside the decode GEMMs (LA_FX=1; measured
  // slower than the separate epilogue kernels: the next GEMM cannot preload
  // while the fix-up holds the SM).  Not with the experimental
  // paths that consume the raw pieces (megakernel, attention+O, QKV fix-up
  // inside attention).
  const bool exp_paths = (getenv("LA_MEGA") && atoi(getenv("LA_MEGA")) == 1) ||
                         (getenv("LA_ATTN_O") && atoi(getenv("LA_ATTN_O")) == 1) ||
                         (getenv("LA_ATTN_FUSE_QKV") && atoi(getenv("LA_ATTN_FUSE_QKV")) == 1);
  const bool fx_on = !fused && !exp_paths && getenv("LA_FX") && atoi(getenv("LA_FX")) == 1;
  // LA_FX_MASK (with LA_FX=1): which GEMMs fix up in-kernel -- bit 0 QKV,
  // 1 O (residual), 2 gate/up (SwiGLU), 3 down (residual); default all
  const int fx_mask = fx_on ? (getenv("LA_FX_MASK") ? atoi(getenv("LA_FX_MASK")) : 15) : 0;
  size_t ws_need = 0;
  auto track = [&](const LaGemm& gg) {
    ws_need = std::max(ws_need, (size_t)gg.args.n_tiles * gg.args.max_segs * 128 * 128);
  };
  for (int l = 0; l < D.layers; ++l) {
    const LlamaLayerW& w = p->lw[l];
    RET_IF(build_gemm(p->qkv[l], w.wqkv, H + 2 * KVH, p->h, d, LA_TPC,
                      fused ? LA_EPI_QKV : (fx_mask & 1) ? LA_EPI_FX_QKV : LA_EPI_PARTIAL));
    p->qkv[l].args.n_real = H + 2 * KVH;
    {
      LaGemmArgs& q = p->qkv[l].args;
      q.q_out = p->q;
      q.kc = kc + (size_t)l * e->slots * KVH * 128;
      q.vc = vc + (size_t)l * e->slots * KVH * 128;
      q.rope_cos = p->rope_cos; q.rope_sin = p->rope_sin;
      q.H = H; q.KVH = KVH;
    }
    track(p->qkv[l]);
    // LA_O_GRID / LA_DOWN_GRID: fewer CTAs = fewer split-K pieces per tile (experiment)
    static const int o_grid = getenv("LA_O_GRID") ? atoi(getenv("LA_O_GRID")) : 0;
    RET_IF(build_gemm(p->o[l], w.wo, d / 128, p->attn, H * 128, narrow_tpc,
                      (fx_mask & 2) ? LA_EPI_FX_RESID : LA_EPI_PARTIAL, o_grid));
    track(p->o[l]);
    // gate/up: whole tiles per CTA with SwiGLU from TMEM + an in-kernel fixed-up
    // stream-K remainder (LA_GU_DPSK=1; measured slower than split-K pieces +
    // the SwiGLU kernel: the per-CTA epilogue / fix-up tail)
    const bool dpsk_on = getenv("LA_GU_DPSK") && atoi(getenv("LA_GU_DPSK")) == 1;
    const int dpsk_segs = la_gemm_dpsk_segs(D.ffn / 64, d / 64, la_sm_count());
    if (dpsk_on && !fused && !exp_paths && !(fx_mask & 4) && dpsk_segs > 0) {
      RET_IF(build_gemm(p->gu[l], w.wgu, D.ffn / 64, p->h, d, 1, LA_EPI_DPSK_SWIGLU));
      p->gu[l].args.max_segs = dpsk_segs;
    } else {
      RET_IF(build_gemm(p->gu[l], w.wgu, D.ffn / 64, p->h, d, LA_TPC,
                        fused ? LA_EPI_SWIGLU : (fx_mask & 4) ? LA_EPI_FX_SWIGLU : LA_EPI_PARTIAL));
    }
    p->gu[l].args.act = p->act;
    p->gu[l].args.n_real = D.ffn / 64;
    track(p->gu[l]);
    static const int down_grid = getenv("LA_DOWN_GRID") ? atoi(getenv("LA_DOWN_GRID")) : 0;
    RET_IF(build_gemm(p->down[l], w.wd, d / 128, p->act, D.ffn, narrow_tpc,
                      (fx_mask & 8) ? LA_EPI_FX_RESID : LA_EPI_PARTIAL, down_grid));
    track(p->down[l]);
    // residual epilogues: x += sum, then the NEXT norm's input and statistics
    for (LaGemm* g : {&p->o[l], &p->down[l]}) {
      g->args.n_real = d / 128;
      g->args.x = p->x; g->args.h_out = p->h; g->args.ss_out = p->ss; g->args.d = d;
    }
    p->o[l].args.gain = w.mlp_norm;
    p->down[l].args.gain = l + 1 < D.layers ? p->lw[l + 1].attn_norm : p->final_norm;
  }
  p->prefill_group = fused ? 1 : std::max(1, std::min(4, getenv("LA_PREFILL_GROUP") ? atoi(getenv("LA_PREFILL_GROUP")) : 4));
  if (p->prefill_group > 1) {
    p->qkv1.resize(D.layers); p->o1.resize(D.layers); p->gu1.resize(D.layers); p->down1.resize(D.layers);
    for (int l = 0; l < D.layers; ++l) {
      const LlamaLayerW& w = p->lw[l];
      RET_IF(build_gemm(p->qkv1[l], w.wqkv, H + 2 * KVH, p->h, d, 1));
      RET_IF(build_gemm(p->o1[l], w.wo, d / 128, p->attn, H * 128, 1));
      RET_IF(build_gemm(p->gu1[l], w.wgu, D.ffn / 64, p->h, d, 1));
      RET_IF(build_gemm(p->down1[l], w.wd, d / 128, p->act, D.ffn, 1));
      track(p->qkv1[l]); track(p->o1[l]); track(p->gu1[l]); track(p->down1[l]);
    }
  }
  p->head_tiles = (D.vocab + 127) / 128;
  // LA_HEAD_FUSED=1: the LM head's logits / argmax epilogue inside its GEMM
  // (most tile pairs are owned whole by one CTA: ~54 units per CTA)
  p->head_fused = fused || (getenv("LA_HEAD_FUSED") && atoi(getenv("LA_HEAD_FUSED")) == 1);
  RET_IF(build_gemm(p->head, p->lm_head, p->head_tiles, p->h, d, LA_TPC,
                    p->head_fused ? LA_EPI_LOGITS : LA_EPI_PARTIAL));
  track(p->head);
  RET_IF(lalloc(e, &p->keys, LA_MAX_ROWS));
  p->head.args.keys = p->keys;
  p->head.args.V = D.vocab;
  int* counters = nullptr;
  RET_IF(lalloc(e, &counters, 4096));
  int* fx_cnt = nullptr;
  RET_IF(lalloc(e, &fx_cnt, 2 * 4096));
  RET_IF(lalloc(e, &p->ws, ws_need));
  for (int j = 0; j + 1 < p->prefill_group; ++j) {
    const size_t R = LA_MAX_ROWS, qd = (size_t)H * 128;
    LlamaPath::ChunkBufs& c = p->cx[j];
    RET_IF(lalloc(e, &c.ws, ws_need));
    RET_IF(lalloc(e, &c.plan, 1));
    RET_IF(lalloc(e, &c.x, R * d));
    RET_IF(lalloc(e, &c.ss, (size_t)d));
    RET_IF(lalloc(e, &c.h, R * d));
    RET_IF(lalloc(e, &c.q, R * qd));
    RET_IF(lalloc(e, &c.attn, R * qd));
    RET_IF(lalloc(e, &c.act, R * (size_t)D.ffn));
  }
  RET_IF(lalloc(e, &p->timing, 48));
  const bool trace = getenv("LA_GEMM_TRACE") != nullptr;
  if (trace) RET_IF(lalloc(e, &p->trace, 5 * 256 * 8));   // qkv, o, gu, head, down
  if (trace && atoi(getenv("LA_GEMM_TRACE")) == 2) RET_IF(lalloc(e, &p->utrace, 5 * 3 * 256 * 32));
  const int dbg = getenv("LA_GEMM_DEBUG") ? atoi(getenv("LA_GEMM_DEBUG")) : 0;
  const int l2pf = getenv("LA_GEMM_L2PF") ? atoi(getenv("LA_GEMM_L2PF")) : 0;
  auto fin = [&](LaGemm& gg, int kind, int tkind) {
    gg.args.plan = e->d_plan; gg.args.ws = p->ws; gg.args.debug = dbg; gg.args.counters = counters;
    gg.args.fx_arrive = fx_cnt; gg.args.fx_depart = fx_cnt + 4096;
    if (gg.epi >= LA_EPI_FX_QKV && gg.epi <= LA_EPI_FX_RESID && !la_gemm_fx_fits(gg)) gg.epi = LA_EPI_PARTIAL;   // staging > ring
    // split-K pieces accumulated swap-AB (default) or as (step rows x weight
    // rows) with LA_GEMM_NT=1 (4x fewer MMAs per unit, but its TMEM drain
    // runs on half the lanes' warps at <= 64 rows; measured slower)
    const bool nt = getenv("LA_GEMM_NT") && atoi(getenv("LA_GEMM_NT")) == 1;
    if (!nt && gg.epi == LA_EPI_PARTIAL) gg.epi = LA_EPI_PARTIAL_SW;
    gg.args.l2pf = l2pf;
    // in-kernel launch timing is opt-in (la_gemm_timing_enable / LA_GEMM_TIMING=1):
    // its atomics sit on the producer thread's path and cost ~4 % of a step
    static const int timing_on = getenv("LA_GEMM_TIMING") ? atoi(getenv("LA_GEMM_TIMING")) : 0;
    gg.args.timing = timing_on ? p->timing + 8 * kind : nullptr;
    gg.args.trace = trace ? p->trace + 256 * 8 * tkind : nullptr;
    gg.args.utrace = p->utrace ? p->utrace + 3 * 256 * 32 * tkind : nullptr;
  };
  for (int l = 0; l < D.layers; ++l) {
    fin(p->qkv[l], 0, 0); fin(p->o[l], 1, 1); fin(p->gu[l], 2, 2); fin(p->down[l], 1, 4);
  }
  for (size_t l = 0; l < p->qkv1.size(); ++l)
    for (LaGemm* g : {&p->qkv1[l], &p->o1[l], &p->gu1[l], &p->down1[l]}) {
      g->args.plan = e->d_plan; g->args.ws = p->ws; g->args.counters = counters;
    }
  for (int l = 0; l < D.layers; ++l) { p->qkv[l].args.nrm = p->nrm; p->gu[l].args.nrm = p->nrm; }
  {
    // O projection ring depth (LA_O_STAGES; 0 = the default 4 stages).  A
    // 3-stage ring fits beside an attention CTA register-wise only when the
    // attention kernel is capped at <= 184 registers (per-SM-sub-partition
    // register files: 2 warps x 32 x (attention + GEMM regs) <= 16384); that
    // configuration co-resided on only part of the SMs and measured no gain.
    const int ost = getenv("LA_O_STAGES") ? atoi(getenv("LA_O_STAGES")) : 0;
    for (int l = 0; l < D.layers; ++l)
      if (p->o[l].args.tpc == LA_TPC) p->o[l].args.nst = ost;
  }
  p->head.args.nrm = p->nrm;
  fin(p->head, 3, 3);
  p->tile_ready = !(getenv("LA_TILE_READY") && atoi(getenv("LA_TILE_READY")) == 0) && !fused && !exp_paths;
  if (p->tile_ready) {
    auto counted = [&](int** ptr, size_t n) -> int {
      RET_IF(lalloc(e, ptr, n));
      p->readiness.emplace_back(*ptr, n * sizeof(int));
      return LA_OK;
    };
    auto ready_for = [&](LaGemm& gg) -> int { return counted(&gg.args.ready, (size_t)(gg.args.n_tiles / gg.args.tpc)); };
    p->runs_qkv.resize(D.layers); p->runs_o.resize(D.layers); p->runs_gu.resize(D.layers); p->runs_down.resize(D.layers);
    for (int l = 0; l < D.layers; ++l) {
      RET_IF(ready_for(p->qkv[l])); RET_IF(ready_for(p->o[l])); RET_IF(ready_for(p->gu[l])); RET_IF(ready_for(p->down[l]));
      RET_IF(counted(&p->runs_qkv[l], (size_t)(H + 2 * KVH) * 16));
      RET_IF(counted(&p->runs_o[l], (size_t)(d / 128) * 16));
      RET_IF(counted(&p->runs_gu[l], (size_t)(D.ffn / 64) * 16));
      RET_IF(counted(&p->runs_down[l], (size_t)(d / 128) * 16));
    }
    RET_IF(ready_for(p->head));
    RET_IF(counted(&p->runs_head, (size_t)((D.vocab + 127) / 128) * 16));
  }
  {
    // cross-GEMM L2 prefetch (LA_NPF=<MB next>[,<MB after next>]): each
    // decode GEMM, once its own loads are issued, pulls the first units of
    // the next GEMMs' per-CTA ranges into L2 (the head wraps to layer 0)
    double mb[2] = {0.0, 0.0};
    if (const char* s = getenv("LA_NPF")) sscanf(s, "%lf,%lf", &mb[0], &mb[1]);
    std::vector<LaGemm*> seq;
    for (int l = 0; l < D.layers; ++l) { seq.push_back(&p->qkv[l]); seq.push_back(&p->o[l]); seq.push_back(&p->gu[l]); seq.push_back(&p->down[l]); }
    seq.push_back(&p->head);
    for (size_t i = 0; i < seq.size(); ++i)
      for (int j = 0; j < 2; ++j) {
        const LaGemm& nx = *seq[(i + 1 + j) % seq.size()];
        const double unit = (double)nx.args.tpc * 16384.0;
        const long per_cta = (long)(nx.args.n_tiles / nx.args.tpc) * nx.args.kb / nx.grid + 1;
        int units = (int)std::min<double>((double)per_cta, mb[j] * 1e6 / (unit * nx.grid));
        LaNextPf& q = seq[i]->args.npf[j];
        // skip what the next GEMM's own smem ring pre-loads during its early
        // (PDL) launch -- except the O projection, which cannot become
        // resident beside attention
        static const int skip_env = getenv("LA_NPF_SKIP") ? atoi(getenv("LA_NPF_SKIP")) : -1;
        const bool is_o = (i + 1 + j) % 4 == 1 && (i + 1 + j) < seq.size() - 1;
        const int skip = skip_env >= 0 ? skip_env : (!is_o ? (nx.args.tpc == LA_TPC ? 4 : 6) : 0);
        q = LaNextPf{nx.args.a, nx.args.n_tiles, nx.args.kb, nx.args.tpc, nx.grid, skip, units};
        if (units <= 0) q.a = nullptr;
      }
  }
  CK(cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking));
  p->pdl = !(getenv("LA_PDL") && !strcmp(getenv("LA_PDL"), "0"));
  p->skip = getenv("LA_SKIP") ? atoi(getenv("LA_SKIP")) : 0;
  cudaError_t ce = cudaFuncSetAttribute(la_attn_chunks_kernel<128>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)la_attn_prefix_smem(128));
  if (ce == cudaSuccess)
    ce = cudaFuncSetAttribute(la_attn_chunks_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)la_attn_prefix_smem(64));
  if (ce != cudaSuccess) { la_set_error("attn smem attr: %s", cudaGetErrorString(ce)); return LA_ERR_CUDA; }
  // fused attention: (KV head, 128 query rows, key chunk) units, one CTA per
  // SM at most; prefix chunk count depends on the model only
  p->attn_fused = !(getenv("LA_ATTN_FUSED") && atoi(getenv("LA_ATTN_FUSED")) == 0);
  {
    LaAttnFusedArgs& af = p->af;
    af.H = p->H; af.KVH = p->KVH;
    af.nrb_max = (LA_MAX_ROWS * g + 127) / 128;
    // key splits per (KV head, row block): sized for the row blocks of a
    // typical step (<= 64 query tokens: ceil(64 g / 128) blocks) rather than
    // the 128-row maximum, so GQA models keep several chunks per KV head; a
    // launch whose active units exceed the SMs falls back to the last-arriver
    // merge in-kernel (same chunk-order combine: identical results)
    const int nrb_typ = std::max(1, std::min(af.nrb_max, (64 * g + 127) / 128));
    int units = std::max(2, std::min(9, la_sm_count() / (p->KVH * nrb_typ)));
    if (getenv("LA_ATTN_SPLITS")) units = std::max(2, std::min(16, atoi(getenv("LA_ATTN_SPLITS")) + 1));
    af.S = units - 1;
    // co-residency (1 CTA per SM, grid <= SMs) makes the spread merge's wait safe
    af.spread_merge = (p->KVH * af.nrb_max * units <= la_sm_count()) && !getenv("LA_ATTN_LAST_MERGE");
    af.sms = getenv("LA_ATTN_LAST_MERGE") ? 0 : la_sm_count();
    // optional (LA_ATTN_FUSE_QKV=1): the QKV epilogue inside the attention
    // kernel behind a grid barrier (needs every CTA co-resident).  Measured
    // slower: 32K threads reduce the partials ~3x slower than the separate
    // wide kernel, more than the saved dependency hop.
    af.fuse_qkv = af.spread_merge && !p->fused && getenv("LA_ATTN_FUSE_QKV") && atoi(getenv("LA_ATTN_FUSE_QKV")) == 1;
    RET_IF(lalloc(e, &af.gbar, 1));
    // tcgen05 chunk attention (LA_ATTN_TC=1): correct (same outputs as the
    // mma.sync path on the parity tests) but measured slower on cfg2 -- its
    // S -> softmax -> PV phases serialise (no cross-tile pipelining yet)
    af.tc = getenv("LA_ATTN_TC") && atoi(getenv("LA_ATTN_TC")) == 1;
    // LA_ATTN_CLUSTER=1: the S+1 chunk CTAs of each (KV head, row block) form
    // a cluster; partials are pushed into the merging CTA's smem (remote
    // stores) and merged after one cluster barrier.  Measured equal to the
    // global partials + counter path (the barrier costs what the atomics did).
    af.cluster = af.spread_merge && !af.tc && !af.fuse_qkv && units <= 8 &&
                 getenv("LA_ATTN_CLUSTER") && atoi(getenv("LA_ATTN_CLUSTER")) == 1;
    af.dbg = getenv("LA_ATTN_DBG") ? atoi(getenv("LA_ATTN_DBG")) : 0;
    // key tiles split by parity over the two warp groups (la_attn_ks_kernel)
    // (2: its K/V tiles by TMA from tensor maps over the whole cache).  Default:
    // the TMA variant when a full cache gives chunks of >= 8 key tiles (13B,
    // 3.5K keys: attention 51 -> 45 us per layer, step -2%, greedy -5%); the
    // plain kernel for short caches (7B, 0.5-1K keys: key-split +1-2 us per
    // layer).  Fixed per engine, so every decode on it computes alike.
    const int cache_tiles = ((e->slots + af.S - 1) / af.S + 63) / 64;
    const char* ks_env = getenv("LA_ATTN_KSPLIT");
    const int ks = ks_env ? std::max(0, std::min(2, atoi(ks_env))) : (cache_tiles >= 8 ? 2 : 0);
    af.ksplit = (!af.tc && !af.cluster && !af.fuse_qkv) ? ks : 0;
    af.kv_pf = getenv("LA_ATTN_KV_PF") && atoi(getenv("LA_ATTN_KV_PF")) == 1;
    // key-split kernel: the step block rides with the last of S + 1 prefix
    // chunks instead of being a unit of its own -- no unit holds one lone tile
    // while the others hold 28 (13B, 3.5K keys: lookahead step 6.77 -> 6.53 ms,
    // greedy 5.96 -> 5.73).  Default with the long-cache (TMA) choice; with
    // short caches (7B, 0.5K keys) measured +0.6 %: LA_ATTN_FOLD=0/1 overrides.
    const char* fold_env = getenv("LA_ATTN_FOLD");
    af.fold_step = af.ksplit && (fold_env ? atoi(fold_env) == 1 : (!ks_env && ks == 2));
    af.spec_ctx = nullptr;
    if (af.ksplit == 2) {
      CUtensorMap maps[2];
      const int rows = p->L * e->slots;
      RET_IF(la_make_tmap(&maps[0], e->kc, rows, p->KVH * 128, 64));
      RET_IF(la_make_tmap(&maps[1], e->vc, rows, p->KVH * 128, 64));
      CUtensorMap* dm = nullptr;
      RET_IF(lalloc(e, reinterpret_cast<uint8_t**>(&dm), sizeof(maps)));
      CK(cudaMemcpy(dm, maps, sizeof(maps), cudaMemcpyHostToDevice));
      af.kmap = dm;
      af.vmap = dm + 1;
    }
    af.scale = 1.0f / sqrtf(128.0f);
    af.q = p->q;
    af.out = p->attn;
    // flat mapping of the key-split kernel (LA_ATTN_FLAT=1): one CTA per SM over
    // the KVH x prefix-tile space; needs one row block and KVH <= SMs (a CTA's
    // range then meets at most two heads)
    af.flat = af.ksplit == 2 && af.nrb_max == 1 && p->KVH <= la_sm_count() && getenv("LA_ATTN_FLAT") &&
              atoi(getenv("LA_ATTN_FLAT")) == 1;
    af.flat_maxp = (la_sm_count() + p->KVH - 1) / p->KVH + 1;
    const size_t groups = (size_t)p->KVH * af.nrb_max;
    const size_t slots_per = af.flat ? std::max<size_t>(units, af.flat_maxp) : units;
    RET_IF(lalloc(e, &af.part_o, groups * slots_per * 128 * 128));
    RET_IF(lalloc(e, &af.part_ml, groups * slots_per * 128));
    RET_IF(lalloc(e, &af.cnt, groups));
    if (af.flat) {
      RET_IF(lalloc(e, &af.fcnt, (size_t)p->KVH));
      RET_IF(lalloc(e, &af.fdone, (size_t)p->KVH));
      p->readiness.emplace_back(af.fcnt, (size_t)p->KVH * sizeof(unsigned));
      p->readiness.emplace_back(af.fdone, (size_t)p->KVH * sizeof(unsigned));
    }
    // attention + O in one persistent launch: needs every attention unit and
    // every O CTA co-resident (one CTA per SM) and the O GEMM on all SMs
    p->attn_o = getenv("LA_ATTN_O") && atoi(getenv("LA_ATTN_O")) == 1 && af.spread_merge && !af.tc &&
                !af.fuse_qkv && !p->fused && !p->mega;
    if (p->attn_o) {
      RET_IF(lalloc(e, &p->ao_head, (size_t)p->KVH));
      RET_IF(lalloc(e, &p->ao_exit, 1));
      RET_IF(lalloc(e, &p->ao_err, 1));
    }
    if (getenv("LA_ATTN_TRACE")) {
      const size_t ctas = std::max(groups * units, (size_t)la_sm_count());
      if (atoi(getenv("LA_ATTN_TRACE")) == 2) {
        // mapped host memory: readable by a host watchdog while a kernel hangs
        void* hp = nullptr;
        CK(cudaHostAlloc(&hp, ctas * 64, cudaHostAllocMapped));
        memset(hp, 0, ctas * 64);
        g_attn_trace_host = hp;
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&af.trace), hp, 0));
      } else {
        RET_IF(lalloc(e, &af.trace, ctas * 8));
      }
    }
    ce = cudaFuncSetAttribute(la_attn_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)la_attn_fused_smem(true));
    if (ce != cudaSuccess) { la_set_error("fused attn smem attr: %s", cudaGetErrorString(ce)); return LA_ERR_CUDA; }
  }
  p->mega = getenv("LA_MEGA") && atoi(getenv("LA_MEGA")) == 1;
  tl_install(e);
  if (p->mega) RET_IF(mega_create(e));
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

// ------------------------------------------------- per-kernel event timing
// LA_KTIME=1 (eager mode only): CUDA events around every launch, summed per
// kernel kind and printed to stderr after each decode -- a warm-cache
// breakdown of the real step (ncu serialises and flushes caches).
struct KTimer {
  bool on = false;
  cudaStream_t st = nullptr;
  std::vector<std::pair<const char*, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  void begin(cudaStream_t s) { st = s; }
  void mark(const char* name, cudaEvent_t a, cudaEvent_t b) { marks.push_back({name, {a, b}}); }
};
static KTimer g_kt;
static cudaEvent_t kt_event() {
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
#define KT_BEGIN(st)                       \
  cudaEvent_t _kt_a = nullptr;             \
  if (g_kt.on) {                           \
    _kt_a = kt_event();                    \
    cudaEventRecord(_kt_a, st);            \
  }
#define KT_END(st, name)                   \
  if (g_kt.on) {                           \
    cudaEvent_t _kt_b = kt_event();        \
    cudaEventRecord(_kt_b, st);            \
    g_kt.mark(name, _kt_a, _kt_b);         \
  }

static void kt_report() {
  if (!g_kt.on || g_kt.marks.empty()) return;
  cudaDeviceSynchronize();
  std::vector<std::pair<std::string, std::pair<double, int>>> acc;
  for (auto& m : g_kt.marks) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, m.second.first, m.second.second);
    bool found = false;
    for (auto& a : acc)
      if (a.first == m.first) { a.second.first += ms; a.second.second++; found = true; }
    if (!found) acc.push_back({m.first, {ms, 1}});
    cudaEventDestroy(m.second.first);
    cudaEventDestroy(m.second.second);
  }
  double tot = 0;
  for (auto& a : acc) tot += a.second.first;
  fprintf(stderr, "[la ktime] %-18s %8s %10s %8s\n", "kernel", "count", "mean_us", "share");
  for (auto& a : acc)
    fprintf(stderr, "[la ktime] %-18s %8d %10.2f %7.1f%%\n", a.first.c_str(), a.second.second,
            a.second.first * 1e3 / a.second.second, 100.0 * a.second.first / tot);
  fprintf(stderr, "[la ktime] total %.3f ms\n", tot);
  g_kt.marks.clear();
}

// ------------------------------------------------------------- timeline
void la_tl_set_gemm(unsigned long long*);
void la_tl_set_reduce(unsigned long long*);
void la_tl_set_attnf(unsigned long long*);
void la_tl_set_attn(unsigned long long*);
void la_tl_set_llama(unsigned long long*);
void la_tl_set_state(unsigned long long*);
void la_tl_set_mega(unsigned long long*);
void la_tl_set_sample(unsigned long long*);
static unsigned long long* g_tl_buf = nullptr;
static void tl_install(la_engine* e) {
  if (!getenv("LA_TIMELINE") || g_tl_buf) return;
  (void)e;   // process-lifetime profiling buffer (not owned by an engine)
  if (cudaMalloc(&g_tl_buf, (1 + 2 * LA_TL_CAP) * 8) != cudaSuccess) { g_tl_buf = nullptr; return; }
  cudaMemset(g_tl_buf, 0, (1 + 2 * LA_TL_CAP) * 8);
  la_tl_set_gemm(g_tl_buf); la_tl_set_reduce(g_tl_buf); la_tl_set_attnf(g_tl_buf); la_tl_set_attn(g_tl_buf);
  la_tl_set_llama(g_tl_buf); la_tl_set_state(g_tl_buf); la_tl_set_mega(g_tl_buf);
  la_tl_set_sample(g_tl_buf);
}

// ------------------------------------------------------------- forward
// timing experiment (LA_EMPTY=K): K empty PDL launches per layer
__global__ void la_empty_kernel(int) { LA_PDL_ENTRY(); }

static int launch_attn(la_engine* e, int l, cudaStream_t st) {
  LlamaPath* p = e->llama;
  LaAttnArgs a;
  // the O projection's remaining weights stream into L2 during attention
  a.pf = prefetch_of(p->o[l], 1.0f);
  a.plan = e->d_plan;
  a.q = p->q;
  const size_t lstride = (size_t)e->slots * p->KVH * 128;
  a.kc = reinterpret_cast<const __nv_bfloat16*>(e->kc) + l * lstride;
  a.vc = reinterpret_cast<const __nv_bfloat16*>(e->vc) + l * lstride;
  a.part_o = p->part_o;
  a.part_ml = p->part_ml;
  a.out = p->attn;
  a.H = p->H; a.KVH = p->KVH; a.NC = p->NC; a.min_chunk = p->attn_min_chunk;
  a.scale = 1.0f / sqrtf(128.0f);
  const int g = p->H / p->KVH;
  const int qr = p->attn_rows;
  dim3 grid(p->KVH, p->NC, (LA_MAX_ROWS * g + qr - 1) / qr);
  {
    KT_BEGIN(st);
    if (qr == 128)
      CK(la_launch(la_attn_chunks_kernel<128>, grid, dim3(256), la_attn_prefix_smem(128), st, p->pdl, a));
    else
      CK(la_launch(la_attn_chunks_kernel<64>, grid, dim3(128), la_attn_prefix_smem(64), st, p->pdl, a));
    KT_END(st, "attn_chunks");
  }
  {
    KT_BEGIN(st);
    CK(la_launch(la_attn_merge_kernel, dim3(LA_MAX_ROWS), dim3(32 * std::min(p->H, 16)), 0, st,
                 p->pdl, a));
    KT_END(st, "attn_merge");
  }
  CK(cudaGetLastError());
  return LA_OK;
}

static int launch_attn_fused(la_engine* e, int l, cudaStream_t st) {
  LlamaPath* p = e->llama;
  LaAttnFusedArgs a = p->af;
  a.plan = e->d_plan;
  {
    // the O projection cannot be co-resident with attention (smem): stream its
    // first weights into L2 meanwhile (LA_ATTN_PF = fraction; measured no gain, off)
    static const float frac = getenv("LA_ATTN_PF") ? (float)atof(getenv("LA_ATTN_PF")) : 0.0f;
    const LaGemm& g = p->o[l];
    a.pf = LaPrefetch{g.args.a, g.args.n_tiles, g.args.kb, g.args.tpc, g.grid, frac};
  }
  const size_t lstride = (size_t)e->slots * p->KVH * 128;
  a.kc = reinterpret_cast<__nv_bfloat16*>(e->kc) + l * lstride;
  a.vc = reinterpret_cast<__nv_bfloat16*>(e->vc) + l * lstride;
  a.kv_row0 = l * e->slots;
  // each WHILE-loop iteration starts after the previous one completed, so the
  // decode state's ctx and the committed prefix K/V are final before any wait
  a.spec_ctx = p->spec_kv ? &e->d_dec->ctx : nullptr;
  if (a.fuse_qkv) {
    __nv_bfloat16* kc = reinterpret_cast<__nv_bfloat16*>(e->kc) + l * lstride;
    __nv_bfloat16* vc = reinterpret_cast<__nv_bfloat16*>(e->vc) + l * lstride;
    a.qkv = LaQkvEpi{LaPrefetch{}, e->d_plan, p->ws, split_of(p->qkv[l]), p->q, kc, vc, p->rope_cos,
                     p->rope_sin, p->H, p->KVH, p->nrm};
  }
  KT_BEGIN(st);
  CK(la_attn_fused_launch(a, a.flat ? la_sm_count() : p->KVH * a.nrb_max * (a.S + 1), st, p->pdl));
  KT_END(st, "attn_fused");
  return LA_OK;
}

static int resid_norm(la_engine* e, const LaGemm* from, const float* g, bool embed, cudaStream_t st,
                      const LaGemm* next, int* runs = nullptr) {
  LlamaPath* p = e->llama;
  LaResidNorm r;
  r.pf = next ? prefetch_of(*next, pf_frac(*next, 40e6)) : LaPrefetch{};
  r.plan = e->d_plan;
  r.ws = from ? p->ws : nullptr;
  r.sp = from ? split_of(*from) : LaSplit{2, 1, 1, 1, 1};
  r.embed = embed ? p->embed : nullptr;
  r.x = p->x; r.g = g; r.h = p->h; r.d = p->d; r.eps = p->eps; r.ss = p->ss;
  if (from && runs && from->args.ready) { r.ready = from->args.ready; r.runs = runs; }
  KT_BEGIN(st);
  static const int rb = getenv("LA_RESID_RB") ? atoi(getenv("LA_RESID_RB")) : LA_MAX_ROWS / 8;
  CK(la_launch(la_resid_norm_kernel, dim3(p->d / 128, rb), dim3(256), 0, st, p->pdl, r));
  KT_END(st, from ? "resid_norm" : "embed_norm");
  CK(cudaGetLastError());
  return LA_OK;
}

// start of a forward part (layers or head): re-zero the readiness counters if
// the previous part was left half-launched (a launch failed mid-way)
static int readiness_reset_if_dirty(la_engine* e, cudaStream_t st) {
  LlamaPath* p = e->llama;
  if (p->ready_dirty)
    for (const auto& r : p->readiness) CK(cudaMemsetAsync(r.first, 0, r.second, st));
  p->ready_dirty = false;
  return LA_OK;
}
static int readiness_begin(la_engine* e, cudaStream_t st) {
  LlamaPath* p = e->llama;
  RET_IF(readiness_reset_if_dirty(e, st));
  p->ready_dirty = !p->readiness.empty();
  return LA_OK;
}

// all decoder layers on the rows of e->d_plan; leaves h = final-norm(x)
static int forward_layers(la_engine* e, cudaStream_t st, int* nk) {
  LlamaPath* p = e->llama;
  RET_IF(readiness_begin(e, st));
  __nv_bfloat16* kc = reinterpret_cast<__nv_bfloat16*>(e->kc);
  __nv_bfloat16* vc = reinterpret_cast<__nv_bfloat16*>(e->vc);
  const size_t lstride = (size_t)e->slots * p->KVH * 128;
  RET_IF(resid_norm(e, nullptr, p->lw[0].attn_norm, true, st, &p->qkv[0]));
  int n = 1;
  for (int l = 0; l < p->L; ++l) {
    {
      KT_BEGIN(st);
      if (!(p->skip & 64)) RET_IF(la_gemm_launch(p->qkv[l], st, p->pdl));
      KT_END(st, "gemm_qkv");
    }
    if (!p->fused && !(p->attn_fused && p->af.fuse_qkv) && p->qkv[l].epi != LA_EPI_FX_QKV) {
      LaQkvEpi q{prefetch_of(p->o[l], pf_frac(p->o[l], 20e6)), e->d_plan, p->ws,
                 split_of(p->qkv[l]), p->q, kc + l * lstride, vc + l * lstride, p->rope_cos,
                 p->rope_sin, p->H, p->KVH, p->nrm};
      if (p->tile_ready) { q.ready = p->qkv[l].args.ready; q.runs = p->runs_qkv[l]; }
      KT_BEGIN(st);
      if (!(p->skip & 1)) {
        static const int rb = getenv("LA_QKV_RB") ? atoi(getenv("LA_QKV_RB")) : LA_MAX_ROWS / 8;
        CK(la_launch(la_qkv_epi_kernel, dim3(p->H + 2 * p->KVH, rb), dim3(128), 0, st, p->pdl, q));
      }
      KT_END(st, "qkv_epi");
      ++n;
    }
    if (p->attn_o && p->o[l].grid == la_sm_count() && p->o[l].args.tpc == LA_TPC) {
      LaAttnOArgs x;
      x.at = p->af;
      x.at.plan = e->d_plan;
      x.at.kc = kc + l * lstride;
      x.at.vc = vc + l * lstride;
      x.at.pf = LaPrefetch{};
      x.at.trace = nullptr;
      x.at.cluster = 0;
      x.g = p->o[l].args;   // trace (LA_GEMM_TRACE): entry, attention done, first head ready, end
      x.g.timing = nullptr;
      x.head_done = p->ao_head; x.exit_cnt = p->ao_exit; x.err = p->ao_err;
      x.nst = 3;
      x.g.l2pf = getenv("LA_ATTN_O_L2") ? atoi(getenv("LA_ATTN_O_L2")) : 0;   // measured slower when on
      KT_BEGIN(st);
      CK(la_attn_o_launch(x, la_sm_count(), st, p->pdl));
      KT_END(st, "attn+o");
      --n;
    } else {
      if (!(p->skip & 2)) RET_IF(p->attn_fused ? launch_attn_fused(e, l, st) : launch_attn(e, l, st));
      KT_BEGIN(st);
      if (!(p->skip & 128)) RET_IF(la_gemm_launch(p->o[l], st, p->pdl));
      KT_END(st, "gemm_o");
    }
    if (!(p->skip & 8) && p->o[l].epi != LA_EPI_FX_RESID)
      RET_IF(resid_norm(e, &p->o[l], p->lw[l].mlp_norm, false, st, &p->gu[l],
                        p->tile_ready ? p->runs_o[l] : nullptr));
    {
      KT_BEGIN(st);
      if (!(p->skip & 256)) RET_IF(la_gemm_launch(p->gu[l], st, p->pdl));
      KT_END(st, "gemm_gu");
    }
    if (!p->fused && p->gu[l].epi != LA_EPI_FX_SWIGLU && p->gu[l].epi != LA_EPI_DPSK_SWIGLU) {
      LaSwigluEpi sw{prefetch_of(p->down[l], pf_frac(p->down[l], 40e6)), e->d_plan, p->ws,
                     split_of(p->gu[l]), p->act, p->ffn, p->nrm};
      if (p->tile_ready) { sw.ready = p->gu[l].args.ready; sw.runs = p->runs_gu[l]; }
      KT_BEGIN(st);
      if (!(p->skip & 16)) {
        static const int rb = getenv("LA_SWIGLU_RB") ? atoi(getenv("LA_SWIGLU_RB")) : LA_MAX_ROWS / 16;
        CK(la_launch(la_swiglu_epi_kernel, dim3(p->ffn / 64, rb), dim3(128), 0, st, p->pdl, sw));
      }
      KT_END(st, "swiglu_epi");
      ++n;
    }
    {
      KT_BEGIN(st);
      if (!(p->skip & 512)) RET_IF(la_gemm_launch(p->down[l], st, p->pdl));
      KT_END(st, "gemm_down");
    }
    {
      static const int n_empty = getenv("LA_EMPTY") ? atoi(getenv("LA_EMPTY")) : 0;
      for (int i = 0; i < n_empty; ++i) CK(la_launch(la_empty_kernel, dim3(148), dim3(128), 0, st, p->pdl, i));
    }
    const float* next = (l + 1 < p->L) ? p->lw[l + 1].attn_norm : p->final_norm;
    if (!(p->skip & 32) && p->down[l].epi != LA_EPI_FX_RESID)
      RET_IF(resid_norm(e, &p->down[l], next, false, st, l + 1 < p->L ? &p->qkv[l + 1] : &p->head,
                        p->tile_ready ? p->runs_down[l] : nullptr));
    CK(cudaGetLastError());
    // 4 GEMMs + attention (1 fused, or chunks + merge) + the residual norms not fused into O / down
    n += (p->attn_fused ? 5 : 6) + (p->o[l].epi != LA_EPI_FX_RESID) + (p->down[l].epi != LA_EPI_FX_RESID);
  }
  *nk += n;
  p->ready_dirty = false;
  return LA_OK;
}

static int forward_head(la_engine* e, cudaStream_t st, bool scatter, int* nk) {
  LlamaPath* p = e->llama;
  RET_IF(readiness_begin(e, st));
  p->head.args.logits = p->logits;
  {
    KT_BEGIN(st);
    RET_IF(la_gemm_launch(p->head, st, p->pdl));
    KT_END(st, "gemm_head");
  }
  KT_BEGIN(st);
  if (!p->head_fused) {
    LaLogitsEpi lg{e->d_plan, p->ws, split_of(p->head), p->keys, p->logits, p->V, p->nrm};
    if (p->tile_ready) { lg.ready = p->head.args.ready; lg.runs = p->runs_head; }
    CK(la_launch(la_logits_epi_kernel, dim3(p->head_tiles, LA_MAX_ROWS / 8), dim3(128), 0, st, p->pdl, lg));
    *nk += 1;
  }
  CK(la_launch(la_argmax_finish_kernel, dim3(1), dim3(LA_MAX_ROWS), 0, st, p->pdl, e->d_plan,
               p->keys, p->row_amax, scatter ? e->d_dec : nullptr));
  KT_END(st, "logits_argmax");
  CK(cudaGetLastError());
  *nk += 2;
  p->ready_dirty = false;
  return LA_OK;
}

// the whole forward (+ LM head / argmax) as ONE persistent launch
static int mega_forward(la_engine* e, cudaStream_t st, bool head, bool scatter, int* nk) {
  LlamaPath* p = e->llama;
  LaMegaArgs a = p->ma;
  a.plan = e->d_plan;
  a.dec = scatter ? e->d_dec : nullptr;
  a.do_head = head ? 1 : 0;
  a.logits = p->logits;
  KT_BEGIN(st);
  CK(la_mega_launch(a, la_sm_count(), st, p->pdl));
  KT_END(st, "mega_forward");
  *nk += 1;
  return LA_OK;
}

// Up to four 128-row prompt chunks through all layers, layer-major: every
// projection streams its weights ONCE for the group (multi-chunk GEMM,
// tpc = 1); the epilogues and attention run per chunk with the chunk's own plan
// and activations, in chunk order (chunk i's attention reads the keys of
// chunks < i of the same layer).
static int prefill_chunks(la_engine* e, const int* d_tokens, int start, int n_chunks, int n_tok,
                          cudaStream_t st) {
  LlamaPath* p = e->llama;
  struct Chunk {
    FwdPlan* plan; float *x, *ss, *ws; __nv_bfloat16 *h, *q, *attn, *act;
  } c[4];
  c[0] = {e->d_plan, p->x, p->ss, p->ws, p->h, p->q, p->attn, p->act};
  for (int j = 1; j < n_chunks; ++j) {
    const LlamaPath::ChunkBufs& b = p->cx[j - 1];
    c[j] = {b.plan, b.x, b.ss, b.ws, b.h, b.q, b.attn, b.act};
  }
  for (int i = 0; i < n_chunks; ++i) {
    const int s0 = start + i * LA_MAX_ROWS;
    la_plan_chain_kernel<<<1, 128, 0, st>>>(c[i].plan, d_tokens, s0, std::min(LA_MAX_ROWS, start + n_tok - s0));
  }
  CK(cudaGetLastError());
  auto nrm = [&](int i) { LaRowNorm r = p->nrm; r.ss = c[i].ss; return r; };
  auto resid = [&](int i, const LaGemm* from, const float* g, bool embed) -> int {
    LaResidNorm r;
    r.pf = LaPrefetch{};
    r.plan = c[i].plan;
    r.ws = from ? c[i].ws : nullptr;
    r.sp = from ? split_of(*from) : LaSplit{2, 1, 1, 1, 1};
    r.embed = embed ? p->embed : nullptr;
    r.x = c[i].x; r.g = g; r.h = c[i].h; r.d = p->d; r.eps = p->eps; r.ss = c[i].ss;
    static const int rb = getenv("LA_RESID_RB") ? atoi(getenv("LA_RESID_RB")) : LA_MAX_ROWS / 8;
  CK(la_launch(la_resid_norm_kernel, dim3(p->d / 128, rb), dim3(256), 0, st, p->pdl, r));
    return LA_OK;
  };
  auto multi = [&](const LaGemm& g0, __nv_bfloat16* Chunk::*b) -> int {
    LaGemm g = g0;
    g.args.nblk = n_chunks;
    g.args.b = c[0].*b; g.args.ws = c[0].ws; g.args.plan = c[0].plan;
    for (int j = 1; j < n_chunks; ++j) {
      g.args.bx[j - 1] = c[j].*b; g.args.wsx[j - 1] = c[j].ws; g.args.planx[j - 1] = c[j].plan;
    }
    return la_gemm_launch(g, st, p->pdl);
  };
  __nv_bfloat16* kc = reinterpret_cast<__nv_bfloat16*>(e->kc);
  __nv_bfloat16* vc = reinterpret_cast<__nv_bfloat16*>(e->vc);
  const size_t lstride = (size_t)e->slots * p->KVH * 128;
  for (int i = 0; i < n_chunks; ++i) RET_IF(resid(i, nullptr, p->lw[0].attn_norm, true));
  for (int l = 0; l < p->L; ++l) {
    RET_IF(multi(p->qkv1[l], &Chunk::h));
    for (int i = 0; i < n_chunks; ++i) {
      LaQkvEpi q{LaPrefetch{}, c[i].plan, c[i].ws, split_of(p->qkv1[l]), c[i].q, kc + l * lstride,
                 vc + l * lstride, p->rope_cos, p->rope_sin, p->H, p->KVH, nrm(i)};
      {
        static const int rb = getenv("LA_QKV_RB") ? atoi(getenv("LA_QKV_RB")) : LA_MAX_ROWS / 8;
        CK(la_launch(la_qkv_epi_kernel, dim3(p->H + 2 * p->KVH, rb), dim3(128), 0, st, p->pdl, q));
      }
    }
    for (int i = 0; i < n_chunks; ++i) {
      LaAttnFusedArgs a = p->af;
      a.plan = c[i].plan; a.q = c[i].q; a.out = c[i].attn;
      a.kc = kc + l * lstride; a.vc = vc + l * lstride;
      a.kv_row0 = l * e->slots;
      a.spec_ctx = nullptr;
      a.pf = LaPrefetch{};
      CK(la_attn_fused_launch(a, a.flat ? la_sm_count() : p->KVH * a.nrb_max * (a.S + 1), st, p->pdl));
    }
    RET_IF(multi(p->o1[l], &Chunk::attn));
    for (int i = 0; i < n_chunks; ++i) RET_IF(resid(i, &p->o1[l], p->lw[l].mlp_norm, false));
    RET_IF(multi(p->gu1[l], &Chunk::h));
    for (int i = 0; i < n_chunks; ++i) {
      LaSwigluEpi sw{LaPrefetch{}, c[i].plan, c[i].ws, split_of(p->gu1[l]), c[i].act, p->ffn, nrm(i)};
      {
        static const int rb = getenv("LA_SWIGLU_RB") ? atoi(getenv("LA_SWIGLU_RB")) : LA_MAX_ROWS / 16;
        CK(la_launch(la_swiglu_epi_kernel, dim3(p->ffn / 64, rb), dim3(128), 0, st, p->pdl, sw));
      }
    }
    RET_IF(multi(p->down1[l], &Chunk::act));
    const float* next = (l + 1 < p->L) ? p->lw[l + 1].attn_norm : p->final_norm;
    for (int i = 0; i < n_chunks; ++i) RET_IF(resid(i, &p->down1[l], next, false));
    CK(cudaGetLastError());
  }
  return LA_OK;
}

int llama_prefill(la_engine* e, const int* d_tokens, int n, cudaStream_t st) {
  LlamaPath* p = e->llama;
  int start = 0;
  // groups of up to prefill_group 128-row chunks share every weight pass
  if (p->prefill_group > 1 && !p->mega && !p->af.fuse_qkv)
    while (start + LA_MAX_ROWS < n) {
      const int chunks = std::min(p->prefill_group, (n - start + LA_MAX_ROWS - 1) / LA_MAX_ROWS);
      const int tok = std::min(n - start, chunks * LA_MAX_ROWS);
      RET_IF(prefill_chunks(e, d_tokens, start, chunks, tok, st));
      start += tok;
    }
  for (; start < n; start += LA_MAX_ROWS) {
    int R = std::min(LA_MAX_ROWS, n - start);
    la_plan_chain_kernel<<<1, 128, 0, st>>>(e->d_plan, d_tokens, start, R);
    CK(cudaGetLastError());
    int nk = 0;
    if (e->llama->mega) RET_IF(mega_forward(e, st, false, false, &nk));
    else RET_IF(forward_layers(e, st, &nk));
  }
  return LA_OK;
}

int llama_forward_plan(la_engine* e, float* d_logits, cudaStream_t st) {
  LlamaPath* p = e->llama;
  p->logits = d_logits;
  int nk = 0;
  int rc;
  if (p->mega) {
    rc = mega_forward(e, st, true, false, &nk);
  } else {
    rc = forward_layers(e, st, &nk);
    if (rc == LA_OK) rc = forward_head(e, st, false, &nk);
  }
  p->logits = nullptr;
  return rc;
}

// one step's kernels: K1 -> forward -> argmax (-> K10 -> commit)
static int record_step(la_engine* e, cudaStream_t st, bool finish, int* nk) {
  LlamaPath* p = e->llama;
  {
    KT_BEGIN(st);
    CK(la_launch(la_step_build_kernel, dim3(1), dim3(256), 0, st, p->pdl, e->d_dec, e->d_plan));
    KT_END(st, "step_build");
  }
  CK(cudaGetLastError());
  *nk += 1;
  // temperature sampler: the LM head also dumps every row's logits for the
  // adjust kernel (one CTA per row verification may read), then one CTA
  // runs verify_sample (la_sample.cu)
  const bool smp = e->h_dec.sample != 0;
  if (smp) p->logits = e->d_logits;
  int rc = p->mega ? mega_forward(e, st, true, true, nk) : forward_layers(e, st, nk);
  if (rc == LA_OK && !p->mega) rc = forward_head(e, st, true, nk);
  if (smp) p->logits = nullptr;
  RET_IF(rc);
  if (finish && smp) {
    const DevDecode& h = e->h_dec;
    const int rows = h.mode == LA_MODE_LOOKAHEAD ? 1 + h.G * (h.N - 1) : 1;
    {
      KT_BEGIN(st);
      CK(la_launch(la_sample_adjust_cluster_kernel, dim3(rows * LA_ADJ_CLUSTER), dim3(LA_ADJ_THREADS), 0,
                   st, p->pdl, e->d_dec));
      KT_END(st, "sample_adjust");
    }
    KT_BEGIN(st);
    CK(la_launch(la_sample_verify_kernel, dim3(1), dim3(1024), 0, st, p->pdl, e->d_dec));
    KT_END(st, "sample_verify");
    *nk += 2;
  }
  if (finish) {
    KT_BEGIN(st);
    CK(la_launch(la_step_finish_kernel, dim3(1), dim3(256), 0, st, p->pdl, e->d_dec));
    KT_END(st, "step_finish+commit");
    CK(la_launch(la_kv_commit_kernel, dim3(std::max(1, std::min(148, p->L * e->row_bytes / 16 / 256))),
                 dim3(256), 0, st, p->pdl, (const DevDecode*)e->d_dec, (uint8_t*)e->kc,
                 (uint8_t*)e->vc, p->L, e->slots, e->row_bytes));
    CK(cudaGetLastError());
    *nk += 2;
  }
  return LA_OK;
}

// one whole step (K1 .. KV commit) as plain launches: step sessions
int llama_session_step(la_engine* e, cudaStream_t st) {
  int nk = 0;
  return record_step(e, st, true, &nk);
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
  p->spec_kv = !(getenv("LA_ATTN_SPEC") && atoi(getenv("LA_ATTN_SPEC")) == 0);
  int rc = record_step(e, p->cap, true, &nk);
  p->spec_kv = false;
  cudaError_t lce = la_launch(la_set_cond_kernel, dim3(1), dim3(1), 0, p->cap, p->pdl, handle, (const DevDecode*)e->d_dec);
  if (lce != cudaSuccess && rc == LA_OK) { la_set_error("set_cond launch: %s", cudaGetErrorString(lce)); rc = LA_ERR_CUDA; }
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

// LA_LAUNCH_MODE=eager: host loop of plain launches (profilers cannot see
// kernel nodes inside conditional graphs); default: one WHILE-graph launch.
static int eager_loop(la_engine* e, cudaStream_t st, int* launches) {
  g_kt.on = getenv("LA_KTIME") != nullptr;
  const bool saved_pdl = e->llama->pdl;
  if (g_kt.on) e->llama->pdl = false;   // events between kernels would serialise anyway
  static thread_local int* pinned = nullptr;
  if (!pinned) CK(cudaMallocHost(&pinned, sizeof(int)));
  int nk = 0;
  for (int step = 0; step < e->h_dec.max_steps; ++step) {
    RET_IF(record_step(e, st, true, &nk));
    if ((step + 1) % 4 == 0) {
      CK(cudaMemcpyAsync(pinned, &e->d_dec->done, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (*pinned) break;
    }
  }
  *launches = nk;
  kt_report();
  g_kt.on = false;
  e->llama->pdl = saved_pdl;
  return LA_OK;
}

int llama_decode_loop(la_engine* e, cudaStream_t st, int* launches) {
  LlamaPath* p = e->llama;
  const char* mode = getenv("LA_LAUNCH_MODE");
  if (mode && !strcmp(mode, "eager")) return eager_loop(e, st, launches);
  // the step graph differs per sampler shape: rebuild when it changes
  const DevDecode& h = e->h_dec;
  const int key = h.sample ? 1 + (h.mode == LA_MODE_LOOKAHEAD ? 1 + h.G * (h.N - 1) : 1) : 0;
  if (p->loop_exec && p->loop_key != key) {
    cudaGraphExecDestroy(p->loop_exec);
    cudaGraphDestroy(p->loop_graph);
    p->loop_exec = nullptr;
    p->loop_graph = nullptr;
  }
  if (!p->loop_exec) RET_IF(build_loop_graph(e));
  p->loop_key = key;
  RET_IF(readiness_reset_if_dirty(e, st));   // (a graph replay records no forward on the host)
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
  RET_IF(readiness_reset_if_dirty(e, st));
  CK(cudaGraphLaunch(p->fwd_exec, st));
  return LA_OK;
}

// debug: internal buffers of the persistent forward kernel (la_debug_read
// what >= 6): 6 sync counters, 7 x, 8 h_attn, 9 ss_attn, 10 q, 11 attn_out,
// 12 h_mlp, 13 ss_mlp, 14 act, 15 row_amax
bool llama_debug_buffer(la_engine* e, int what, const void** src, size_t* bytes) {
  LlamaPath* p = e->llama;
  if (!p) return false;
  const LaMegaArgs& a = p->ma;
  const size_t R = LA_MAX_ROWS;
  switch (what) {
    case 6: *src = a.sync; *bytes = (size_t)a.sm.total * 4; return a.sync != nullptr;
    case 7: *src = p->x; *bytes = R * p->d * 4; return true;
    case 8: *src = p->h; *bytes = R * p->d * 2; return true;
    case 9: *src = a.ss_attn; *bytes = (size_t)p->d * 4; return a.ss_attn != nullptr;
    case 10: *src = p->q; *bytes = R * p->H * 128 * 2; return true;
    case 11: *src = p->attn; *bytes = R * p->H * 128 * 2; return true;
    case 12: *src = a.h_mlp; *bytes = R * p->d * 2; return a.h_mlp != nullptr;
    case 13: *src = a.ss_mlp; *bytes = (size_t)p->d * 4; return a.ss_mlp != nullptr;
    case 14: *src = p->act; *bytes = R * p->ffn * 2; return true;
    case 15: *src = p->row_amax; *bytes = R * 4; return true;
    case 17:
      *src = p->af.trace;
      *bytes = std::max((size_t)p->KVH * p->af.nrb_max * (p->af.S + 1), (size_t)la_sm_count()) * 64;
      return p->af.trace != nullptr;
    case 18: *src = g_tl_buf; *bytes = (1 + 2 * LA_TL_CAP) * 8; return g_tl_buf != nullptr;
    case 20: *src = p->utrace; *bytes = 5 * 3 * 256 * 32 * 8; return p->utrace != nullptr;
    case 16: *src = a.trace; *bytes = (size_t)la_sm_count() * a.trace_slots * 64; return a.trace != nullptr;
    default: return false;
  }
}

// debug: per-CTA trace of the last launch of each GEMM kind (LA_GEMM_TRACE=1)
int llama_read_trace(la_engine* e, void* host, size_t bytes) {
  if (!e->llama || !e->llama->trace) { la_set_error("trace disabled (set LA_GEMM_TRACE=1)"); return LA_ERR_INVALID_CONFIG; }
  CK(cudaMemcpy(host, e->llama->trace, std::min<size_t>(bytes, 5 * 256 * 8 * 8), cudaMemcpyDeviceToHost));
  return LA_OK;
}

// ------------------------------------------------------- GEMM timing ABI
// switch the in-kernel launch timing of the GEMMs on / off (the cached step
// graphs bake the kernel arguments: they are rebuilt on next use)
extern "C" int32_t la_gemm_timing_enable(la_engine* e, int32_t on) {
  if (!e || !e->llama) { la_set_error("no bf16 path on this engine"); return LA_ERR_INVALID_CONFIG; }
  LlamaPath* p = e->llama;
  CK(cudaSetDevice(e->device));
  CK(cudaDeviceSynchronize());
  auto set = [&](LaGemm& g, int kind) { g.args.timing = on ? p->timing + 8 * kind : nullptr; };
  for (int l = 0; l < p->L; ++l) { set(p->qkv[l], 0); set(p->o[l], 1); set(p->gu[l], 2); set(p->down[l], 1); }
  set(p->head, 3);
  if (p->loop_exec) { cudaGraphExecDestroy(p->loop_exec); p->loop_exec = nullptr; }
  if (p->loop_graph) { cudaGraphDestroy(p->loop_graph); p->loop_graph = nullptr; }
  if (p->fwd_exec) { cudaGraphExecDestroy(p->fwd_exec); p->fwd_exec = nullptr; }
  if (p->fwd_graph) { cudaGraphDestroy(p->fwd_graph); p->fwd_graph = nullptr; }
  return LA_OK;
}

extern "C" int32_t la_gemm_timing_reset(la_engine* e) {
  if (!e || !e->llama) { la_set_error("no bf16 path on this engine"); return LA_ERR_INVALID_CONFIG; }
  CK(cudaSetDevice(e->device));
  CK(cudaMemset(e->llama->timing, 0, 48 * sizeof(unsigned long long)));
  return LA_OK;
}

// device time of the persistent forward kernel: [summed ns, launches] since
// the last la_gemm_timing_reset; 0 launches when the multi-kernel path ran
extern "C" int32_t la_forward_timing_read(la_engine* e, double* out2) {
  if (!e || !e->llama || !out2) { la_set_error("no bf16 path on this engine"); return LA_ERR_INVALID_CONFIG; }
  CK(cudaSetDevice(e->device));
  unsigned long long t[8];
  CK(cudaMemcpy(t, e->llama->timing + 32, sizeof(t), cudaMemcpyDeviceToHost));
  out2[0] = (double)t[1];
  out2[1] = (double)t[2];
  return LA_OK;
}

// per-row greedy argmax of the last forward (la_argmax_finish_kernel / the
// megakernel's head fix-up write row_amax)
cudaError_t llama_copy_argmax(la_engine* e, int32_t* host, int n, cudaStream_t st) {
  return cudaMemcpyAsync(host, e->llama->row_amax, (size_t)n * 4, cudaMemcpyDeviceToHost, st);
}

// spin-timeout flag of the persistent kernel (a dependency never satisfied)
int llama_mega_error(la_engine* e) {
  LlamaPath* p = e->llama;
  if (p && p->attn_o) {
    unsigned v = 0;
    if (cudaMemcpy(&v, p->ao_err, sizeof(v), cudaMemcpyDeviceToHost) == cudaSuccess && v) return 1;
  }
  if (!p || !p->mega) return 0;
  unsigned v = 0;
  if (cudaMemcpy(&v, p->ma.sync + p->ma.sm.err, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return (int)v;
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

LA_TL_DEFINE_SETTER(llama)
