// C-ABI implementation: engine lifetime, decode orchestration, parity hook.
//
// The host side of a decode is: validate -> upload inputs once -> launch the
// device decode (one megakernel for fp32 tiny models, one CUDA graph per
// step for the bf16 path) -> read outputs once.  No token crosses PCIe inside
// the decode loop.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "la_engine.h"
#include "la_kernels.h"
#include "la_sample.cuh"

static thread_local char g_err[2048];

void la_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* la_last_error(void) { return g_err; }
extern "C" int32_t la_abi_version(void) { return 2; }   // 2: la_decode_io.pool_capacity

#define CK(x) LA_CUDA_CHECK(x)
#define RET_IF(x)              \
  do {                         \
    int _r = (x);              \
    if (_r != LA_OK) return _r; \
  } while (0)

// ------------------------------------------------------------------ weights
static const char* kGptLayer[] = {"wq", "wk", "wv", "wo", "w1", "b1",
                                  "w2", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b"};
static const char* kGptTop[] = {"embed", "unembed", "lnf_g", "lnf_b"};
static const char* kLlamaLayer[] = {"wq", "wk", "wv", "wo", "w_gate",
                                    "w_up", "w_down", "attn_norm", "mlp_norm"};
static const char* kLlamaTop[] = {"embed", "lm_head", "final_norm"};
// bf16 path: projection matrices in the packed LA-tile layout (la_pack_weight)
static const char* kPackedLayer[] = {"wqkv_tiles", "wo_tiles", "wgu_tiles", "wd_tiles",
                                     "attn_norm", "mlp_norm"};
static const char* kPackedTop[] = {"embed", "lm_head_tiles", "final_norm"};

extern "C" int32_t la_weight_count(const la_model_desc* d) {
  if (!d) return 0;
  if (d->arch == LA_ARCH_GPT_F32) return 4 + 12 * d->layers;
  if (d->arch == LA_ARCH_LLAMA_BF16) return 3 + 6 * d->layers;
  return 3 + 9 * d->layers;
}

extern "C" const char* la_weight_name(const la_model_desc* d, int32_t i) {
  static thread_local char buf[64];
  if (!d || i < 0 || i >= la_weight_count(d)) return nullptr;
  if (d->arch == LA_ARCH_GPT_F32) {
    if (i < 4) return kGptTop[i];
    snprintf(buf, sizeof(buf), "%d.%s", (i - 4) / 12, kGptLayer[(i - 4) % 12]);
  } else if (d->arch == LA_ARCH_LLAMA_BF16) {
    if (i < 3) return kPackedTop[i];
    snprintf(buf, sizeof(buf), "%d.%s", (i - 3) / 6, kPackedLayer[(i - 3) % 6]);
  } else {
    if (i < 3) return kLlamaTop[i];
    snprintf(buf, sizeof(buf), "%d.%s", (i - 3) / 9, kLlamaLayer[(i - 3) % 9]);
  }
  return buf;
}

// ------------------------------------------------------------------ helpers
template <typename T>
static int dalloc(la_engine* e, T** p, size_t count) {
  void* q = nullptr;
  size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  CK(cudaMalloc(&q, bytes));
  CK(cudaMemset(q, 0, bytes));
  e->owned.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return LA_OK;
}

template <typename T>
static int dgrow(la_engine* e, T** p, int* cap, size_t need) {
  if (*p && (size_t)*cap >= need) return LA_OK;
  if (*p) {
    auto it = std::find(e->owned.begin(), e->owned.end(), (void*)*p);
    if (it != e->owned.end()) e->owned.erase(it);
    CK(cudaFree(*p));
    *p = nullptr;
  }
  size_t n = std::max<size_t>(need, 64);
  RET_IF(dalloc(e, p, n));
  *cap = (int)n;
  return LA_OK;
}

static size_t pow2_at_least(size_t x) {
  size_t p = 16;
  while (p < x) p <<= 1;
  return p;
}

static int check_desc(const la_model_desc* d) {
  if (!d) { la_set_error("null model descriptor"); return LA_ERR_INVALID_CONFIG; }
  if (d->arch < 0 || d->arch > 2) { la_set_error("unknown arch %d", d->arch); return LA_ERR_INVALID_CONFIG; }
  if (d->vocab < 1 || d->dim < 1 || d->layers < 1 || d->heads < 1 || d->kv_heads < 1 ||
      d->head_dim < 1 || d->ffn < 1 || d->max_context < 2) {
    la_set_error("all model dimensions must be positive");
    return LA_ERR_INVALID_CONFIG;
  }
  if (d->heads % d->kv_heads) { la_set_error("heads must be a multiple of kv_heads"); return LA_ERR_INVALID_CONFIG; }
  if (d->arch == LA_ARCH_GPT_F32 && (d->heads * d->head_dim != d->dim || d->kv_heads != d->heads)) {
    la_set_error("GPT model needs dim == heads * head_dim and no GQA");
    return LA_ERR_INVALID_CONFIG;
  }
  if (d->arch != LA_ARCH_LLAMA_BF16 && d->layers > TINY_MAX_LAYERS) {
    la_set_error("fp32 SIMT path supports at most %d layers", TINY_MAX_LAYERS);
    return LA_ERR_UNSUPPORTED;
  }
  if (d->arch == LA_ARCH_GPT_F32 && (d->dim % 2)) { la_set_error("dim must be even"); return LA_ERR_INVALID_CONFIG; }
  if (d->arch != LA_ARCH_GPT_F32 && (d->head_dim % 2)) { la_set_error("head_dim must be even"); return LA_ERR_INVALID_CONFIG; }
  if (d->arch != LA_ARCH_LLAMA_BF16 && d->head_dim > TINY_MAX_HD) {
    la_set_error("fp32 SIMT path supports head_dim <= %d", TINY_MAX_HD);
    return LA_ERR_UNSUPPORTED;
  }
  int elt = d->arch == LA_ARCH_LLAMA_BF16 ? 2 : 4;
  if ((d->kv_heads * d->head_dim * elt) % 16) {
    la_set_error("kv_heads*head_dim*%d must be a multiple of 16 bytes", elt);
    return LA_ERR_UNSUPPORTED;
  }
  return LA_OK;
}

// ------------------------------------------------------------- tiny setup
static int tiny_setup(la_engine* e) {
  const la_model_desc& d = e->desc;
  TinyModel& m = e->tm;
  m.arch = d.arch == LA_ARCH_GPT_F32 ? TINY_ARCH_GPT : TINY_ARCH_LLAMA;
  m.V = d.vocab; m.d = d.dim; m.L = d.layers; m.H = d.heads; m.KVH = d.kv_heads;
  m.hd = d.head_dim; m.ff = d.ffn; m.eps = d.norm_eps; m.slots = e->slots;
  auto W = [&](int i) { return reinterpret_cast<const float*>(e->w[i]); };
  if (m.arch == TINY_ARCH_GPT) {
    m.embed = W(0); m.unembed = W(1); m.lnf_g = W(2); m.lnf_b = W(3);
    for (int l = 0; l < d.layers; ++l) {
      int b = 4 + 12 * l;
      TinyLayer& L = m.layers[l];
      L.wq = W(b); L.wk = W(b + 1); L.wv = W(b + 2); L.wo = W(b + 3);
      L.w1 = W(b + 4); L.b1 = W(b + 5); L.w2 = W(b + 6); L.b2 = W(b + 7);
      L.ln1_g = W(b + 8); L.ln1_b = W(b + 9); L.ln2_g = W(b + 10); L.ln2_b = W(b + 11);
      L.wu = nullptr;
    }
    // sinusoidal table in float64, stored fp32 (models.py:174-180)
    std::vector<float> tab((size_t)e->slots * d.dim);
    for (int p = 0; p < e->slots; ++p)
      for (int i = 0; i < d.dim / 2; ++i) {
        double inv = std::pow(10000.0, -(2.0 * i) / d.dim);
        double a = p * inv;
        tab[(size_t)p * d.dim + 2 * i] = (float)std::sin(a);
        tab[(size_t)p * d.dim + 2 * i + 1] = (float)std::cos(a);
      }
    float* dt;
    RET_IF(dalloc(e, &dt, tab.size()));
    CK(cudaMemcpy(dt, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
    m.pos_tab = dt;
  } else {
    m.embed = W(0); m.unembed = W(1); m.lnf_g = W(2); m.lnf_b = nullptr;
    for (int l = 0; l < d.layers; ++l) {
      int b = 3 + 9 * l;
      TinyLayer& L = m.layers[l];
      L.wq = W(b); L.wk = W(b + 1); L.wv = W(b + 2); L.wo = W(b + 3);
      L.w1 = W(b + 4); L.wu = W(b + 5); L.w2 = W(b + 6); L.b1 = nullptr; L.b2 = nullptr;
      L.ln1_g = W(b + 7); L.ln1_b = nullptr; L.ln2_g = W(b + 8); L.ln2_b = nullptr;
    }
  }
  if (m.arch == TINY_ARCH_LLAMA) {
    const int half = d.head_dim / 2;
    std::vector<float> c((size_t)e->slots * half), s((size_t)e->slots * half);
    for (int p = 0; p < e->slots; ++p)
      for (int i = 0; i < half; ++i) {
        double inv = 1.0 / std::pow((double)d.rope_theta, (2.0 * i) / d.head_dim);
        c[(size_t)p * half + i] = (float)std::cos(p * inv);
        s[(size_t)p * half + i] = (float)std::sin(p * inv);
      }
    float *dc, *ds;
    RET_IF(dalloc(e, &dc, c.size()));
    RET_IF(dalloc(e, &ds, s.size()));
    CK(cudaMemcpy(dc, c.data(), c.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice));
    m.rope_cos = dc; m.rope_sin = ds;
  }
  {
    // transposed weight copies ([in][out]) for coalesced reads in la_tiny.cu
    const int qd = m.H * m.hd, kvd = m.KVH * m.hd, nqkv = qd + 2 * kvd;
    auto tr = [&](const float* src, int rows, int cols, float* dst, int ld, int off) -> int {
      la_tiny_transpose<<<64, 256>>>(src, rows, cols, dst, ld, off);
      CK(cudaGetLastError());
      return LA_OK;
    };
    for (int l = 0; l < m.L; ++l) {
      TinyLayer& L = m.layers[l];
      float *qkv, *o, *w1, *w2, *wu = nullptr;
      RET_IF(dalloc(e, &qkv, (size_t)m.d * nqkv));
      RET_IF(dalloc(e, &o, (size_t)qd * m.d));
      RET_IF(dalloc(e, &w1, (size_t)m.d * m.ff));
      RET_IF(dalloc(e, &w2, (size_t)m.ff * m.d));
      RET_IF(tr(L.wq, qd, m.d, qkv, nqkv, 0));
      RET_IF(tr(L.wk, kvd, m.d, qkv, nqkv, qd));
      RET_IF(tr(L.wv, kvd, m.d, qkv, nqkv, qd + kvd));
      RET_IF(tr(L.wo, m.d, qd, o, m.d, 0));
      RET_IF(tr(L.w1, m.ff, m.d, w1, m.ff, 0));
      RET_IF(tr(L.w2, m.d, m.ff, w2, m.d, 0));
      if (L.wu) {
        RET_IF(dalloc(e, &wu, (size_t)m.d * m.ff));
        RET_IF(tr(L.wu, m.ff, m.d, wu, m.ff, 0));
      }
      L.wqkvT = qkv; L.woT = o; L.w1T = w1; L.w2T = w2; L.wuT = wu;
    }
    float* ut;
    RET_IF(dalloc(e, &ut, (size_t)m.d * m.V));
    RET_IF(tr(m.unembed, m.V, m.d, ut, m.V, 0));
    m.unembedT = ut;
    CK(cudaDeviceSynchronize());
  }
  m.kcache = reinterpret_cast<float*>(e->kc);
  m.vcache = reinterpret_cast<float*>(e->vc);
  TinyScratch& s = e->ts;
  const int R = LA_MAX_ROWS;
  const int qd = d.heads * d.head_dim;
  RET_IF(dalloc(e, &s.x, (size_t)R * d.dim));
  RET_IF(dalloc(e, &s.h, (size_t)R * d.dim));
  RET_IF(dalloc(e, &s.q, (size_t)R * qd));
  RET_IF(dalloc(e, &s.att, (size_t)R * qd));
  RET_IF(dalloc(e, &s.ff, (size_t)R * d.ffn));
  RET_IF(dalloc(e, &s.row_amax, R));
  e->tiny_smem = la_tiny_smem_bytes(m, &s.smem);
  if (e->tiny_smem && la_tiny_set_smem(e->tiny_smem) != 0) {
    la_set_error("fp32 path: dynamic shared memory attribute (%zu B) refused", e->tiny_smem);
    return LA_ERR_CUDA;
  }
  return LA_OK;
}

// ------------------------------------------------------------------ create
extern "C" int32_t la_create(const la_model_desc* desc, const void* const* weights,
                             int32_t n_weights, int32_t device, la_engine** out) {
  if (!out) { la_set_error("null output pointer"); return LA_ERR_INVALID_CONFIG; }
  *out = nullptr;
  RET_IF(check_desc(desc));
  if (n_weights != la_weight_count(desc) || !weights) {
    la_set_error("expected %d weight pointers, got %d", la_weight_count(desc), n_weights);
    return LA_ERR_INVALID_CONFIG;
  }
  for (int i = 0; i < n_weights; ++i)
    if (!weights[i]) { la_set_error("weight %d (%s) is null", i, la_weight_name(desc, i)); return LA_ERR_INVALID_CONFIG; }
  CK(cudaSetDevice(device));
  auto* e = new la_engine();
  e->desc = *desc;
  e->device = device;
  e->w.assign(weights, weights + n_weights);
  const int elt = desc->arch == LA_ARCH_LLAMA_BF16 ? 2 : 4;
  e->slots = desc->max_context + LA_MAX_ROWS;
  e->row_bytes = desc->kv_heads * desc->head_dim * elt;
  int rc = LA_OK;
  do {
    size_t kv_bytes = (size_t)desc->layers * e->slots * e->row_bytes;
    if ((rc = dalloc(e, reinterpret_cast<uint8_t**>(&e->kc), kv_bytes))) break;
    if ((rc = dalloc(e, reinterpret_cast<uint8_t**>(&e->vc), kv_bytes))) break;
    if ((rc = dalloc(e, &e->d_dec, 1))) break;
    if ((rc = dalloc(e, &e->d_plan, 1))) break;
    if ((rc = dalloc(e, &e->d_window, 64 * LA_MAX_NGRAM))) break;
    if ((rc = dalloc(e, &e->d_cand, 64 * LA_MAX_NGRAM))) break;
    if ((rc = dalloc(e, &e->d_amax, LA_MAX_ROWS))) break;
    if ((rc = dalloc(e, &e->d_acc, LA_MAX_NGRAM + 2))) break;
    e->out_cap = desc->max_context + 2 * LA_MAX_NGRAM;
    e->rec_cap = desc->max_context + 1;
    if ((rc = dalloc(e, &e->d_out, e->out_cap))) break;
    if ((rc = dalloc(e, &e->d_rec, (size_t)e->rec_cap * 4))) break;
    for (auto& ev : e->ev) {
      cudaError_t ce = cudaEventCreate(&ev);
      if (ce != cudaSuccess) { la_set_error("cudaEventCreate: %s", cudaGetErrorString(ce)); rc = LA_ERR_CUDA; break; }
    }
    if (rc) break;
    if (e->is_tiny()) rc = tiny_setup(e);
    else rc = llama_create(e);
  } while (0);
  if (rc != LA_OK) {
    std::string msg = g_err;
    la_destroy(e);
    la_set_error("%s", msg.c_str());
    return rc;
  }
  *out = e;
  return LA_OK;
}

void lp_destroy(la_engine* e);

extern "C" int32_t la_destroy(la_engine* e) {
  if (!e) return LA_OK;
  cudaSetDevice(e->device);
  cudaDeviceSynchronize();
  if (e->llama) llama_destroy(e);
  if (e->lp) lp_destroy(e);
  for (auto ev : e->ev)
    if (ev) cudaEventDestroy(ev);
  for (void* p : e->owned) cudaFree(p);
  delete e;
  return LA_OK;
}

// ------------------------------------------------------------- decode setup
struct DecodeArgs {
  int mode;
  int W, N, G, max_tokens, eos, seed_pool;
  const la_sampler* smp = nullptr;   // temperature sampler (null: greedy)
  bool greedy_verify = false;        // smp only carries the generator (greedy step session)
  bool pcg_window = false;           // window refills from the generator (step sessions)
};

// SamplerSpec.__post_init__ (types.py:59-67)
static int validate_sampler(const la_sampler* s) {
  if (!(s->temperature > 0.0)) { la_set_error("temperature must be positive"); return LA_ERR_INVALID_CONFIG; }
  if (s->top_k < 0) { la_set_error("top_k must be a positive integer"); return LA_ERR_INVALID_CONFIG; }
  if (!(s->top_p > 0.0 && s->top_p <= 1.0)) { la_set_error("top_p must lie in (0, 1]"); return LA_ERR_INVALID_CONFIG; }
  return LA_OK;
}

static LaPcg64 pcg_of(const la_sampler* s) {
  LaPcg64 g;
  g.s_hi = s->state_hi; g.s_lo = s->state_lo; g.i_hi = s->inc_hi; g.i_lo = s->inc_lo;
  g.has32 = s->has_uint32 ? 1 : 0; g.u32 = s->uinteger;
  return g;
}

// sampler buffers: logits of every step row, adjusted rows, working row
static int sampler_buffers(la_engine* e, int adj_rows) {
  const size_t V = (size_t)e->desc.vocab;
  RET_IF(dgrow(e, &e->d_logits, &e->logits_cap, (size_t)LA_MAX_ROWS * V));
  RET_IF(dgrow(e, &e->d_adj, &e->adj_cap, (size_t)adj_rows * V));
  RET_IF(dgrow(e, &e->d_work, &e->work_cap, V));
  RET_IF(dgrow(e, &e->d_flag, &e->flag_cap, (size_t)LA_MAX_ROWS));
  return LA_OK;
}

static int validate_gen(const la_engine* e, const DecodeArgs& a, const la_decode_io* io) {
  if (!io || !io->prompt || io->n_prompt < 1) { la_set_error("prompt must be nonempty"); return LA_ERR_INVALID_CONFIG; }
  if (a.max_tokens < 1) { la_set_error("max_tokens must be positive"); return LA_ERR_INVALID_CONFIG; }
  for (int i = 0; i < io->n_prompt; ++i)
    if (io->prompt[i] < 0 || io->prompt[i] >= e->desc.vocab) {
      la_set_error("token %d outside vocabulary of size %d", io->prompt[i], e->desc.vocab);
      return LA_ERR_INVALID_CONFIG;
    }
  if (a.mode == LA_MODE_LOOKAHEAD) {
    if (a.W < 1) { la_set_error("window size W must be >= 1"); return LA_ERR_INVALID_CONFIG; }
    if (a.N < 2) { la_set_error("n-gram size N must be >= 2"); return LA_ERR_INVALID_CONFIG; }
    if (a.G < 0) { la_set_error("max candidate count G must be >= 0"); return LA_ERR_INVALID_CONFIG; }
    if (a.W > 64 || a.N > LA_MAX_NGRAM || a.G > 64 || (a.N - 1) * (a.W + a.G) > LA_MAX_ROWS) {
      la_set_error("device limits: W <= 64, N <= %d, G <= 64, (N-1)(W+G) <= %d", LA_MAX_NGRAM, LA_MAX_ROWS);
      return LA_ERR_UNSUPPORTED;
    }
    if (a.W + a.N - 2 >= LA_MAX_CHAIN) { la_set_error("chain too long"); return LA_ERR_UNSUPPORTED; }
  }
  if (a.smp && !a.greedy_verify) {
    RET_IF(validate_sampler(a.smp));
    if (e->world > 1) {
      la_set_error("lookahead parallelism exchanges argmax ids only: temperature sampling is single-replica");
      return LA_ERR_UNSUPPORTED;
    }
  }
  long need = (long)io->n_prompt + a.max_tokens + LA_MAX_NGRAM;
  if (need > e->desc.max_context) {
    la_set_error("prompt + max_tokens (%ld) exceeds the engine's max_context %d", need,
                 e->desc.max_context);
    return LA_ERR_CAPACITY;
  }
  if (io->out_tokens && io->out_cap < a.max_tokens) {
    la_set_error("out_cap %d < max_tokens %d", io->out_cap, a.max_tokens);
    return LA_ERR_INVALID_CONFIG;
  }
  return LA_OK;
}

// Size/reset the pool, upload prompt + RNG stream + seeding n-grams, and
// initialise the device DevDecode (start_session, decoding.py:67-93).
static int setup_decode(la_engine* e, const DecodeArgs& a, const la_decode_io* io,
                        cudaStream_t st) {
  const int V = e->desc.vocab;
  const int N = a.mode == LA_MODE_LOOKAHEAD ? a.N : 2;
  const int W = a.mode == LA_MODE_LOOKAHEAD ? a.W : 1;
  const int ncell = a.mode == LA_MODE_LOOKAHEAD ? (N - 1) * W - 1 : 0;
  const int max_steps = a.max_tokens;
  // --- pool sizing
  long n_seed = 0;
  if (a.mode == LA_MODE_LOOKAHEAD && a.seed_pool) n_seed = std::max(0, io->n_prompt - N + 1);
  long n_init = (a.mode == LA_MODE_LOOKAHEAD && io->pool_init) ? io->pool_init_n : 0;
  long inserts = n_init + n_seed + (long)max_steps * W + 1;
  size_t LT = pow2_at_least(2 * std::min<long>(V, inserts) + 2);
  size_t ST = pow2_at_least(2 * inserts + 2);
  // LRU cap (pool.py:41-61): only a cap the decode can reach changes anything;
  // the capped pool keeps each lead's live entries in a linked list over the
  // distinct-set slots (O(LT + ST) memory for any capacity)
  int cap = (a.mode == LA_MODE_LOOKAHEAD && io->pool_capacity > 0 && io->pool_capacity < inserts)
                ? io->pool_capacity : 0;
  if (io->pool_capacity < 0) { la_set_error("capacity must be a positive integer"); return LA_ERR_INVALID_CONFIG; }
  size_t C = std::max(1, a.G);
  size_t logc = (size_t)inserts + 1;
  if (!e->p_lead || LT > e->p_lt || ST > e->p_st || C > e->p_C || logc > e->p_log_cap) {
    for (int* p : {e->p_lead, e->p_cnt, e->p_suf, e->p_set, e->p_counters, e->p_log, e->p_stamp,
                   e->p_fifo, e->p_head, e->p_prev, e->p_next}) {
      if (!p) continue;
      auto it = std::find(e->owned.begin(), e->owned.end(), (void*)p);
      if (it != e->owned.end()) e->owned.erase(it);
      CK(cudaFree(p));
    }
    LT = std::max(LT, e->p_lt); ST = std::max(ST, e->p_st);
    C = std::max(C, e->p_C); logc = std::max(logc, e->p_log_cap);
    RET_IF(dalloc(e, &e->p_lead, LT));
    RET_IF(dalloc(e, &e->p_cnt, LT));
    RET_IF(dalloc(e, &e->p_suf, LT * C * (LA_MAX_NGRAM - 1)));
    RET_IF(dalloc(e, &e->p_set, ST * LA_MAX_NGRAM));
    RET_IF(dalloc(e, &e->p_counters, 4));
    RET_IF(dalloc(e, &e->p_log, logc * LA_MAX_NGRAM));
    RET_IF(dalloc(e, &e->p_stamp, ST));
    RET_IF(dalloc(e, &e->p_fifo, logc));
    RET_IF(dalloc(e, &e->p_head, LT));
    RET_IF(dalloc(e, &e->p_prev, ST));
    RET_IF(dalloc(e, &e->p_next, ST));
    e->p_lt = LT; e->p_st = ST; e->p_C = C; e->p_N = LA_MAX_NGRAM; e->p_log_cap = logc;
  }
  C = std::max(1, a.G);
  LT = e->p_lt; ST = e->p_st;
  CK(cudaMemsetAsync(e->p_lead, 0xff, LT * sizeof(int), st));
  CK(cudaMemsetAsync(e->p_cnt, 0, LT * sizeof(int), st));
  CK(cudaMemsetAsync(e->p_set, 0xff, ST * N * sizeof(int), st));
  CK(cudaMemsetAsync(e->p_counters, 0, 4 * sizeof(int), st));
  // --- RNG stream (window init + refills), prompt, seeding n-grams
  int rng_len = (a.mode == LA_MODE_LOOKAHEAD && io->rng_stream) ? io->rng_len : 0;
  if (a.mode == LA_MODE_LOOKAHEAD && rng_len < ncell) {
    la_set_error("rng stream has %d entries, the window needs %d", rng_len, ncell);
    return LA_ERR_INVALID_CONFIG;
  }
  RET_IF(dgrow(e, &e->d_rng, &e->rng_cap, std::max(rng_len, 1)));
  if (rng_len) CK(cudaMemcpyAsync(e->d_rng, io->rng_stream, (size_t)rng_len * 4, cudaMemcpyHostToDevice, st));
  RET_IF(dgrow(e, &e->d_tokens, &e->tokens_cap, io->n_prompt));
  CK(cudaMemcpyAsync(e->d_tokens, io->prompt, (size_t)io->n_prompt * 4, cudaMemcpyHostToDevice, st));
  if (ncell > 0) CK(cudaMemcpyAsync(e->d_window, io->rng_stream, (size_t)ncell * 4, cudaMemcpyHostToDevice, st));
  // host-built list: caller pool (oldest first), then prompt n-grams
  std::vector<int> grams;
  if (n_init) grams.insert(grams.end(), io->pool_init, io->pool_init + n_init * N);
  for (long i = 0; i < n_seed; ++i)
    grams.insert(grams.end(), io->prompt + i, io->prompt + i + N);
  if (!grams.empty()) {
    RET_IF(dgrow(e, &e->d_grams, &e->grams_cap, grams.size()));
    CK(cudaMemcpyAsync(e->d_grams, grams.data(), grams.size() * 4, cudaMemcpyHostToDevice, st));
  }
  // --- DevDecode
  DevDecode& d = e->h_dec;
  memset(&d, 0, sizeof(d));
  d.mode = a.mode; d.W = W; d.N = N; d.G = a.mode == LA_MODE_LOOKAHEAD ? a.G : 0;
  d.V = V; d.max_tokens = a.max_tokens; d.eos = a.eos;
  d.rank = e->rank; d.world = e->world; d.max_steps = max_steps;
  d.ctx = io->n_prompt - 1; d.last = io->prompt[io->n_prompt - 1];
  d.rng_cur = ncell; d.rng_len = rng_len; d.winner = -1;
  d.window = e->d_window; d.rng = e->d_rng; d.out = e->d_out; d.rec = e->d_rec;
  d.cand = e->d_cand; d.amax = e->d_amax; d.accepted = e->d_acc;
  d.pool.ngram = N; d.pool.C = (int)C; d.pool.lt_mask = (int)LT - 1; d.pool.st_mask = (int)ST - 1;
  d.pool.log_cap = (int)e->p_log_cap;
  d.pool.lead_keys = e->p_lead; d.pool.bkt_cnt = e->p_cnt; d.pool.bkt_suf = e->p_suf;
  d.pool.set_keys = e->p_set; d.pool.counters = e->p_counters; d.pool.log = e->p_log;
  d.pool.capacity = cap; d.pool.set_stamp = e->p_stamp; d.pool.fifo = e->p_fifo;
  d.pool.lead_head = e->p_head; d.pool.set_prev = e->p_prev; d.pool.set_next = e->p_next;
  if (a.smp) {
    d.pcg = pcg_of(a.smp);
    d.pcg_window = a.pcg_window ? 1 : 0;
  }
  if (a.smp && !a.greedy_verify) {
    RET_IF(sampler_buffers(e, a.mode == LA_MODE_LOOKAHEAD ? 1 + d.G * (N - 1) : 1));
    d.sample = 1;
    d.temperature = a.smp->temperature;
    d.top_k = a.smp->top_k;
    d.top_p = a.smp->top_p;
    d.pcg = pcg_of(a.smp);
    d.logits = e->d_logits; d.adj = e->d_adj; d.work = e->d_work;
  }
  CK(cudaMemcpyAsync(e->d_dec, &d, sizeof(d), cudaMemcpyHostToDevice, st));
  if (!grams.empty()) {
    la_pool_seed_kernel<<<1, 32, 0, st>>>(e->d_dec, e->d_grams, (int)(grams.size() / N), (int)n_init);
    CK(cudaGetLastError());
  }
  return LA_OK;
}

static int prefill(la_engine* e, int n, cudaStream_t st) {
  if (n <= 0) return LA_OK;
  if (e->is_tiny()) {
    la_tiny_prefill<<<1, TINY_THREADS, e->tiny_smem, st>>>(e->tm, e->ts, e->d_plan, e->d_tokens, n);
    CK(cudaGetLastError());
    return LA_OK;
  }
  return llama_prefill(e, e->d_tokens, n, st);
}

static int readback(la_engine* e, la_decode_io* io, cudaStream_t st) {
  DevDecode d;
  CK(cudaMemcpyAsync(&d, e->d_dec, sizeof(d), cudaMemcpyDeviceToHost, st));
  int counters[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(counters, e->p_counters, sizeof(counters), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (d.overflow) { la_set_error("device capacity exceeded (pool table, log or RNG stream)"); return LA_ERR_CAPACITY; }
  if (d.degenerate) { la_set_error("all probability mass truncated away (degenerate distribution)"); return LA_ERR_DEGENERATE; }
  if (!e->is_tiny() && llama_mega_error(e)) {
    la_set_error("persistent forward kernel: dependency wait timed out (engine state is invalid)");
    return LA_ERR_CUDA;
  }
  io->n_out = d.n_out;
  io->n_steps = d.n_steps;
  io->pool_log_n = counters[1];
  if (io->out_tokens && d.n_out > 0)
    CK(cudaMemcpyAsync(io->out_tokens, e->d_out, (size_t)std::min(d.n_out, io->out_cap) * 4,
                       cudaMemcpyDeviceToHost, st));
  if (io->step_records && d.n_steps > 0)
    CK(cudaMemcpyAsync(io->step_records, e->d_rec,
                       (size_t)std::min(d.n_steps, io->rec_cap) * 16, cudaMemcpyDeviceToHost, st));
  if (io->pool_log && counters[1] > 0)
    CK(cudaMemcpyAsync(io->pool_log, e->p_log,
                       (size_t)std::min(counters[1], io->pool_log_cap) * d.N * 4,
                       cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e->ev[0], e->ev[1]));
  io->prefill_ms = ms;
  CK(cudaEventElapsedTime(&ms, e->ev[1], e->ev[2]));
  io->decode_ms = ms;
  return LA_OK;
}

int lp_decode_loop(la_engine* e, cudaStream_t st, int* launches);

static int run_decode(la_engine* e, const DecodeArgs& a, la_decode_io* io, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(e->device));
  e->session = false;   // a whole decode reuses (and ends) any step session's state
  RET_IF(validate_gen(e, a, io));
  if (a.mode == LA_MODE_AUTOREGRESSIVE && e->world > 1) {
    la_set_error("autoregressive decode is single-replica");
    return LA_ERR_INVALID_CONFIG;
  }
  RET_IF(setup_decode(e, a, io, st));
  CK(cudaEventRecord(e->ev[0], st));
  RET_IF(prefill(e, io->n_prompt - 1, st));
  CK(cudaEventRecord(e->ev[1], st));
  int launches = 0;
  if (e->world > 1) {
    RET_IF(lp_decode_loop(e, st, &launches));
  } else if (e->is_tiny()) {
    static const bool tiny_prof = getenv("LA_TINY_PROF") != nullptr;
    if (tiny_prof) la_tiny_prof(true, nullptr);
    la_tiny_decode<<<1, TINY_THREADS, e->tiny_smem, st>>>(e->tm, e->ts, e->d_plan, e->d_dec,
                                       e->h_dec.sample ? e->d_logits : nullptr);
    CK(cudaGetLastError());
    launches = 1;
  } else {
    RET_IF(llama_decode_loop(e, st, &launches));
  }
  CK(cudaEventRecord(e->ev[2], st));
  io->launches = launches;
  RET_IF(readback(e, io, st));
  // graph-launched decodes report kernels per step (negative): scale by steps
  if (io->launches < 0) io->launches = -io->launches * io->n_steps;
  return LA_OK;
}

extern "C" int32_t la_decode_lookahead(la_engine* e, const la_gen_config* cfg, la_decode_io* io,
                                       void* stream) {
  if (!e || !cfg) { la_set_error("null engine or config"); return LA_ERR_INVALID_CONFIG; }
  DecodeArgs a{LA_MODE_LOOKAHEAD, cfg->window, cfg->ngram, cfg->max_candidates,
               cfg->max_tokens, cfg->eos_token < 0 ? -1 : cfg->eos_token,
               cfg->seed_pool_from_prompt};
  return run_decode(e, a, io, stream);
}

extern "C" int32_t la_decode_autoregressive(la_engine* e, int32_t max_tokens, int32_t eos_token,
                                            la_decode_io* io, void* stream) {
  if (!e) { la_set_error("null engine"); return LA_ERR_INVALID_CONFIG; }
  DecodeArgs a{LA_MODE_AUTOREGRESSIVE, 1, 2, 0, max_tokens, eos_token < 0 ? -1 : eos_token, 0};
  return run_decode(e, a, io, stream);
}

extern "C" int32_t la_decode_lookahead_sampled(la_engine* e, const la_gen_config* cfg,
                                               const la_sampler* s, la_decode_io* io, void* stream) {
  if (!e || !cfg || !s) { la_set_error("null engine, config or sampler"); return LA_ERR_INVALID_CONFIG; }
  DecodeArgs a{LA_MODE_LOOKAHEAD, cfg->window, cfg->ngram, cfg->max_candidates,
               cfg->max_tokens, cfg->eos_token < 0 ? -1 : cfg->eos_token,
               cfg->seed_pool_from_prompt, s};
  return run_decode(e, a, io, stream);
}

extern "C" int32_t la_decode_autoregressive_sampled(la_engine* e, int32_t max_tokens,
                                                    int32_t eos_token, const la_sampler* s,
                                                    la_decode_io* io, void* stream) {
  if (!e || !s) { la_set_error("null engine or sampler"); return LA_ERR_INVALID_CONFIG; }
  DecodeArgs a{LA_MODE_AUTOREGRESSIVE, 1, 2, 0, max_tokens, eos_token < 0 ? -1 : eos_token, 0, s};
  return run_decode(e, a, io, stream);
}

// ------------------------------------------------------------ step session
// start_session (decoding.py:67-93): pool reset + seeding, window from the
// caller's generator (io->rng_stream = window_init's (N-1)W-1 cells), the
// generator state after it in *s, prompt prefill.  The device never stops on
// its own (no EOS, the budget is the engine's context): the caller folds the
// steps' tokens (collect_output, decoding.py:214-232).
extern "C" int32_t la_session_start(la_engine* e, const la_gen_config* cfg, int32_t greedy,
                                    const la_sampler* s, la_decode_io* io, void* stream) {
  if (!e || !cfg || !s || !io) { la_set_error("null engine, config, sampler or io"); return LA_ERR_INVALID_CONFIG; }
  if (e->world > 1) { la_set_error("step sessions are single-replica"); return LA_ERR_UNSUPPORTED; }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(e->device));
  e->session = false;
  const int budget = e->desc.max_context - (io->n_prompt > 0 ? io->n_prompt : 0) - LA_MAX_NGRAM;
  if (budget < 1) { la_set_error("prompt does not fit the engine's max_context"); return LA_ERR_CAPACITY; }
  DecodeArgs a{LA_MODE_LOOKAHEAD, cfg->window, cfg->ngram, cfg->max_candidates,
               std::min(budget, e->rec_cap - 1), -1, cfg->seed_pool_from_prompt, s,
               greedy != 0, true};
  io->out_tokens = nullptr;
  io->step_records = nullptr;
  RET_IF(validate_gen(e, a, io));
  RET_IF(setup_decode(e, a, io, st));
  RET_IF(prefill(e, io->n_prompt - 1, st));
  CK(cudaMemcpyAsync(&e->sess, e->d_dec, sizeof(DevDecode), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  e->session = true;
  return LA_OK;
}

// lookahead_step (decoding.py:207-211): one step on the device, outcome read back
extern "C" int32_t la_session_step(la_engine* e, la_step_outcome* out, void* stream) {
  if (!e || !out) { la_set_error("null engine or outcome"); return LA_ERR_INVALID_CONFIG; }
  if (!e->session) { la_set_error("no active step session (la_session_start)"); return LA_ERR_INVALID_CONFIG; }
  const DevDecode& h = e->sess;
  if (h.done || h.ctx + h.N + 1 > e->desc.max_context) {
    la_set_error("session reached the engine's max_context (%d)", e->desc.max_context);
    return LA_ERR_CAPACITY;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(e->device));
  if (e->is_tiny()) {
    la_tiny_step_forward<<<1, TINY_THREADS, e->tiny_smem, st>>>(e->tm, e->ts, e->d_plan, e->d_dec,
                                             h.sample ? e->d_logits : nullptr);
    if (h.sample) {
      la_sample_adjust_kernel<<<1 + h.G * (h.N - 1), 1024, 0, st>>>(e->d_dec);
      la_sample_verify_kernel<<<1, 1024, 0, st>>>(e->d_dec);
    }
    la_step_finish_kernel<<<1, 256, 0, st>>>(e->d_dec);
    la_kv_commit_kernel<<<std::max(1, std::min(148, e->desc.layers * e->row_bytes / 16 / 256)), 256, 0, st>>>(
        e->d_dec, (uint8_t*)e->kc, (uint8_t*)e->vc, e->desc.layers, e->slots, e->row_bytes);
    CK(cudaGetLastError());
  } else {
    RET_IF(llama_session_step(e, st));
  }
  DevDecode d;
  int counters[4];
  CK(cudaMemcpyAsync(&d, e->d_dec, sizeof(d), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(counters, e->p_counters, sizeof(counters), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out->accepted, e->d_acc, sizeof(int32_t) * (LA_MAX_NGRAM + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out->new_top, e->d_amax + (h.N - 2) * h.W, sizeof(int32_t) * h.W,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (d.overflow) { la_set_error("device capacity exceeded (pool table or log)"); return LA_ERR_CAPACITY; }
  if (d.degenerate) { la_set_error("all probability mass truncated away (degenerate distribution)"); return LA_ERR_DEGENERATE; }
  if (!e->is_tiny() && llama_mega_error(e)) { la_set_error("persistent forward kernel: dependency wait timed out"); return LA_ERR_CUDA; }
  if (d.n_steps != h.n_steps + 1) { la_set_error("session step did not run"); return LA_ERR_CUDA; }
  e->sess = d;
  out->n_accepted = d.k;
  out->n_new_top = h.W;
  out->candidate_count = d.c;
  out->query_count = d.M;
  out->pool_size = counters[0];
  out->pool_log_n = counters[1];
  return LA_OK;
}

// session state readers: what 0 = window cells ((N-1)W-1), 1 = pool-log
// n-grams [offset, offset+n) (N ints each), 2 = the generator state (10 words)
extern "C" int32_t la_session_read(la_engine* e, int32_t what, int32_t offset, int32_t n,
                                   int32_t* out) {
  if (!e || !out || offset < 0 || n < 0) { la_set_error("bad arguments"); return LA_ERR_INVALID_CONFIG; }
  if (!e->session) { la_set_error("no active step session"); return LA_ERR_INVALID_CONFIG; }
  CK(cudaSetDevice(e->device));
  const DevDecode& h = e->sess;
  if (what == 0) {
    const int ncell = (h.N - 1) * h.W - 1;
    if (offset + n > ncell) { la_set_error("window has %d cells", ncell); return LA_ERR_INVALID_CONFIG; }
    if (n) CK(cudaMemcpy(out, e->d_window + offset, (size_t)n * 4, cudaMemcpyDeviceToHost));
    return LA_OK;
  }
  if (what == 1) {
    if ((size_t)(offset + n) > e->p_log_cap) { la_set_error("pool log holds %zu entries", e->p_log_cap); return LA_ERR_CAPACITY; }
    if (n) CK(cudaMemcpy(out, e->p_log + (size_t)offset * h.N, (size_t)n * h.N * 4, cudaMemcpyDeviceToHost));
    return LA_OK;
  }
  if (what == 2) {
    // the session generator (numpy PCG64: state, inc, has_uint32, uinteger) as
    // 10 words: state hi/lo, inc hi/lo (64-bit little-endian pairs), has32, u32
    if (offset != 0 || n != 10) { la_set_error("generator state is 10 words"); return LA_ERR_INVALID_CONFIG; }
    const unsigned long long q[4] = {h.pcg.s_hi, h.pcg.s_lo, h.pcg.i_hi, h.pcg.i_lo};
    for (int i = 0; i < 4; ++i) {
      out[2 * i] = (int32_t)(uint32_t)(q[i] & 0xffffffffull);
      out[2 * i + 1] = (int32_t)(uint32_t)(q[i] >> 32);
    }
    out[8] = h.pcg.has32;
    out[9] = (int32_t)h.pcg.u32;
    return LA_OK;
  }
  la_set_error("unknown session field %d", what);
  return LA_ERR_INVALID_CONFIG;
}

// ------------------------------------------------------------- pool hook
// Tests only: a fresh device pool (N, capacity; bucket size C) fed n_grams
// n-grams in batches of `batch` through the K10 insert path; after each batch
// lookup(lead, limit) of every lead and len(pool).  out[b][q][limit][N-1],
// counts[b][q], lens[b] (host).
extern "C" int32_t la_pool_test(int32_t N, int32_t capacity, int32_t C, const int32_t* grams,
                                int32_t n_grams, int32_t batch, const int32_t* leads, int32_t n_leads,
                                int32_t limit, int32_t* out, int32_t* counts, int32_t* lens) {
  if (N < 2 || N > LA_MAX_NGRAM || C < 1 || n_grams < 1 || batch < 1 || batch > 64 || n_leads < 1 ||
      limit < 1 || limit > C || capacity < 0 || !grams || !leads || !out || !counts || !lens) {
    la_set_error("bad arguments");
    return LA_ERR_INVALID_CONFIG;
  }
  const size_t LT = pow2_at_least(2 * (size_t)n_grams + 2), ST = LT;
  const int nb = (n_grams + batch - 1) / batch;
  const int Cb = C;
  std::vector<void*> bufs;
  auto dev = [&](size_t bytes, int fill) -> void* {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
    cudaMemset(q, fill, std::max<size_t>(bytes, 16));
    bufs.push_back(q);
    return q;
  };
  DevPool p{};
  p.ngram = N; p.C = Cb; p.lt_mask = (int)LT - 1; p.st_mask = (int)ST - 1;
  p.log_cap = n_grams + 1; p.capacity = capacity;
  p.lead_keys = (int*)dev(LT * 4, 0xff);
  p.bkt_cnt = (int*)dev(LT * 4, 0);
  p.bkt_suf = (int*)dev(LT * Cb * (N - 1) * 4, 0);
  p.set_keys = (int*)dev(ST * N * 4, 0xff);
  p.set_stamp = (int*)dev(ST * 4, 0);
  p.fifo = (int*)dev((size_t)p.log_cap * 4, 0);
  p.lead_head = (int*)dev(LT * 4, 0xff);
  p.set_prev = (int*)dev(ST * 4, 0xff);
  p.set_next = (int*)dev(ST * 4, 0xff);
  p.counters = (int*)dev(16, 0);
  p.log = (int*)dev((size_t)p.log_cap * N * 4, 0);
  int* d_grams = (int*)dev((size_t)n_grams * N * 4, 0);
  int* d_leads = (int*)dev((size_t)n_leads * 4, 0);
  int* d_out = (int*)dev((size_t)nb * n_leads * limit * (N - 1) * 4, 0);
  int* d_counts = (int*)dev((size_t)nb * n_leads * 4, 0);
  int* d_lens = (int*)dev((size_t)nb * 4, 0);
  int* d_ovf = (int*)dev(16, 0);
  int rc = LA_OK;
  for (void* q : bufs)
    if (!q) rc = LA_ERR_CUDA;
  int ovf = 0;
  if (rc == LA_OK) {
    cudaMemcpy(d_grams, grams, (size_t)n_grams * N * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_leads, leads, (size_t)n_leads * 4, cudaMemcpyHostToDevice);
    la_pool_test_kernel<<<1, 256>>>(p, d_grams, n_grams, batch, d_leads, n_leads, limit, d_out,
                                    d_counts, d_lens, d_ovf);
    cudaError_t ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) { la_set_error("pool test: %s", cudaGetErrorString(ce)); rc = LA_ERR_CUDA; }
    else {
      cudaMemcpy(out, d_out, (size_t)nb * n_leads * limit * (N - 1) * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(counts, d_counts, (size_t)nb * n_leads * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(lens, d_lens, (size_t)nb * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(&ovf, d_ovf, 4, cudaMemcpyDeviceToHost);
    }
  }
  for (void* q : bufs) if (q) cudaFree(q);
  if (rc == LA_OK && ovf) { la_set_error("pool overflow"); rc = LA_ERR_CAPACITY; }
  return rc;
}

// ---------------------------------------------------------- sampler hooks
extern "C" int32_t la_adjust_distributions(la_engine* e, const double* probs, int32_t n_rows,
                                           int32_t V, const la_sampler* s, double* out,
                                           void* stream) {
  if (!e || !probs || !out || !s || n_rows < 1 || V < 1) { la_set_error("bad arguments"); return LA_ERR_INVALID_CONFIG; }
  RET_IF(validate_sampler(s));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(e->device));
  RET_IF(dgrow(e, &e->d_adj, &e->adj_cap, (size_t)n_rows * V));
  RET_IF(dgrow(e, &e->d_flag, &e->flag_cap, (size_t)n_rows));
  CK(cudaMemcpyAsync(e->d_adj, probs, (size_t)n_rows * V * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(e->d_flag, 0, (size_t)n_rows * 4, st));
  // LA_ADJ_HOOK_CLUSTER=1: the bf16 path's cluster-scope kernel instead of one CTA per row
  if (getenv("LA_ADJ_HOOK_CLUSTER") && atoi(getenv("LA_ADJ_HOOK_CLUSTER")) == 1)
    la_adjust_probs_cluster_kernel<<<n_rows * LA_ADJ_CLUSTER, LA_ADJ_THREADS, 0, st>>>(
        e->d_adj, V, s->temperature, s->top_k, s->top_p, e->d_flag);
  else
    la_adjust_probs_kernel<<<n_rows, 1024, 0, st>>>(e->d_adj, V, s->temperature, s->top_k, s->top_p,
                                                    e->d_flag);
  CK(cudaGetLastError());
  std::vector<int> flags(n_rows);
  CK(cudaMemcpyAsync(out, e->d_adj, (size_t)n_rows * V * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(flags.data(), e->d_flag, (size_t)n_rows * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int f : flags)
    if (f) { la_set_error("all probability mass truncated away"); return LA_ERR_DEGENERATE; }
  return LA_OK;
}

extern "C" int32_t la_verify_sample_dists(la_engine* e, const double* dists, int32_t V, int32_t S,
                                          int32_t c, const int32_t* suffixes, const la_sampler* s,
                                          int32_t* out, int32_t* n_out, void* stream) {
  if (!e || !dists || !s || !out || !n_out || V < 1 || S < 1 || S > LA_MAX_SUFFIX || c < 0 ||
      c > 32 || (c > 0 && !suffixes)) {
    la_set_error("bad arguments (S <= %d, c <= 32)", LA_MAX_SUFFIX);
    return LA_ERR_INVALID_CONFIG;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(e->device));
  const size_t rows = 1 + (size_t)c * S;
  RET_IF(dgrow(e, &e->d_adj, &e->adj_cap, rows * V));
  RET_IF(dgrow(e, &e->d_work, &e->work_cap, (size_t)V));
  CK(cudaMemcpyAsync(e->d_adj, dists, rows * V * 8, cudaMemcpyHostToDevice, st));
  if (c) CK(cudaMemcpyAsync(e->d_cand, suffixes, (size_t)c * S * 4, cudaMemcpyHostToDevice, st));
  DevDecode d;
  memset(&d, 0, sizeof(d));
  d.mode = LA_MODE_LOOKAHEAD; d.N = S + 1; d.W = 1; d.V = V; d.c = c;
  d.cand = e->d_cand; d.accepted = e->d_acc; d.adj = e->d_adj; d.work = e->d_work;
  d.sample = 1; d.pcg = pcg_of(s); d.winner = -1;
  CK(cudaMemcpyAsync(e->d_dec, &d, sizeof(d), cudaMemcpyHostToDevice, st));
  la_verify_hook_kernel<<<1, 1024, 0, st>>>(e->d_dec);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&d, e->d_dec, sizeof(d), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (d.degenerate) { la_set_error("verification renormalized to zero mass"); return LA_ERR_DEGENERATE; }
  CK(cudaMemcpy(out, e->d_acc, (size_t)d.k * 4, cudaMemcpyDeviceToHost));
  *n_out = d.k;
  return LA_OK;
}

extern "C" int32_t la_pcg64_draws(const la_sampler* s, int32_t kind, int32_t high, int32_t n,
                                  double* out) {
  if (!s || !out || n < 0 || (kind == 1 && high < 1)) { la_set_error("bad arguments"); return LA_ERR_INVALID_CONFIG; }
  LaPcg64 g = pcg_of(s);
  for (int i = 0; i < n; ++i)
    out[i] = kind == 0 ? la_pcg_random(g) : (double)la_pcg_integers(g, (unsigned)high);
  return LA_OK;
}

// ------------------------------------------------------------- parity hook
// Validate a query layout (models.py:33-64 contract: row 0 at rel 0; row i
// sees one row per rel 0..rel[i]-1, listed in rel order) and build its plan.
static int build_layout_plan(la_engine* e, int n_prefix, int n_rows, const int32_t* ids, const int32_t* rel,
                             const int32_t* chain, int chain_stride, FwdPlan* P) {
  const int V = e->desc.vocab;
  if (n_rows < 1 || n_rows > LA_MAX_ROWS) { la_set_error("n_rows must be in [1, %d]", LA_MAX_ROWS); return LA_ERR_UNSUPPORTED; }
  if (n_prefix < 0 || n_prefix + n_rows + 1 > e->desc.max_context) { la_set_error("prefix too long"); return LA_ERR_CAPACITY; }
  for (int i = 0; i < n_rows; ++i)
    if (ids[i] < 0 || ids[i] >= V) { la_set_error("token %d outside vocabulary of size %d", ids[i], V); return LA_ERR_INVALID_CONFIG; }
  if (rel[0] != 0) { la_set_error("query 0 must sit at relative position 0"); return LA_ERR_LAYOUT; }
  memset(P, 0, sizeof(FwdPlan));
  P->n_rows = n_rows; P->n_pad = (n_rows + 15) & ~15; P->n_prefix = n_prefix; P->n_global = n_rows;
  P->want_logits = 1;
  for (int i = 0; i < n_rows; ++i) {
    if (rel[i] < 0 || rel[i] >= LA_MAX_CHAIN) { la_set_error("rel_pos out of range"); return LA_ERR_LAYOUT; }
    P->ids[i] = ids[i];
    P->pos[i] = n_prefix + rel[i];
    P->slot[i] = n_prefix + i;
    P->grow[i] = i;
    P->own[i] = 1;
    P->chain_n[i] = rel[i];
    for (int j = 0; j < rel[i]; ++j) {
      int v = chain[(size_t)i * chain_stride + j];
      if (v < 0 || v >= n_rows || v == i || rel[v] != j) {
        la_set_error("query %d has an invalid chain entry %d at rel_pos %d", i, v, j);
        return LA_ERR_LAYOUT;
      }
      P->chain[i][j] = n_prefix + v;
    }
  }
  return LA_OK;
}

static int prefill_prefix(la_engine* e, const int32_t* prefix, int n_prefix, cudaStream_t st) {
  const int V = e->desc.vocab;
  for (int i = 0; i < n_prefix; ++i)
    if (prefix[i] < 0 || prefix[i] >= V) { la_set_error("token %d outside vocabulary of size %d", prefix[i], V); return LA_ERR_INVALID_CONFIG; }
  if (n_prefix == 0) return LA_OK;
  int rc = dgrow(e, &e->d_tokens, &e->tokens_cap, n_prefix);
  if (rc) return rc;
  CK(cudaMemcpyAsync(e->d_tokens, prefix, (size_t)n_prefix * 4, cudaMemcpyHostToDevice, st));
  return prefill(e, n_prefix, st);
}

// one forward of an uploaded plan: logits[n_rows][V] to host (if non-null)
// and/or the per-row greedy argmax (ties -> lowest id) to host
static int run_plan(la_engine* e, const FwdPlan* P, float* logits, int32_t* amax, cudaStream_t st) {
  const int V = e->desc.vocab, n_rows = P->n_rows;
  CK(cudaMemcpyAsync(e->d_plan, P, sizeof(FwdPlan), cudaMemcpyHostToDevice, st));
  float* d_logits = nullptr;
  const bool need_logits = logits != nullptr || e->is_tiny();
  if (need_logits && cudaMallocAsync(&d_logits, (size_t)n_rows * V * 4, st) != cudaSuccess) {
    la_set_error("cudaMallocAsync failed");
    return LA_ERR_CUDA;
  }
  int rc = LA_OK;
  std::vector<float> host;
  if (e->is_tiny()) {
    la_tiny_forward<<<1, TINY_THREADS, e->tiny_smem, st>>>(e->tm, e->ts, e->d_plan, d_logits);
    if (cudaGetLastError() != cudaSuccess) { la_set_error("forward launch failed"); rc = LA_ERR_CUDA; }
  } else {
    rc = llama_forward_plan(e, d_logits, st);
  }
  if (rc == LA_OK) {
    cudaError_t ce = cudaSuccess;
    float* lg = logits;
    if (e->is_tiny() && !lg) { host.resize((size_t)n_rows * V); lg = host.data(); }
    if (lg) ce = cudaMemcpyAsync(lg, d_logits, (size_t)n_rows * V * 4, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess && amax && !e->is_tiny()) ce = llama_copy_argmax(e, amax, n_rows, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) { la_set_error("forward failed: %s", cudaGetErrorString(ce)); rc = LA_ERR_CUDA; }
    if (rc == LA_OK && amax && e->is_tiny())
      for (int r = 0; r < n_rows; ++r) {   // np.argmax semantics: first maximum
        const float* row = lg + (size_t)r * V;
        int best = 0;
        for (int v = 1; v < V; ++v)
          if (row[v] > row[best]) best = v;
        amax[r] = best;
      }
  }
  if (d_logits) cudaFreeAsync(d_logits, st);
  return rc;
}

extern "C" int32_t la_forward_layout(la_engine* e, const int32_t* prefix, int32_t n_prefix,
                                     int32_t n_rows, const int32_t* ids, const int32_t* rel,
                                     const int32_t* chain, int32_t chain_stride, float* logits,
                                     void* stream) {
  if (!e) { la_set_error("null engine"); return LA_ERR_INVALID_CONFIG; }
  e->session = false;   // the parity forward reuses the plan and KV cache
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(e->device));
  FwdPlan* P = new FwdPlan();
  int rc = build_layout_plan(e, n_prefix, n_rows, ids, rel, chain, chain_stride, P);
  if (rc == LA_OK) rc = prefill_prefix(e, prefix, n_prefix, st);
  if (rc == LA_OK) rc = run_plan(e, P, logits, nullptr, st);
  delete P;
  return rc;
}

// Jacobi decoding (decoding.py:119-149): m-token greedy continuation by
// parallel fixed-point iteration over the triangular chain layout
// (layout.py:185-194); the prompt is prefilled once, every iteration is one
// forward of m+1 rows whose per-row argmax (device) is the next iterate.
extern "C" int32_t la_decode_jacobi(la_engine* e, const int32_t* prompt, int32_t n_prompt, int32_t m,
                                    const int32_t* init, int32_t* out_tokens, int32_t* iterates,
                                    int32_t* n_iterations, void* stream) {
  if (!e || !prompt || !init || !out_tokens || !n_iterations) { la_set_error("null argument"); return LA_ERR_INVALID_CONFIG; }
  e->session = false;
  if (n_prompt < 1) { la_set_error("prompt must be nonempty"); return LA_ERR_INVALID_CONFIG; }
  if (m < 1) { la_set_error("generation length m must be >= 1"); return LA_ERR_INVALID_CONFIG; }
  if (m + 1 > LA_MAX_ROWS) { la_set_error("m + 1 must be <= %d rows", LA_MAX_ROWS); return LA_ERR_UNSUPPORTED; }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(e->device));
  const int V = e->desc.vocab;
  for (int i = 0; i < m; ++i)
    if (init[i] < 0 || init[i] >= V) { la_set_error("token %d outside vocabulary of size %d", init[i], V); return LA_ERR_INVALID_CONFIG; }
  const int n_prefix = n_prompt - 1;
  int rc = prefill_prefix(e, prompt, n_prefix, st);
  if (rc) return rc;
  std::vector<int32_t> ids(m + 1), rel(m + 1), chain((size_t)(m + 1) * (m + 1), 0), cur(init, init + m),
      amax(m + 1);
  for (int i = 0; i <= m; ++i) {
    rel[i] = i;
    for (int j = 0; j < i; ++j) chain[(size_t)i * (m + 1) + j] = j;
  }
  ids[0] = prompt[n_prompt - 1];
  FwdPlan* P = new FwdPlan();
  int it = 0;
  for (; it < m; ++it) {
    for (int i = 0; i < m; ++i) ids[i + 1] = cur[i];
    if ((rc = build_layout_plan(e, n_prefix, m + 1, ids.data(), rel.data(), chain.data(), m + 1, P))) break;
    if ((rc = run_plan(e, P, nullptr, amax.data(), st))) break;
    if (iterates) memcpy(iterates + (size_t)it * m, amax.data(), (size_t)m * 4);
    const bool same = std::equal(cur.begin(), cur.end(), amax.begin());
    std::copy(amax.begin(), amax.begin() + m, cur.begin());
    if (same) { ++it; break; }
  }
  delete P;
  if (rc) return rc;
  memcpy(out_tokens, cur.data(), (size_t)m * 4);
  *n_iterations = it;
  return LA_OK;
}

// ------------------------------------------------- in-process LP group
int lp_buffers(la_engine* e, int world);
int lp_group_loop(la_engine* const* es, int n, cudaStream_t st, int* launches);

extern "C" int32_t la_decode_lookahead_group(la_engine* const* es, int32_t n,
                                             const la_gen_config* cfg, la_decode_io* io,
                                             void* stream) {
  if (!es || n < 1 || !cfg) { la_set_error("need >= 1 engine and a config"); return LA_ERR_INVALID_CONFIG; }
  for (int r = 0; r < n; ++r)
    if (es[r]) es[r]->session = false;
  if (n > cfg->window) {
    la_set_error("device count must lie in [1, %d], got %d", cfg->window, n);
    return LA_ERR_INVALID_CONFIG;
  }
  for (int r = 0; r < n; ++r)
    if (!es[r] || es[r]->device != es[0]->device || es[r]->desc.arch != es[0]->desc.arch ||
        es[r]->desc.vocab != es[0]->desc.vocab) {
      la_set_error("group engines must share device and model");
      return LA_ERR_INVALID_CONFIG;
    }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(es[0]->device));
  DecodeArgs a{LA_MODE_LOOKAHEAD, cfg->window, cfg->ngram, cfg->max_candidates,
               cfg->max_tokens, cfg->eos_token < 0 ? -1 : cfg->eos_token,
               cfg->seed_pool_from_prompt};
  RET_IF(validate_gen(es[0], a, io));
  int rc = LA_OK;
  for (int r = 0; r < n && rc == LA_OK; ++r) {
    es[r]->rank = r;
    es[r]->world = n;
    rc = lp_buffers(es[r], n);
    if (rc == LA_OK) rc = setup_decode(es[r], a, io, st);
  }
  if (rc == LA_OK) {
    cudaEventRecord(es[0]->ev[0], st);
    for (int r = 0; r < n && rc == LA_OK; ++r) rc = prefill(es[r], io->n_prompt - 1, st);
    cudaEventRecord(es[0]->ev[1], st);
  }
  int launches = 0;
  if (rc == LA_OK) rc = lp_group_loop(es, n, st, &launches);
  if (rc == LA_OK) {
    cudaEventRecord(es[0]->ev[2], st);
    io->launches = launches;
    rc = readback(es[0], io, st);
  }
  for (int r = 0; r < n; ++r) { es[r]->rank = 0; es[r]->world = 1; }
  return rc;
}

int llama_read_trace(la_engine* e, void* host, size_t bytes);
bool llama_debug_buffer(la_engine* e, int what, const void** src, size_t* bytes);

// ------------------------------------------------------------ debug copy
extern void* g_attn_trace_host;
extern "C" int32_t la_debug_read(la_engine* e, int32_t what, void* host, int64_t bytes) {
  if (!e || !host) { la_set_error("null engine or buffer"); return LA_ERR_INVALID_CONFIG; }
  if (what == 19) {   // host address of the mapped attention trace (no device sync: usable on a hang)
    *reinterpret_cast<void**>(host) = g_attn_trace_host;
    return LA_OK;
  }
  CK(cudaSetDevice(e->device));
  CK(cudaDeviceSynchronize());
  const void* src = nullptr;
  size_t avail = 0;
  const size_t kv = (size_t)e->desc.layers * e->slots * e->row_bytes;
  switch (what) {
    case 0: src = e->d_amax; avail = LA_MAX_ROWS * sizeof(int); break;
    case 1: src = e->kc; avail = kv; break;
    case 2: src = e->vc; avail = kv; break;
    case 3: src = e->d_dec; avail = sizeof(DevDecode); break;
    case 4: src = e->d_plan; avail = sizeof(FwdPlan); break;
    case 5: return llama_read_trace(e, host, (size_t)bytes);
    case 21: {   // la_tiny_decode per-phase cycles (LA_TINY_PROF=1)
      unsigned long long t[16];
      if (la_tiny_prof(false, t) != 0) { la_set_error("tiny profile read failed"); return LA_ERR_CUDA; }
      memcpy(host, t, std::min<size_t>(sizeof(t), (size_t)bytes));
      return LA_OK;
    }
    default:
      if (what >= 6 && !e->is_tiny() && llama_debug_buffer(e, what, &src, &avail)) break; la_set_error("unknown debug buffer %d", what); return LA_ERR_INVALID_CONFIG;
  }
  CK(cudaMemcpy(host, src, std::min<size_t>(avail, (size_t)bytes), cudaMemcpyDeviceToHost));
  return LA_OK;
}
