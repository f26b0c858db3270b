// fp32 SIMT single-CTA decode megakernel for tiny models.
//
// BASELINE config 1 is the reference's own TinyTransformer (models.py:189-271,
// d=16, L=2, H=2): every op is a few hundred FLOPs, so the whole decode --
// prefill, every lookahead step (K1 build, forward, argmax, K10 finish, KV
// commit) -- runs inside ONE persistent CTA with __syncthreads between phases.
// No launch per step, no host round trip.  fp32 FFMA only (no TF32): the
// reference is float64 and greedy parity needs ~1e-7 relative logit error
// (SURVEY.md §2.4).  The same kernel also serves a tiny Llama-style decoder
// (RMSNorm, rotate-half RoPE, SwiGLU, GQA) used to pin the Llama math.
#include "la_state.cuh"
#include "la_tiny.h"

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (value, index) argmax, ties -> lowest index (sampling.py:17-19)
__device__ __forceinline__ void argmax_merge(float& v, int& i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

// row-wise norm: GPT LayerNorm (population variance, models.py:183-186) or RMSNorm
__device__ void norm_rows(const TinyModel& m, const float* x, float* h, int R, const float* g,
                          const float* b) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int d = m.d;
  for (int r = warp; r < R; r += nw) {
    const float* xr = x + (size_t)r * d;
    float* hr = h + (size_t)r * d;
    if (m.arch == TINY_ARCH_GPT) {
      float sum = 0.f;
      for (int i = lane; i < d; i += 32) sum += xr[i];
      float mean = warp_sum(sum) / d;
      float sq = 0.f;
      for (int i = lane; i < d; i += 32) { float t = xr[i] - mean; sq += t * t; }
      float var = warp_sum(sq) / d;
      float inv = 1.0f / sqrtf(var + 1e-8f);
      for (int i = lane; i < d; i += 32) hr[i] = (xr[i] - mean) * inv * g[i] + b[i];
    } else {
      float sq = 0.f;
      for (int i = lane; i < d; i += 32) sq += xr[i] * xr[i];
      float inv = 1.0f / sqrtf(warp_sum(sq) / d + m.eps);
      for (int i = lane; i < d; i += 32) hr[i] = xr[i] * inv * g[i];
    }
  }
}

// out[r][o] (+)= sum_i in[r][i] * W[o][i]  (+ bias), W given transposed (WT[i][o])
__device__ void gemv_rows(const float* in, int in_ld, const float* WT, const float* bias, float* out,
                          int out_ld, int R, int n_out, int n_in, bool accumulate) {
  for (int idx = threadIdx.x; idx < R * n_out; idx += blockDim.x) {
    int r = idx / n_out, o = idx % n_out;
    const float* a = in + (size_t)r * in_ld;
    const float* w = WT + o;
    float acc = 0.f;
    for (int i = 0; i < n_in; ++i) acc = fmaf(a[i], w[(size_t)i * n_out], acc);
    if (bias) acc += bias[o];
    float* dst = out + (size_t)r * out_ld + o;
    *dst = accumulate ? (*dst + acc) : acc;
  }
}

// Optional per-phase cycle accounting of la_tiny_decode (LA_TINY_PROF=1,
// profiling only; read with la_debug_read(engine, 21, ...)): [0] K1 build,
// [1] forward, [2] argmax scatter, [3] sampler, [4] K10 finish, [5] KV commit,
// [6] steps
__device__ unsigned long long g_tiny_prof[16];
__device__ int g_tiny_prof_on;

__device__ __forceinline__ long long tiny_clock() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

struct TinyProf {
  bool on;
  long long t;
  __device__ TinyProf() : on(g_tiny_prof_on != 0), t(on ? tiny_clock() : 0) {}
  __device__ void mark(int k) {
    if (!on) return;
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long n = tiny_clock();
      g_tiny_prof[k] += (unsigned long long)(n - t);
      t = n;
    }
  }
};


// Attention of R rows, one warp per (row, head).  Lane-parallel online
// softmax: lane t takes keys t, t+32, ... of the row's key list (prefix slots,
// chain slots in relative-position order, self) keeping a running max / sum /
// weighted V in registers (no score buffer), then the 32 lane states combine
// in a fixed butterfly order.  A row's arithmetic depends only on its own key
// list, so lookahead rows compute exactly what the greedy rows do.  HD >= hd
// bounds the register arrays (TINY_THREADS threads: 65536 / TINY_THREADS registers each).
template <int HD>
__device__ void attn_rows(const TinyModel& m, const TinyScratch& s, const FwdPlan& P, const float* kc,
                          const float* vc, int R) {
  const int H = m.H, KVH = m.KVH, hd = m.hd, qd = H * hd, kvd = KVH * hd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const float scale = 1.0f / sqrtf((float)hd);
  const bool vec = (hd & 3) == 0;
  for (int job = warp; job < R * H; job += nw) {
    const int r = job / H, hh = job % H, kvh = hh / (H / KVH);
    const float* q = s.q + (size_t)r * qd + hh * hd;
    const int npre = P.n_prefix, nch = P.chain_n[r];
    const int nk = npre + nch + 1, self = P.slot[r];
    float qr[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) qr[i] = i < hd ? q[i] : 0.f;
    float mx = -INFINITY, sum = 0.f, o[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) o[i] = 0.f;
    // (K / V through L1: the prefix rows stay cached across steps; this
    // CTA's own stores keep its L1 coherent)
    for (int j = lane; j < nk; j += 32) {
      const int slot = (j < npre) ? j : (j < npre + nch ? P.chain[r][j - npre] : self);
      const float* kk = kc + (size_t)slot * kvd + kvh * hd;
      const float* vv = vc + (size_t)slot * kvd + kvh * hd;
      float kr[HD], vr[HD];   // the key's and value's rows in flight together
      if (vec) {
#pragma unroll
        for (int i4 = 0; i4 < HD / 4; ++i4)
          if (4 * i4 < hd) {
            const float4 a = reinterpret_cast<const float4*>(kk)[i4];
            const float4 b = reinterpret_cast<const float4*>(vv)[i4];
            kr[4 * i4] = a.x; kr[4 * i4 + 1] = a.y; kr[4 * i4 + 2] = a.z; kr[4 * i4 + 3] = a.w;
            vr[4 * i4] = b.x; vr[4 * i4 + 1] = b.y; vr[4 * i4 + 2] = b.z; vr[4 * i4 + 3] = b.w;
          }
      } else {
#pragma unroll
        for (int i = 0; i < HD; ++i)
          if (i < hd) { kr[i] = kk[i]; vr[i] = vv[i]; }
      }
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < HD; ++i)
        if (i < hd) dot = fmaf(qr[i], kr[i], dot);
      dot *= scale;
      if (dot > mx) {
        const float a = expf(mx - dot);   // 0 on the lane's first key (mx = -inf)
        sum *= a;
#pragma unroll
        for (int i = 0; i < HD; ++i) o[i] *= a;
        mx = dot;
      }
      const float e = expf(dot - mx);
      sum += e;
#pragma unroll
      for (int i = 0; i < HD; ++i)
        if (i < hd) o[i] = fmaf(e, vr[i], o[i]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, mx, off);
      const float s2 = __shfl_xor_sync(0xffffffffu, sum, off);
      const float mn = fmaxf(mx, m2);
      const float a = mx == -INFINITY ? 0.f : expf(mx - mn);
      const float b = m2 == -INFINITY ? 0.f : expf(m2 - mn);
      sum = sum * a + s2 * b;
#pragma unroll
      for (int i = 0; i < HD; ++i) {
        const float o2 = __shfl_xor_sync(0xffffffffu, o[i], off);
        o[i] = o[i] * a + o2 * b;
      }
      mx = mn;
    }
    const float inv = 1.0f / sum;
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < HD; ++i)
      if (i == lane) v = o[i];
    if (lane < hd) s.att[(size_t)r * qd + hh * hd + lane] = v * inv;
  }
}

__device__ void forward_rows(const TinyModel& m, const TinyScratch& s, const FwdPlan& P,
                             float* logits_out, TinyProf* pf = nullptr) {
  auto mark = [&](int k) { if (pf) pf->mark(k); };
  const int R = P.n_rows;
  const int d = m.d, H = m.H, KVH = m.KVH, hd = m.hd;
  const int qd = H * hd, kvd = KVH * hd;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nth >> 5;
  // embedding (+ sinusoidal absolute positions for the GPT model, models.py:245-247)
  for (int idx = tid; idx < R * d; idx += nth) {
    int r = idx / d, i = idx % d;
    float v = m.embed[(size_t)P.ids[r] * d + i];
    if (m.arch == TINY_ARCH_GPT) v += m.pos_tab[(size_t)P.pos[r] * d + i];
    s.x[idx] = v;
  }
  __syncthreads();
  mark(8);
  for (int l = 0; l < m.L; ++l) {
    const TinyLayer& w = m.layers[l];
    float* kc = m.kcache + (size_t)l * m.slots * kvd;
    float* vc = m.vcache + (size_t)l * m.slots * kvd;
    norm_rows(m, s.x, s.h, R, w.ln1_g, w.ln1_b);
    __syncthreads();
    mark(9);
    // q / k / v projections; k, v go straight to the row's cache slot
    const int nqkv = qd + 2 * kvd;
    for (int idx = tid; idx < R * nqkv; idx += nth) {
      int r = idx / nqkv, o = idx % nqkv;
      const float* a = s.h + (size_t)r * d;
      float acc = 0.f;
      for (int i = 0; i < d; ++i) acc = fmaf(a[i], w.wqkvT[(size_t)i * nqkv + o], acc);
      if (o < qd) s.q[(size_t)r * qd + o] = acc;
      else if (o < qd + kvd) kc[(size_t)P.slot[r] * kvd + (o - qd)] = acc;
      else vc[(size_t)P.slot[r] * kvd + (o - qd - kvd)] = acc;
    }
    __syncthreads();
    mark(10);
    if (m.arch == TINY_ARCH_LLAMA) {
      // rotate-half RoPE on q and on the freshly written k
      const int half = hd / 2;
      for (int idx = tid; idx < R * (H + KVH) * half; idx += nth) {
        int r = idx / ((H + KVH) * half);
        int rem = idx % ((H + KVH) * half);
        int hh = rem / half, i = rem % half;
        float c = m.rope_cos[(size_t)P.pos[r] * half + i];
        float sn = m.rope_sin[(size_t)P.pos[r] * half + i];
        float* base = (hh < H) ? (s.q + (size_t)r * qd + hh * hd)
                               : (kc + (size_t)P.slot[r] * kvd + (hh - H) * hd);
        float a = base[i], b = base[i + half];
        base[i] = a * c - b * sn;
        base[i + half] = b * c + a * sn;
      }
      __syncthreads();
    }
    // attention: one warp per (row, head); keys = prefix slots, chain slots
    // (relative-position order), self -- the structured mask as a chain
    if (hd <= 8) attn_rows<8>(m, s, P, kc, vc, R);
    else attn_rows<TINY_MAX_HD>(m, s, P, kc, vc, R);
    __syncthreads();
    mark(11);
    gemv_rows(s.att, qd, w.woT, nullptr, s.x, d, R, d, qd, true);   // x += ctx @ Wo
    __syncthreads();
    mark(12);
    norm_rows(m, s.x, s.h, R, w.ln2_g, w.ln2_b);
    __syncthreads();
    if (m.arch == TINY_ARCH_GPT) {
      // ReLU(h W1 + b1) W2 + b2 (models.py:263-265)
      for (int idx = tid; idx < R * m.ff; idx += nth) {
        int r = idx / m.ff, o = idx % m.ff;
        const float* a = s.h + (size_t)r * d;
        float acc = 0.f;
        for (int i = 0; i < d; ++i) acc = fmaf(a[i], w.w1T[(size_t)i * m.ff + o], acc);
        acc += w.b1[o];
        s.ff[idx] = acc > 0.f ? acc : 0.f;
      }
    } else {
      for (int idx = tid; idx < R * m.ff; idx += nth) {
        int r = idx / m.ff, o = idx % m.ff;
        const float* a = s.h + (size_t)r * d;
        float g = 0.f, u = 0.f;
        for (int i = 0; i < d; ++i) {
          g = fmaf(a[i], w.w1T[(size_t)i * m.ff + o], g);
          u = fmaf(a[i], w.wuT[(size_t)i * m.ff + o], u);
        }
        s.ff[idx] = g / (1.0f + expf(-g)) * u;
      }
    }
    __syncthreads();
    mark(13);
    gemv_rows(s.ff, m.ff, w.w2T, w.b2, s.x, d, R, d, m.ff, true);
    __syncthreads();
    mark(14);
  }
  // final norm + unembedding + per-row argmax (models.py:267-271, sampling.py:17-19)
  norm_rows(m, s.x, s.h, R, m.lnf_g, m.lnf_b);
  __syncthreads();
  for (int r = warp; r < R; r += nw) {
    const float* a = s.h + (size_t)r * d;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int v = lane; v < m.V; v += 32) {
      float acc = 0.f;
      for (int i = 0; i < d; ++i) acc = fmaf(a[i], m.unembedT[(size_t)i * m.V + v], acc);
      if (logits_out) logits_out[(size_t)r * m.V + v] = acc;
      argmax_merge(best, bi, acc, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float v2 = __shfl_xor_sync(0xffffffffu, best, o);
      int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(best, bi, v2, i2);
    }
    if (lane == 0) s.row_amax[r] = bi;
  }
  __syncthreads();
  mark(15);
}

// copy the K/V of accepted branch rows into place.
// One thread per (layer, element) walks i ascending: destination slot ctx+i
// can only alias the source of an i' <= i, which that thread already read.
__device__ void commit_kv(const TinyModel& m, const DevDecode& d) {
  const int n = d.commit_n;
  if (n <= 0) return;
  const int kvd = m.KVH * m.hd;
  for (int idx = threadIdx.x; idx < m.L * kvd; idx += blockDim.x) {
    int l = idx / kvd, e = idx % kvd;
    float* kc = m.kcache + (size_t)l * m.slots * kvd;
    float* vc = m.vcache + (size_t)l * m.slots * kvd;
    for (int i = 1; i <= n; ++i) {
      size_t src = (size_t)(d.commit_ctx + d.commit_base + i - 1) * kvd + e;
      size_t dst = (size_t)(d.commit_ctx + i) * kvd + e;
      kc[dst] = kc[src];
      vc[dst] = vc[src];
    }
  }
}

}  // namespace

int la_tiny_prof(bool enable, unsigned long long* out) {
  if (out) return cudaMemcpyFromSymbol(out, g_tiny_prof, sizeof(g_tiny_prof)) == cudaSuccess ? 0 : -1;
  int v = enable ? 1 : 0;
  unsigned long long z[16] = {};
  if (cudaMemcpyToSymbol(g_tiny_prof, z, sizeof(z)) != cudaSuccess) return -1;
  return cudaMemcpyToSymbol(g_tiny_prof_on, &v, sizeof(v)) == cudaSuccess ? 0 : -1;
}

// Activations in dynamic shared memory when the host sized it (s.smem): the
// phases' dependent reads then hit the SM instead of L2 (global stores bypass
// L1).  Layout [x | h | q | att | ff], LA_MAX_ROWS rows each.
__device__ __forceinline__ TinyScratch tiny_local(const TinyModel& m, TinyScratch s) {
  if (s.smem) {
    extern __shared__ float tiny_sm[];
    const int R = LA_MAX_ROWS, qd = m.H * m.hd;
    s.x = tiny_sm;
    s.h = s.x + R * m.d;
    s.q = s.h + R * m.d;
    s.att = s.q + R * qd;
    s.ff = s.att + R * qd;
  }
  return s;
}

__global__ void la_tiny_transpose(const float* in, int rows, int cols, float* out, int out_ld, int col_off) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < (long)rows * cols; i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols), c = (int)(i % cols);
    out[(size_t)c * out_ld + col_off + r] = in[i];
  }
}

size_t la_tiny_smem_bytes(const TinyModel& m, int* mode) {
  const size_t R = LA_MAX_ROWS, qd = (size_t)m.H * m.hd;
  const size_t act = R * (2 * (size_t)m.d + 2 * qd + (size_t)m.ff) * sizeof(float);
  // static smem (sampler, decode state, K1 / K10) stays below 24 KB
  if (act + sizeof(FwdPlan) <= 196 * 1024) { *mode = 2; return act + sizeof(FwdPlan); }
  if (act <= 160 * 1024) { *mode = 1; return act; }
  *mode = 0;                              // larger models keep the activations in global memory
  return 0;
}

int la_tiny_set_smem(size_t bytes) {
  const int b = (int)bytes;
  if (cudaFuncSetAttribute(la_tiny_prefill, cudaFuncAttributeMaxDynamicSharedMemorySize, b) != cudaSuccess ||
      cudaFuncSetAttribute(la_tiny_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, b) != cudaSuccess ||
      cudaFuncSetAttribute(la_tiny_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, b) != cudaSuccess ||
      cudaFuncSetAttribute(la_tiny_step_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, b) != cudaSuccess)
    return -1;
  return 0;
}

// The step plan in dynamic shared memory (s.smem == 2: after the activations).
__device__ __forceinline__ FwdPlan* tiny_plan(const TinyModel& m, const TinyScratch& s, FwdPlan* Pg) {
  if (s.smem != 2) return Pg;
  extern __shared__ float tiny_sm[];
  const size_t R = LA_MAX_ROWS, qd = (size_t)m.H * m.hd;
  return reinterpret_cast<FwdPlan*>(tiny_sm + R * (2 * (size_t)m.d + 2 * qd + (size_t)m.ff));
}
__device__ __forceinline__ void tiny_plan_store(const FwdPlan& src, FwdPlan* dst) {
  const int* a = reinterpret_cast<const int*>(&src);
  int* b = reinterpret_cast<int*>(dst);
  for (size_t i = threadIdx.x; i < sizeof(FwdPlan) / sizeof(int); i += blockDim.x) b[i] = a[i];
}

// Prefill: causal chain over prompt[0 .. n-1) in chunks of LA_MAX_ROWS rows.
__global__ void __launch_bounds__(TINY_THREADS) la_tiny_prefill(TinyModel m, TinyScratch sg, FwdPlan* P,
                                                       const int* tokens, int n) {
  const TinyScratch s = tiny_local(m, sg);
  for (int start = 0; start < n; start += LA_MAX_ROWS) {
    int R = min(LA_MAX_ROWS, n - start);
    if (threadIdx.x == 0) {
      P->n_rows = R; P->n_pad = la_round16(R); P->n_prefix = start; P->n_global = R;
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
    __syncthreads();
    forward_rows(m, s, *P, nullptr);
  }
}

// The decode loop: K1 build -> forward -> argmax -> K10 finish -> KV commit,
// until done (EOS / max_tokens) -- entirely on the device.  Under a
// temperature sampler (logits != null) the step also adjusts row 0 and the
// branch rows and runs verify_sample, in this CTA (la_sample.cuh).
__global__ void __launch_bounds__(TINY_THREADS) la_tiny_decode(TinyModel m, TinyScratch sg, FwdPlan* Pg,
                                                      DevDecode* dp, float* logits) {
  __shared__ LaSampleSmem sm;
  // the decode state (scalars, window, candidates, argmax table, accepted
  // tokens) and -- when the host sized it -- the step plan live in shared
  // memory for the whole decode: K1 / K10 / the forward chase them serially,
  // so every access is an SM round trip instead of an L2 one.  Written back
  // at the end (the host reads the state; tests read the plan).
  __shared__ DevDecode d;
  __shared__ int s_window[64 * LA_MAX_SUFFIX], s_cand[64 * LA_MAX_SUFFIX], s_amax[LA_MAX_ROWS],
      s_acc[LA_MAX_SUFFIX + 2];
  const TinyScratch s = tiny_local(m, sg);
  FwdPlan* P = tiny_plan(m, s, Pg);
  const int tid = threadIdx.x;
  if (tid == 0) d = *dp;
  __syncthreads();
  const int ncell = d.mode == LA_MODE_LOOKAHEAD ? (d.N - 1) * d.W - 1 : 0;
  const int ncand = d.mode == LA_MODE_LOOKAHEAD ? d.G * (d.N - 1) : 0;
  int* const g_window = d.window;
  int* const g_cand = d.cand;
  int* const g_amax = d.amax;
  int* const g_acc = d.accepted;
  for (int i = tid; i < ncell; i += blockDim.x) s_window[i] = g_window[i];
  for (int i = tid; i < ncand; i += blockDim.x) s_cand[i] = g_cand[i];
  for (int i = tid; i < LA_MAX_ROWS; i += blockDim.x) s_amax[i] = g_amax[i];
  for (int i = tid; i < d.N; i += blockDim.x) s_acc[i] = g_acc[i];
  __syncthreads();
  if (tid == 0) { d.window = s_window; d.cand = s_cand; d.amax = s_amax; d.accepted = s_acc; }
  TinyProf prof;
  for (int it = 0; it < d.max_steps; ++it) {
    __syncthreads();
    if (d.done) break;
    prof.mark(7);
    la_step_build(d, *P);
    if (P->n_rows == 0) break;
    prof.mark(0);
    forward_rows(m, s, *P, d.sample ? logits : nullptr, &prof);
    prof.mark(1);
    for (int r = threadIdx.x; r < P->n_rows; r += blockDim.x)
      if (P->own[r]) d.amax[P->grow[r]] = s.row_amax[r];
    __syncthreads();
    prof.mark(2);
    if (d.sample) {
      const int nr = la_sample_rows(d);
      bool ok = true;
      for (int j = 0; j < nr && ok; ++j)
        ok = la_adjust_row(logits + (size_t)la_sample_row(d, j) * m.V, m.V, d.temperature,
                           d.top_k, d.top_p, d.adj + (size_t)j * m.V, sm);
      if (ok) ok = la_verify_sample(d, sm);
      if (!ok && threadIdx.x == 0) d.degenerate = 1;
      __syncthreads();
    }
    prof.mark(3);
    la_step_finish(d);
    prof.mark(4);
    if (d.mode == LA_MODE_LOOKAHEAD) commit_kv(m, d);
    __syncthreads();
    prof.mark(5);
    if (prof.on && threadIdx.x == 0) g_tiny_prof[6] += 1;
  }
  __syncthreads();
  for (int i = tid; i < ncell; i += blockDim.x) g_window[i] = s_window[i];
  for (int i = tid; i < ncand; i += blockDim.x) g_cand[i] = s_cand[i];
  for (int i = tid; i < LA_MAX_ROWS; i += blockDim.x) g_amax[i] = s_amax[i];
  for (int i = tid; i < d.N; i += blockDim.x) g_acc[i] = s_acc[i];
  if (P != Pg) tiny_plan_store(*P, Pg);
  __syncthreads();
  if (tid == 0) {
    DevDecode out = d;
    out.window = g_window; out.cand = g_cand; out.amax = g_amax; out.accepted = g_acc;
    *dp = out;
  }
}

// Parity hook: evaluate an explicit plan (prefix already cached) and dump logits.
__global__ void __launch_bounds__(TINY_THREADS) la_tiny_forward(TinyModel m, TinyScratch sg, FwdPlan* P,
                                                       float* logits) {
  const TinyScratch s = tiny_local(m, sg);
  forward_rows(m, s, *P, logits);
}

// Step-granular variants for lookahead parallelism (la_decode_lookahead_group):
// phase A = K1 build + forward + owned-row argmax; the host-side group then
// exchanges the argmax table and the winner's K/V; phase B = K10 finish.
__global__ void __launch_bounds__(TINY_THREADS) la_tiny_step_forward(TinyModel m, TinyScratch sg,
                                                            FwdPlan* P, DevDecode* dp, float* logits) {
  const TinyScratch s = tiny_local(m, sg);
  DevDecode& d = *dp;
  la_step_build(d, *P);
  if (P->n_rows == 0) return;
  forward_rows(m, s, *P, logits);
  for (int r = threadIdx.x; r < P->n_rows; r += blockDim.x)
    if (P->own[r]) d.amax[P->grow[r]] = s.row_amax[r];
}

__global__ void __launch_bounds__(256) la_tiny_step_finish(DevDecode* dp) {
  la_step_finish(*dp);
}
