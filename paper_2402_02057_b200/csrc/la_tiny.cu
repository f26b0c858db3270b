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

// out[r][o] (+)= sum_i in[r][i] * W[o][i]  (+ bias)
__device__ void gemv_rows(const float* in, int in_ld, const float* W, const float* bias, float* out,
                          int out_ld, int R, int n_out, int n_in, bool accumulate) {
  for (int idx = threadIdx.x; idx < R * n_out; idx += blockDim.x) {
    int r = idx / n_out, o = idx % n_out;
    const float* a = in + (size_t)r * in_ld;
    const float* w = W + (size_t)o * n_in;
    float acc = 0.f;
    for (int i = 0; i < n_in; ++i) acc = fmaf(a[i], w[i], acc);
    if (bias) acc += bias[o];
    float* dst = out + (size_t)r * out_ld + o;
    *dst = accumulate ? (*dst + acc) : acc;
  }
}

__device__ void forward_rows(const TinyModel& m, const TinyScratch& s, const FwdPlan& P,
                             float* logits_out) {
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
  for (int l = 0; l < m.L; ++l) {
    const TinyLayer& w = m.layers[l];
    float* kc = m.kcache + (size_t)l * m.slots * kvd;
    float* vc = m.vcache + (size_t)l * m.slots * kvd;
    norm_rows(m, s.x, s.h, R, w.ln1_g, w.ln1_b);
    __syncthreads();
    // q / k / v projections; k, v go straight to the row's cache slot
    for (int idx = tid; idx < R * (qd + 2 * kvd); idx += nth) {
      int r = idx / (qd + 2 * kvd), o = idx % (qd + 2 * kvd);
      const float* Wt;
      int oo;
      if (o < qd) { Wt = w.wq; oo = o; }
      else if (o < qd + kvd) { Wt = w.wk; oo = o - qd; }
      else { Wt = w.wv; oo = o - qd - kvd; }
      const float* a = s.h + (size_t)r * d;
      const float* ww = Wt + (size_t)oo * d;
      float acc = 0.f;
      for (int i = 0; i < d; ++i) acc = fmaf(a[i], ww[i], acc);
      if (o < qd) s.q[(size_t)r * qd + oo] = acc;
      else if (o < qd + kvd) kc[(size_t)P.slot[r] * kvd + oo] = acc;
      else vc[(size_t)P.slot[r] * kvd + oo] = acc;
    }
    __syncthreads();
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
    // (relative-position order), self -- the structured mask as a chain.
    const float scale = 1.0f / sqrtf((float)hd);
    for (int job = warp; job < R * H; job += nw) {
      int r = job / H, hh = job % H, kvh = hh / (H / KVH);
      const float* q = s.q + (size_t)r * qd + hh * hd;
      float* sc = s.scores + (size_t)job * s.max_keys;
      const int npre = P.n_prefix, nch = P.chain_n[r];
      const int nk = npre + nch + 1;
      float mx = -INFINITY;
      for (int j = lane; j < nk; j += 32) {
        int slot = (j < npre) ? j : (j < npre + nch ? P.chain[r][j - npre] : P.slot[r]);
        const float* kk = kc + (size_t)slot * kvd + kvh * hd;
        float dot = 0.f;
        for (int i = 0; i < hd; ++i) dot = fmaf(q[i], kk[i], dot);
        dot *= scale;
        sc[j] = dot;
        mx = fmaxf(mx, dot);
      }
      mx = warp_max(mx);
      float sum = 0.f;
      for (int j = lane; j < nk; j += 32) {
        float e = expf(sc[j] - mx);
        sc[j] = e;
        sum += e;
      }
      sum = warp_sum(sum);
      __syncwarp();
      float inv = 1.0f / sum;
      for (int i = lane; i < hd; i += 32) {
        float acc = 0.f;
        for (int j = 0; j < nk; ++j) {
          int slot = (j < npre) ? j : (j < npre + nch ? P.chain[r][j - npre] : P.slot[r]);
          acc = fmaf(sc[j], vc[(size_t)slot * kvd + kvh * hd + i], acc);
        }
        s.att[(size_t)r * qd + hh * hd + i] = acc * inv;
      }
    }
    __syncthreads();
    gemv_rows(s.att, qd, w.wo, nullptr, s.x, d, R, d, qd, true);   // x += ctx @ Wo
    __syncthreads();
    norm_rows(m, s.x, s.h, R, w.ln2_g, w.ln2_b);
    __syncthreads();
    if (m.arch == TINY_ARCH_GPT) {
      // ReLU(h W1 + b1) W2 + b2 (models.py:263-265)
      for (int idx = tid; idx < R * m.ff; idx += nth) {
        int r = idx / m.ff, o = idx % m.ff;
        const float* a = s.h + (size_t)r * d;
        const float* ww = w.w1 + (size_t)o * d;
        float acc = 0.f;
        for (int i = 0; i < d; ++i) acc = fmaf(a[i], ww[i], acc);
        acc += w.b1[o];
        s.ff[idx] = acc > 0.f ? acc : 0.f;
      }
    } else {
      for (int idx = tid; idx < R * m.ff; idx += nth) {
        int r = idx / m.ff, o = idx % m.ff;
        const float* a = s.h + (size_t)r * d;
        const float* wg = w.w1 + (size_t)o * d;
        const float* wu = w.wu + (size_t)o * d;
        float g = 0.f, u = 0.f;
        for (int i = 0; i < d; ++i) { g = fmaf(a[i], wg[i], g); u = fmaf(a[i], wu[i], u); }
        s.ff[idx] = g / (1.0f + expf(-g)) * u;
      }
    }
    __syncthreads();
    gemv_rows(s.ff, m.ff, w.w2, w.b2, s.x, d, R, d, m.ff, true);
    __syncthreads();
  }
  // final norm + unembedding + per-row argmax (models.py:267-271, sampling.py:17-19)
  norm_rows(m, s.x, s.h, R, m.lnf_g, m.lnf_b);
  __syncthreads();
  for (int r = warp; r < R; r += nw) {
    const float* a = s.h + (size_t)r * d;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int v = lane; v < m.V; v += 32) {
      const float* ww = m.unembed + (size_t)v * d;
      float acc = 0.f;
      for (int i = 0; i < d; ++i) acc = fmaf(a[i], ww[i], acc);
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

// Prefill: causal chain over prompt[0 .. n-1) in chunks of LA_MAX_ROWS rows.
__global__ void __launch_bounds__(1024) la_tiny_prefill(TinyModel m, TinyScratch s, FwdPlan* P,
                                                       const int* tokens, int n) {
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
__global__ void __launch_bounds__(1024) la_tiny_decode(TinyModel m, TinyScratch s, FwdPlan* P,
                                                      DevDecode* dp, float* logits) {
  __shared__ LaSampleSmem sm;
  DevDecode& d = *dp;
  for (int it = 0; it < d.max_steps; ++it) {
    __syncthreads();
    if (d.done) break;
    la_step_build(d, *P);
    if (P->n_rows == 0) break;
    forward_rows(m, s, *P, d.sample ? logits : nullptr);
    for (int r = threadIdx.x; r < P->n_rows; r += blockDim.x)
      if (P->own[r]) d.amax[P->grow[r]] = s.row_amax[r];
    __syncthreads();
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
    la_step_finish(d);
    if (d.mode == LA_MODE_LOOKAHEAD) commit_kv(m, d);
    __syncthreads();
  }
}

// Parity hook: evaluate an explicit plan (prefix already cached) and dump logits.
__global__ void __launch_bounds__(1024) la_tiny_forward(TinyModel m, TinyScratch s, FwdPlan* P,
                                                       float* logits) {
  forward_rows(m, s, *P, logits);
}

// Step-granular variants for lookahead parallelism (la_decode_lookahead_group):
// phase A = K1 build + forward + owned-row argmax; the host-side group then
// exchanges the argmax table and the winner's K/V; phase B = K10 finish.
__global__ void __launch_bounds__(1024) la_tiny_step_forward(TinyModel m, TinyScratch s,
                                                            FwdPlan* P, DevDecode* dp, float* logits) {
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
