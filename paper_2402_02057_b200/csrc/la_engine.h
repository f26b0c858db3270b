// Internal engine object behind the C ABI (include/lookahead_b200.h).
#pragma once
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "../../include/lookahead_b200.h"
#include "la_common.cuh"
#include "la_tiny.h"

void la_set_error(const char* fmt, ...);

struct LlamaPath;   // bf16 multi-kernel path (la_llama.cu)
struct LpComm;      // NCCL state (la_lp.cu)

struct la_engine {
  la_model_desc desc{};
  int device = 0;
  std::vector<const void*> w;          // borrowed device weight pointers
  std::vector<void*> owned;            // device allocations freed by la_destroy

  // ---- decode state (device)
  DevDecode h_dec{};                   // host mirror (pointers + config)
  DevDecode* d_dec = nullptr;
  FwdPlan* d_plan = nullptr;
  int *d_window = nullptr, *d_out = nullptr, *d_rec = nullptr, *d_cand = nullptr;
  int *d_amax = nullptr, *d_acc = nullptr;
  int *d_rng = nullptr;  int rng_cap = 0;
  int *d_tokens = nullptr; int tokens_cap = 0;
  int *d_grams = nullptr; int grams_cap = 0;
  int out_cap = 0, rec_cap = 0;
  // temperature sampler buffers (grown on demand)
  float* d_logits = nullptr; int logits_cap = 0;   // [LA_MAX_ROWS][V]
  double* d_adj = nullptr; int adj_cap = 0;        // [rows][V]
  double* d_work = nullptr; int work_cap = 0;      // [V]
  int* d_flag = nullptr; int flag_cap = 0;
  // pool arrays (grown on demand)
  int *p_lead = nullptr, *p_cnt = nullptr, *p_suf = nullptr, *p_set = nullptr;
  int *p_counters = nullptr, *p_log = nullptr;
  int *p_stamp = nullptr, *p_fifo = nullptr;   // LRU cap: [ST] stamps, [log_cap] fifo
  int *p_head = nullptr, *p_prev = nullptr, *p_next = nullptr;   // LRU cap: [LT] list heads, [ST] links
  size_t p_lt = 0, p_st = 0, p_log_cap = 0, p_C = 0, p_N = 0;

  // ---- KV cache [layer][slot][row_bytes]
  void *kc = nullptr, *vc = nullptr;
  int slots = 0, row_bytes = 0;

  // ---- fp32 tiny path
  TinyModel tm{};
  TinyScratch ts{};
  size_t tiny_smem = 0;                // dynamic smem of the fp32 kernels (activations), 0: global

  // ---- bf16 path
  LlamaPath* llama = nullptr;

  // ---- lookahead parallelism
  LpComm* lp = nullptr;
  int rank = 0, world = 1;
  uint8_t* kv_send = nullptr;          // [layers][N_MAX-1][2][row_bytes]
  uint8_t* kv_recv = nullptr;          // [world][...]
  int* amax_recv = nullptr;            // [world][LA_MAX_ROWS]
  size_t kv_seg = 0;
  int kv_world = 0;

  cudaEvent_t ev[4] = {};

  // ---- step session (la_session_start / la_session_step)
  bool session = false;
  DevDecode sess{};                    // device state after the last step

  bool is_tiny() const { return desc.arch != LA_ARCH_LLAMA_BF16; }
};

#define LA_MAX_NGRAM 8

// bf16 path entry points (la_llama.cu)
int llama_create(la_engine* e);
void llama_destroy(la_engine* e);
int llama_prefill(la_engine* e, const int* d_tokens, int n, cudaStream_t st);
int llama_decode_loop(la_engine* e, cudaStream_t st, int* launches);
int llama_forward_plan(la_engine* e, float* d_logits, cudaStream_t st);
int llama_step_forward(la_engine* e, cudaStream_t st);   // K1 + forward + owned argmax
int llama_session_step(la_engine* e, cudaStream_t st);   // one eager step (K1 .. commit)
int llama_mega_error(la_engine* e);                      // persistent-kernel dependency timeout flag
cudaError_t llama_copy_argmax(la_engine* e, int32_t* host, int n, cudaStream_t st);   // last forward's row argmax
