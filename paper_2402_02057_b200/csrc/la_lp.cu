// Lookahead parallelism (reference parallel.py:145-192).
//
// Each replica holds the full model and evaluates its visibility-closed
// share of the step rows (contiguous window columns + round-robin candidate
// branches, la_lp_row_role).  Per step there are exactly two exchanges:
//   1. an all-gather of the per-global-row argmax table (int32[128] per rank)
//      after the forward -- every replica then runs the identical,
//      deterministic K10 (verify / pool / window / RNG) like the reference's
//      coordinator (parallel.py:166-167);
//   2. an all-gather of the accepted branch's K/V rows, packed by the branch
//      owner, so every replica commits the same KV.
// Transport: NCCL over NVLink for one process per GPU (la_lp_init), or a
// device copy between engines of one process (la_decode_lookahead_group,
// the reference's in-process simulation).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <vector>

#include "la_engine.h"
#include "la_kernels.h"

struct LpComm {
  ncclComm_t comm = nullptr;
};

// NCCL is resolved at la_lp_init time (dlopen), not at library load: the
// process usually already holds torch's libnccl.so.2, which must win, and
// single-GPU users never need NCCL at all.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi& nccl() {
  static NcclApi api;
  if (api.ok) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
           api.GetErrorString;
  return api;
}

#define ncclGetUniqueId nccl().GetUniqueId
#define ncclCommInitRank nccl().CommInitRank
#define ncclCommDestroy nccl().CommDestroy
#define ncclAllGather nccl().AllGather
#define ncclGetErrorString nccl().GetErrorString

static int need_nccl() {
  if (!nccl().ok) { la_set_error("libnccl.so.2 could not be loaded"); return LA_ERR_NCCL; }
  return LA_OK;
}

#define NCK(x)                                                                   \
  do {                                                                           \
    ncclResult_t _r = (x);                                                       \
    if (_r != ncclSuccess) {                                                     \
      la_set_error("%s:%d %s: %s", __FILE__, __LINE__, #x, ncclGetErrorString(_r)); \
      return LA_ERR_NCCL;                                                        \
    }                                                                            \
  } while (0)
#define CK(x) LA_CUDA_CHECK(x)

void lp_destroy(la_engine* e) {
  if (e->lp) {
    if (e->lp->comm) ncclCommDestroy(e->lp->comm);
    delete e->lp;
    e->lp = nullptr;
  }
}

int lp_buffers(la_engine* e, int world) {
  const size_t seg = (size_t)e->desc.layers * (LA_MAX_NGRAM - 1) * 2 * e->row_bytes;
  if (e->kv_send && e->kv_seg == seg && e->kv_world == world) return LA_OK;
  if (e->kv_send) {
    for (void* p : {(void*)e->kv_send, (void*)e->kv_recv, (void*)e->amax_recv}) {
      auto it = std::find(e->owned.begin(), e->owned.end(), p);
      if (it != e->owned.end()) e->owned.erase(it);
      cudaFree(p);
    }
  }
  CK(cudaMalloc(&e->kv_send, seg));
  CK(cudaMalloc(&e->kv_recv, seg * world));
  CK(cudaMalloc(&e->amax_recv, sizeof(int) * LA_MAX_ROWS * world));
  e->owned.push_back(e->kv_send);
  e->owned.push_back(e->kv_recv);
  e->owned.push_back(e->amax_recv);
  e->kv_seg = seg;
  e->kv_world = world;
  return LA_OK;
}

extern "C" int32_t la_lp_unique_id(void* out) {
  if (!out) { la_set_error("null output"); return LA_ERR_INVALID_CONFIG; }
  if (int rc = need_nccl()) return rc;
  ncclUniqueId id;
  NCK(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out, &id, sizeof(id));
  return LA_OK;
}

extern "C" int32_t la_lp_init(la_engine* e, const void* unique_id, int32_t rank, int32_t world) {
  if (!e || !unique_id) { la_set_error("null engine or id"); return LA_ERR_INVALID_CONFIG; }
  if (world < 1 || rank < 0 || rank >= world) { la_set_error("bad rank/world"); return LA_ERR_INVALID_CONFIG; }
  CK(cudaSetDevice(e->device));
  lp_destroy(e);
  if (world > 1) {
    if (int rc = need_nccl()) return rc;
    e->lp = new LpComm();
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    NCK(ncclCommInitRank(&e->lp->comm, world, id, rank));
  }
  int rc = lp_buffers(e, world);
  if (rc) return rc;
  e->rank = rank;
  e->world = world;
  return LA_OK;
}

// forward half of a step on one replica: K1 build + forward + owned argmax
static int step_forward(la_engine* e, cudaStream_t st) {
  if (e->is_tiny()) {
    la_tiny_step_forward<<<1, TINY_THREADS, e->tiny_smem, st>>>(e->tm, e->ts, e->d_plan, e->d_dec, nullptr);
    CK(cudaGetLastError());
    return LA_OK;
  }
  return llama_step_forward(e, st);
}

static int step_finish(la_engine* e, const int* gathered_amax, int world, cudaStream_t st) {
  la_merge_amax_kernel<<<1, 128, 0, st>>>(e->d_dec, gathered_amax, world);
  la_step_finish_kernel<<<1, 256, 0, st>>>(e->d_dec);
  la_kv_pack_kernel<<<64, 256, 0, st>>>(e->d_dec, (const uint8_t*)e->kc, (const uint8_t*)e->vc,
                                        e->kv_send, e->desc.layers, e->slots, e->row_bytes);
  CK(cudaGetLastError());
  return LA_OK;
}

static int step_unpack(la_engine* e, cudaStream_t st) {
  la_kv_unpack_kernel<<<64, 256, 0, st>>>(e->d_dec, e->kv_recv, e->kv_seg, (uint8_t*)e->kc, (uint8_t*)e->vc,
                                          e->desc.layers, e->slots, e->row_bytes);
  CK(cudaGetLastError());
  return LA_OK;
}

static int poll_done(la_engine* e, cudaStream_t st, bool* done) {
  static thread_local int* pinned = nullptr;
  if (!pinned) CK(cudaMallocHost(&pinned, sizeof(int)));
  CK(cudaMemcpyAsync(pinned, &e->d_dec->done, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *done = *pinned != 0;
  return LA_OK;
}

// NCCL replica loop (one process per GPU).
int lp_decode_loop(la_engine* e, cudaStream_t st, int* launches) {
  if (!e->lp || !e->lp->comm) { la_set_error("la_lp_init was not called"); return LA_ERR_INVALID_CONFIG; }
  const int world = e->world;
  const int max_steps = e->h_dec.max_steps;
  const int poll_every = 4;
  int n = 0;
  for (int step = 0; step < max_steps; ++step) {
    int rc = step_forward(e, st);
    if (rc) return rc;
    NCK(ncclAllGather(e->d_amax, e->amax_recv, LA_MAX_ROWS, ncclInt32, e->lp->comm, st));
    if ((rc = step_finish(e, e->amax_recv, world, st))) return rc;
    NCK(ncclAllGather(e->kv_send, e->kv_recv, e->kv_seg, ncclUint8, e->lp->comm, st));
    if ((rc = step_unpack(e, st))) return rc;
    n += 6;
    if ((step + 1) % poll_every == 0) {
      bool done;
      if ((rc = poll_done(e, st, &done))) return rc;
      if (done) break;
    }
  }
  *launches = n;
  return LA_OK;
}

// In-process group: engine i is rank i; exchanges are device copies.
int lp_group_loop(la_engine* const* es, int n, cudaStream_t st, int* launches) {
  const int max_steps = es[0]->h_dec.max_steps;
  int count = 0;
  for (int step = 0; step < max_steps; ++step) {
    for (int r = 0; r < n; ++r) {
      int rc = step_forward(es[r], st);
      if (rc) return rc;
    }
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q)
        CK(cudaMemcpyAsync(es[r]->amax_recv + q * LA_MAX_ROWS, es[q]->d_amax,
                           sizeof(int) * LA_MAX_ROWS, cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < n; ++r) {
      int rc = step_finish(es[r], es[r]->amax_recv, n, st);
      if (rc) return rc;
    }
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q)
        CK(cudaMemcpyAsync(es[r]->kv_recv + q * es[r]->kv_seg, es[q]->kv_send, es[q]->kv_seg,
                           cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < n; ++r) {
      int rc = step_unpack(es[r], st);
      if (rc) return rc;
    }
    count += 6 * n;
    bool done;
    int rc = poll_done(es[0], st, &done);
    if (rc) return rc;
    if (done) break;
  }
  *launches = count;
  return LA_OK;
}
