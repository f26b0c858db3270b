// Small-M weight-streaming GEMM on tcgen05 (declarations).
//
//   P[tok][f] = sum_k X[tok][k] * Wt[f][k]      (X: <= 128 step rows, Wt: weights [out][in])
//
// Swap-AB: the weight tile is the MMA "A" operand (M = 128 output features),
// the step rows are "B" (N = n_pad tokens), accumulators live in TMEM.
// Weights are stored PACKED ("LA tiles"): 128-row x 64-column bf16 blocks,
// each 16 KB contiguous and already in the 128-byte-swizzled shared-memory
// image, ordered tile-major / k-minor.  A stream-K work unit (tile, k-block)
// is therefore one contiguous 16 KB read (cp.async.bulk), and a CTA's whole
// unit range is one contiguous stretch of HBM.
//
// The GEMM writes fp32 partial tiles (one per (tile, contributing CTA)
// segment) to a workspace; separate fused reduce kernels sum the segments
// in fixed order (deterministic, layout-independent) and apply the epilogue
// (RoPE + KV write, residual + RMSNorm, SwiGLU, argmax) spread over the
// whole GPU instead of serialised in the last-arriving CTA.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "la_common.cuh"

// Tiles processed per stream-K unit: one step-row (B) load feeds two 128-row
// weight tiles, halving the L2->SM traffic of the activations.
#define LA_TPC 2

// Packed activation layout ("LA rows"): [K/64 blocks][128 rows][64] bf16,
// every 16 KB block the SWIZZLE_128B image of a 128 x 64 tile, so the first
// n_pad rows of a k-block are ONE contiguous n_pad*128-byte bulk copy.
__host__ __device__ __forceinline__ size_t la_act_off(int r, int k) {
  return (size_t)(k >> 6) * 8192 + (size_t)r * 64 + ((((k >> 3) & 7) ^ (r & 7)) << 3) + (k & 7);
}

struct LaNextPf {
  const void* a;   // packed weights of a following GEMM (null: none)
  int n_tiles, kb, tpc, grid;
  int skip, units;  // per CTA: units [skip, skip + units) of its stream-K range
};

struct LaGemmArgs {
  const __nv_bfloat16* a;   // packed weight tiles [n_tiles/2][kb][2][128*64]
  const __nv_bfloat16* b;   // packed step rows [kb][128][64]
  int n_tiles;              // 128-row feature tiles (even)
  int tpc;                  // tiles per stream-K unit (1 or LA_TPC)
  int kb;                   // K / 64
  int max_segs;             // workspace segments per tile
  const FwdPlan* plan;
  float* ws;                // [n_tiles][max_segs][128 tok][128 f] fp32 partials
  // launch timing (device globaltimer): [0] first-CTA start, [1] sum ns,
  // [2] launches, [3] started CTAs, [4] finished CTAs; null = off
  unsigned long long* timing;
  // optional per-CTA trace [gridDim][4]: start, prologue done, MMA done, end
  unsigned long long* trace;
  // optional per-CTA unit trace [gridDim][32]: when the MMA thread saw unit
  // i's stage full (i < 32), to read the weight stream's ramp
  unsigned long long* utrace;
  int debug;   // experiments: bit0 skip step-row loads, bit1 skip MMAs
  int l2pf;    // units beyond the smem ring prefetched to L2 before the dependency wait
  int nst;     // smem ring stages (0: the default for tpc); fewer stages = a smaller CTA
               // that fits beside the previous kernel's CTA and streams its weights early
  // ---- multi-chunk mode (prefill, nblk > 1, tpc == 1, split-K pieces only):
  // every weight stage multiplies nblk <= 4 row blocks -- block 0 = b / ws /
  // plan, block j = bx[j-1] / wsx[j-1] / planx[j-1] -- so one weight pass
  // serves up to 512 rows (TMEM: double-buffered for <= 2 blocks, single above)
  int nblk;
  const __nv_bfloat16* bx[3];
  float* wsx[3];
  const FwdPlan* planx[3];
  // ---- fused epilogue (LA_EPI_QKV / SWIGLU / LOGITS): stream-K fix-up in
  // the GEMM -- the CTA owning a tile's k = 0 piece adds the other pieces'
  // partials (in piece order) and applies the epilogue
  int* counters;                     // [unit tiles] pieces arrived (reset by the owner)
  __nv_bfloat16* q_out;              // QKV: [128][H][128]
  __nv_bfloat16 *kc, *vc;            // QKV: layer base [slots][KVH][128]
  const float *rope_cos, *rope_sin;  // QKV: [slots][64]
  int H, KVH;
  __nv_bfloat16* act;                // SWIGLU: packed LA rows
  unsigned long long* keys;          // LOGITS: [128] (value, -index) atomicMax keys
  float* logits;                     // LOGITS: [128][V] dump or null
  int V;
  LaRowNorm nrm;                     // fused epilogues: deferred RMSNorm of the input rows
  // ---- split-K fix-up inside the GEMM (LA_EPI_FX_*): every CTA writes its
  // pieces and counts them in (fx_arrive); after its own unit range it waits
  // until each unit tile it touched has all pieces, bulk-copies ITS row slice
  // of every piece into the (now idle) smem ring and applies the epilogue to
  // that slice -- the n contributors of a tile finish n disjoint row slices,
  // so the reduction is spread and needs no separate kernel
  int* fx_arrive;                    // [unit tiles] pieces written (reset by the last departer)
  int* fx_depart;                    // [unit tiles] slices finished
  int n_real;                        // real feature tiles (the packing pads to LA_TPC)
  float* x;                          // FX_RESID: [128][d] fp32 residual stream (x += piece sum)
  const float* gain;                 // FX_RESID: next RMSNorm gain
  __nv_bfloat16* h_out;              // FX_RESID: next GEMM input bf16(x * gain), packed LA rows
  float* ss_out;                     // FX_RESID: [d/128][128] per-tile sums of x^2
  int d;
  // ---- cross-GEMM L2 prefetch: after issuing its last weight load, CTA c
  // pulls the units [skip, skip + units) of CTA c's range in the next GEMMs
  // into L2, so HBM keeps streaming through the latency-bound kernels that
  // separate two GEMMs (their data then arrives from L2)
  LaNextPf npf[2];
  // per-unit-tile piece counters (monotonic: + contributors per launch) that
  // the epilogue kernel polls instead of waiting for the whole grid (null: off)
  int* ready;
};

enum LaGemmEpi { LA_EPI_PARTIAL = 0, LA_EPI_QKV = 1, LA_EPI_SWIGLU = 2, LA_EPI_LOGITS = 3,
                 LA_EPI_MULTI = 4,     // split-K pieces, nblk row blocks (prefill; chosen by nblk > 1)
                 // split-K fix-up + epilogue in the GEMM (decode step; la_gemm.cu)
                 LA_EPI_FX_QKV = 5,    // RoPE, q / K / V out (la_qkv_epi_kernel's math)
                 LA_EPI_FX_SWIGLU = 6, // SwiGLU -> act (la_swiglu_epi_kernel's math)
                 LA_EPI_FX_RESID = 7,  // x += sum, next norm's h and sums of x^2 (la_resid_norm_kernel's)
                 // split-K pieces accumulated swap-AB (weight rows x step rows,
                 // N = padded rows; LA_GEMM_NT=0) instead of the default
                 // (step rows x weight rows, N = 128 tpc)
                 LA_EPI_PARTIAL_SW = 8,
                 // whole tiles per CTA (SwiGLU from TMEM) + stream-K remainder
                 // fixed up in-kernel (la_gemm_dpsk_kernel; gate/up)
                 LA_EPI_DPSK_SWIGLU = 9};

struct LaGemm {
  LaGemmArgs args;
  int grid;
  int epi;    // LaGemmEpi
};

int la_make_tmap(CUtensorMap* map, const void* base, int rows, int K, int box_rows);
int la_gemm_launch(const LaGemm& g, cudaStream_t st, bool pdl = false);
bool la_gemm_fx_fits(const LaGemm& g);   // the fix-up staging fits the smem ring
int la_gemm_workspace_segs(int n_tiles, int kb, int grid, int tpc);
int la_gemm_dpsk_segs(int n_real, int kb, int grid);
int la_sm_count();
size_t la_packed_elems(int rows, int K);   // bf16 elements of a packed matrix

__host__ __device__ __forceinline__ long la_cta_of(long u, long U, long P) {
  return ((u + 1) * P + U - 1) / U - 1;
}
// contributing CTAs [c0, c0 + n) of feature tile t (n_tiles tiles, tpc per unit)
__host__ __device__ __forceinline__ void la_tile_segs(int t, int kb, int n_tiles, long P, long& c0,
                                                      int& n, int tpc = LA_TPC) {
  const long U = (long)(n_tiles / tpc) * kb;
  const long pair = t / tpc;
  c0 = la_cta_of(pair * kb, U, P);
  long c1 = la_cta_of((pair + 1) * kb - 1, U, P);
  n = (int)(c1 - c0 + 1);
}
