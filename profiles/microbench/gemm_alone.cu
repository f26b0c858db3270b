// The decode GEMM (la_gemm_kernel, split-K pieces, no epilogue) launched
// back to back on one stream: steady-state weight-streaming rate of the
// kernel itself, with and without programmatic dependent launch, against the
// plain bulk-copy streaming rate (stream_sms.cu).  7B shapes, 60 step rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../include \
//        -I ../../paper_2402_02057_b200/csrc gemm_alone.cu -L ../../paper_2402_02057_b200/lib \
//        -llookahead_b200 -o gemm_alone
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "la_gemm.cuh"

int la_gemm_workspace_segs(int n_tiles, int kb, int grid, int tpc);

int main(int argc, char** argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 60;
  struct Shape { const char* name; int tiles, K, tpc; } shapes[] = {
      {"qkv", 96, 4096, 2}, {"o", 32, 4096, 2}, {"gu", 172, 4096, 2}, {"down", 32, 11008, 2}, {"head", 250, 4096, 2}};
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  FwdPlan hp;
  memset(&hp, 0, sizeof(hp));
  hp.n_rows = rows; hp.n_pad = (rows + 15) & ~15;
  FwdPlan* dp;
  cudaMalloc(&dp, sizeof(FwdPlan));
  cudaMemcpy(dp, &hp, sizeof(hp), cudaMemcpyHostToDevice);
  void* act;
  cudaMalloc(&act, (size_t)128 * 11008 * 2);
  cudaMemset(act, 0, (size_t)128 * 11008 * 2);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& s : shapes) {
    const int kb = s.K / 64;
    const size_t wbytes = (size_t)s.tiles * kb * 16384;
    // 4 copies of the matrix (> L2) so every launch streams from HBM
    const int ncopy = argc > 2 ? atoi(argv[2]) : 4;   // 1: the same matrix every launch (L2-resident when it fits)
    void* w;
    cudaMalloc(&w, wbytes * ncopy);
    cudaMemset(w, 0, wbytes * ncopy);
    LaGemm g[8];
    const int grid = sms;
    const int segs = la_gemm_workspace_segs(s.tiles, kb, grid, s.tpc);
    float* ws;
    cudaMalloc(&ws, (size_t)s.tiles * segs * 128 * 128 * 4);
    for (int c = 0; c < ncopy; ++c) {
      memset(&g[c], 0, sizeof(LaGemm));
      g[c].epi = getenv("NT") && atoi(getenv("NT")) ? LA_EPI_PARTIAL : LA_EPI_PARTIAL_SW;
      g[c].grid = grid;
      g[c].args.a = reinterpret_cast<const __nv_bfloat16*>((char*)w + c * wbytes);
      g[c].args.b = reinterpret_cast<const __nv_bfloat16*>(act);
      g[c].args.n_tiles = s.tiles; g[c].args.tpc = s.tpc; g[c].args.kb = kb; g[c].args.max_segs = segs;
      g[c].args.plan = dp; g[c].args.ws = ws;
    }
    const int dbgs[] = {0, 1, 2, 3};
    for (int di = 0; di < 5; ++di) {
      const int pdl = di == 0 ? 0 : 1, dbg = di == 0 ? 0 : dbgs[di - 1];
      for (int c = 0; c < ncopy; ++c) g[c].args.debug = dbg;
      for (int i = 0; i < 8; ++i) la_gemm_launch(g[i % ncopy], st, pdl);
      const int n = 40;
      cudaEventRecord(a, st);
      for (int i = 0; i < n; ++i) la_gemm_launch(g[i % ncopy], st, pdl);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double us = ms * 1e3 / n;
      printf("%-5s rows %3d  %6.1f MB  pdl %d  dbg %d (1: no B loads, 2: no MMAs)  %7.2f us/launch  %7.1f GB/s\n", s.name,
             rows, wbytes / 1e6, pdl, dbg, us, wbytes / (us * 1e-6) / 1e9);
    }
    {
      // unit-arrival cadence of one more launch (utrace: MMA thread passing
      // each unit's full barrier), pdl 1, no debug flags
      unsigned long long* ut;
      cudaMalloc(&ut, 256 * 32 * 8);
      cudaMemset(ut, 0, 256 * 32 * 8);
      for (int c = 0; c < ncopy; ++c) { g[c].args.debug = 0; g[c].args.utrace = ut; }
      la_gemm_launch(g[0], st, true);
      cudaStreamSynchronize(st);
      unsigned long long h[148 * 32];
      cudaMemcpy(h, ut, sizeof(h), cudaMemcpyDeviceToHost);
      printf("  cadence (CTA 0..3, us after unit 0):");
      for (int c = 0; c < 4; ++c) {
        printf(" |");
        for (int i = 1; i < 8; ++i) if (h[c * 32 + i]) printf(" %.2f", (h[c * 32 + i] - h[c * 32]) / 1e3);
      }
      printf("\n");
      for (int c = 0; c < ncopy; ++c) g[c].args.utrace = nullptr;
      cudaFree(ut);
    }
    cudaFree(w);
    cudaFree(ws);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
