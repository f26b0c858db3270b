// Do bulk copies issued by a PDL secondary BEFORE griddepcontrol.wait make
// progress while the primary grid is still running?
//   A (primary): 148 CTAs x 256 threads, launch_dependents at once, spin S us
//   B (secondary): at entry thread 0 issues 4 x 32 KB cp.async.bulk loads
//   (one mbarrier each); mode 0: griddepcontrol.wait, then wait the loads;
//   mode 1: wait the loads first (before griddepcontrol.wait), then wait.
// Prints per-CTA medians of entry, load arrivals and wait return relative to
// A's end.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_preload pdl_preload.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void kA(unsigned long long* t, int spin_ns, int self_load, const uint8_t* buf) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const unsigned long long t0 = gt();
  unsigned acc = 0;
  if (self_load) {   // light L2 traffic like an epilogue kernel
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) acc += buf[(size_t)blockIdx.x * 65536 + i * 16];
  }
  while (gt() - t0 < (unsigned long long)spin_ns) {}
  if (acc == 12345) t[1] = acc;
  if (threadIdx.x == 0) atomicMax(&t[0], gt());
}

__global__ void __launch_bounds__(64, 1) kB(unsigned long long* t, const uint8_t* w, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 4 * 32768);
  const unsigned long long t_entry = gt();
  unsigned long long ta[4] = {0, 0, 0, 0}, tw = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < 4; ++s) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(32768) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(sm + s * 32768)), "l"(w + ((size_t)blockIdx.x * 4 + s) * 32768), "r"(32768), "r"(su32(&bar[s]))
                   : "memory");
    }
    auto wait_loads = [&]() {
      for (int s = 0; s < 4; ++s) {
        asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W%=;\n}\n"
                     ::"r"(su32(&bar[s])) : "memory");
        ta[s] = gt();
      }
    };
    if (mode == 1) wait_loads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    tw = gt();
    if (mode == 0) wait_loads();
    unsigned long long* r = t + 8 + blockIdx.x * 8;
    r[0] = t_entry; r[1] = tw; r[2] = ta[0]; r[3] = ta[1]; r[4] = ta[2]; r[5] = ta[3];
  }
}

int main() {
  uint8_t* w;
  uint8_t* l2buf;
  unsigned long long* t;
  const size_t wbytes = 1ull << 30;
  cudaMalloc(&w, wbytes);
  cudaMalloc(&l2buf, 148 * 65536);
  cudaMemset(w, 1, wbytes);
  cudaMalloc(&t, (8 + 148 * 8) * 8);
  const int smem = 4 * 32768 + 64;
  cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  size_t woff = 0;
  for (int carve = 0; carve < 2; ++carve)
  for (int a_pdl = 1; a_pdl < 2; ++a_pdl)
  for (int a_grid : {148})
  for (int self_load = 0; self_load < 1; ++self_load)
    for (int spin : {20000})
      for (int mode = 0; mode < 2; ++mode) {
        int early = 0;
        std::vector<double> med(6, 0.0);
        const int reps = 5;
        for (int rep = 0; rep < reps; ++rep) {
          cudaMemsetAsync(t, 0, (8 + 148 * 8) * 8, st);
          cudaGraph_t graph;
          cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
          cudaFuncSetAttribute(kA, cudaFuncAttributePreferredSharedMemoryCarveout, carve ? 100 : -1);
          {
            cudaLaunchConfig_t ca = {};
            ca.gridDim = a_grid; ca.blockDim = 256; ca.stream = st;
            cudaLaunchAttribute aa[1];
            aa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            aa[0].val.programmaticStreamSerializationAllowed = 1;
            ca.attrs = aa; ca.numAttrs = a_pdl;
            cudaLaunchKernelEx(&ca, kA, t, spin, self_load, (const uint8_t*)l2buf);
          }
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = 148; cfg.blockDim = 64; cfg.dynamicSmemBytes = smem; cfg.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at; cfg.numAttrs = 1;
          if (woff + 148ull * 4 * 32768 > wbytes) woff = 0;
          cudaLaunchKernelEx(&cfg, kB, t, (const uint8_t*)(w + woff), mode);
          woff += 148ull * 4 * 32768;
          cudaStreamEndCapture(st, &graph);
          cudaGraphExec_t ge;
          cudaGraphInstantiate(&ge, graph, 0);
          cudaGraphLaunch(ge, st);
          cudaStreamSynchronize(st);
          cudaGraphExecDestroy(ge);
          cudaGraphDestroy(graph);
          std::vector<unsigned long long> h(8 + 148 * 8);
          cudaMemcpyAsync(h.data(), t, h.size() * 8, cudaMemcpyDeviceToHost, st);
          cudaStreamSynchronize(st);
          const double a_end = (double)h[0];
          for (int b = 0; b < 148; ++b) early += (double)h[8 + b * 8] < a_end;
          for (int c = 0; c < 6; ++c) {
            std::vector<double> v;
            for (int b = 0; b < 148; ++b) v.push_back(((double)h[8 + b * 8 + c] - a_end) / 1e3);
            std::sort(v.begin(), v.end());
            med[c] += v[74] / reps;
          }
        }
        printf("carveout %s ", carve ? "max-smem" : "default ");
        printf("A pdl %d grid %3d: B CTAs entered before A end %5.1f/148;  ", a_pdl, a_grid, early / 5.0);
        printf("A spin %5d ns  A loads %d  mode %d (%s): median us rel. A end: entry %7.2f  wait %6.2f  "
               "load0 %6.2f  load1 %6.2f  load2 %6.2f  load3 %6.2f\n",
               spin, self_load, mode, mode ? "loads before wait" : "wait then loads", med[0], med[1], med[2], med[3],
               med[4], med[5]);
      }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
