// PDL chain A -> B -> C: when do C's CTAs start relative to A's end and B's span?
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void kA(unsigned long long* t, int spin) {   // plain primary
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned long long t0 = gt();
  while (gt() - t0 < (unsigned long long)spin) {}
  if (threadIdx.x == 0) atomicMax(&t[0], gt());          // A end
}
__global__ void kB(unsigned long long* t, int spin) {   // secondary of A, primary of C
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) atomicMin(&t[1], gt());          // B first entry
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t0 = gt();
  if (threadIdx.x == 0) atomicMin(&t[2], t0);            // B first wait return
  while (gt() - t0 < (unsigned long long)spin) {}
  if (threadIdx.x == 0) atomicMax(&t[3], gt());          // B end
}
__global__ void kC(unsigned long long* t) {
  if (threadIdx.x == 0) { atomicMin(&t[4], gt()); }
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
static void pdl_launch(void (*k)(unsigned long long*, int), unsigned long long* t, int spin, int grid) {
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = 256;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, t, spin);
}
int main() {
  unsigned long long* t; cudaMalloc(&t, 64);
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long init[5] = {0, ~0ull, ~0ull, 0, ~0ull};
    cudaMemcpy(t, init, sizeof(init), cudaMemcpyHostToDevice);
    kA<<<148, 256>>>(t, 10000);
    pdl_launch(kB, t, 20000, 128);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = 148; cfg.blockDim = 192;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kC, t);
    cudaDeviceSynchronize();
    unsigned long long h[5]; cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    double a_end = 0;
    printf("B entry %.1f  B wait-ret %.1f  B end %.1f  C first entry %.1f   (us rel. A end)\n",
           ((double)h[1] - (double)h[0]) / 1e3, ((double)h[2] - (double)h[0]) / 1e3,
           ((double)h[3] - (double)h[0]) / 1e3, ((double)h[4] - (double)h[0]) / 1e3);
  }
  return 0;
}
