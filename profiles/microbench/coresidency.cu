// Micro-test: does a PDL dependent grid's CTA become resident on an SM while the
// primary grid's CTA still runs there?  A: grid 148, smem SA, spins 30 us after
// triggering.  B: grid 148, smem SB, records entry time and SM id.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %smid;" : "=r"(s)); return s; }
#ifndef NR
#define NR 176
#endif
__global__ void __maxnreg__(200) kA(unsigned long long* t, int spin_ns) {
  extern __shared__ char sm[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned long long t0 = gt();
  if (threadIdx.x == 0) { t[blockIdx.x * 2] = t0; sm[0] = 1; }
  float r[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) r[i] = threadIdx.x * 0.001f + i;
  while (gt() - t0 < (unsigned long long)spin_ns) {
#pragma unroll
    for (int i = 0; i < NR; ++i) r[i] = r[i] * 1.0001f + r[(i + 1) % NR] * 1e-7f;
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < NR; ++i) acc += r[i];
  if (acc == 12345.f) sm[1] = 2;
  if (threadIdx.x == 0) t[blockIdx.x * 2 + 1] = gt();
}
#ifndef NRB
#define NRB 4
#endif
__global__ void __launch_bounds__(192, 1) kB(unsigned long long* t, unsigned* s) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) { t[blockIdx.x] = gt(); s[blockIdx.x] = smid(); sm[0] = 1; }
#ifdef TMEM
  __shared__ unsigned slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((unsigned)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef TMEM
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot) : "memory");
#endif
  float r[NRB];
#pragma unroll
  for (int i = 0; i < NRB; ++i) r[i] = threadIdx.x * 0.5f + i;
  for (int it = 0; it < 10; ++it)
#pragma unroll
    for (int i = 0; i < NRB; ++i) r[i] = r[i] * 1.0001f + r[(i + 3) % NRB];
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < NRB; ++i) acc += r[i];
  if (acc == 12345.f) sm[1] = 2;
}
int main(int argc, char** argv) {
  int sa = atoi(argv[1]) * 1024, sb = atoi(argv[2]) * 1024, carve = argc > 3 ? atoi(argv[3]) : -1;
  int sa_attr = argc > 4 ? atoi(argv[4]) * 1024 : sa;
  int sb_attr = argc > 5 ? atoi(argv[5]) * 1024 : sb;
  unsigned long long *ta, *tb; unsigned* sbm;
  cudaMalloc(&ta, 148 * 16); cudaMalloc(&tb, 148 * 8); cudaMalloc(&sbm, 148 * 4);
  cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, sa_attr);
  cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, sb_attr);
  if (carve >= 0) {
    cudaFuncSetAttribute(kA, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    cudaFuncSetAttribute(kB, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  }
  for (int rep = 0; rep < 3; ++rep) {
    kA<<<148, 256, sa>>>(ta, 30000);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = 148; cfg.blockDim = 192; cfg.dynamicSmemBytes = sb;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kB, tb, sbm);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  }
  unsigned long long a[296], b[148];
  cudaMemcpy(a, ta, sizeof(a), cudaMemcpyDeviceToHost); cudaMemcpy(b, tb, sizeof(b), cudaMemcpyDeviceToHost);
  unsigned long long a0 = ~0ull, aend = 0; for (int i = 0; i < 148; ++i) { a0 = a[2*i] < a0 ? a[2*i] : a0; aend = a[2*i+1] > aend ? a[2*i+1] : aend; }
  int early = 0; for (int i = 0; i < 148; ++i) early += b[i] < aend;
  double bmed; { unsigned long long v[148]; for (int i=0;i<148;++i) v[i]=b[i]; for(int i=0;i<148;++i)for(int j=i+1;j<148;++j)if(v[j]<v[i]){auto x=v[i];v[i]=v[j];v[j]=x;} bmed = ((double)v[74] - (double)a0) / 1e3; }
  printf("attrB %d KB attrA %d KB smemA %d KB smemB %d KB carve %d: A span %.1f us; B CTAs entered before A ended: %d/148; B median entry %.1f us after A start\n",
         sb_attr / 1024, sa_attr / 1024, sa / 1024, sb / 1024, carve, (aend - a0) / 1e3, early, bmed);
  return 0;
}
