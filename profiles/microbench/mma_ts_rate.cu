// tcgen05.mma issue/execution rate with the A operand in shared memory (SS)
// versus in tensor memory (TS), no memory traffic: one thread issues `units`
// x (tiles x 4 k-steps) MMAs of M=128, N=n, K=16 (bf16) with a commit at the
// end, timed by globaltimer.  The question it answers: is the per-MMA cost of
// the small-N decode shapes the SMEM read of A?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2402_02057_b200/csrc \
//        -o mma_ts_rate mma_ts_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "la_ptx.cuh"

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}

__global__ void __launch_bounds__(128, 1) kern(int units, int n, int tiles, int ts, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
  uint8_t* sA = sm;                    // 4 x 16 KB weight tiles
  uint8_t* sB = sm + 4 * 16384;        // 32 KB step rows
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 6 * 16384);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  for (int i = threadIdx.x; i < 6 * 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::umma_idesc_bf16(128, (uint32_t)n);
    const uint32_t a0 = ptx::smem_u32(sA), b0 = ptx::smem_u32(sB);
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (int u = 0; u < units; ++u) {
      for (int tt = 0; tt < tiles; ++tt)
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t d = tmem + tt * 128;
          const uint64_t bd = ptx::umma_desc_sw128(b0 + kk * 32);
          if (ts)   // A: 128 lanes x (K = 16 bf16 = 8 columns) per k-step, at column 256 + 32 tt + 8 kk
            umma_ts(d, tmem + 256 + 32 * tt + 8 * kk, bd, idesc, (u > 0 || kk > 0) ? 1u : 0u);
          else
            ptx::umma_bf16(d, ptx::umma_desc_sw128(a0 + tt * 16384 + kk * 32), bd, idesc, (u > 0 || kk > 0) ? 1u : 0u);
        }
    }
    ptx::umma_commit(&bar[0]);
    ptx::mbar_wait(&bar[0], 0);
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 6 * 16384 + 2048;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int units = 256;
  for (int ts = 0; ts < 2; ++ts)
    for (int tiles : {1, 2})
      for (int n : {16, 64, 128}) {
        kern<<<148, 128, smem>>>(units, n, tiles, ts, d);
        kern<<<148, 128, smem>>>(units, n, tiles, ts, d);
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%s tiles %d N %3d: %7.1f cycles per MMA (M=128, K=16)\n", ts ? "A in TMEM" : "A in SMEM", tiles, n,
               mx * 1.965 / (units * tiles * 4.0));
      }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
