// mma.sync (HMMA) tile rate of the decode attention's inner loop versus warps
// per SM sub-partition: each warp runs `tiles` iterations of one 64-key tile
// for 16 query rows -- QK^T (8 key blocks x 8 dim steps of m16n8k16, fragments
// by ldmatrix from smem), an exp2 per score, PV (16 dim blocks x 4 key steps,
// V fragments by ldmatrix.trans) -- with no global traffic.  The question it
// answers: is the attention tile HMMA-latency-bound per warp (more warps per
// sub-partition => proportionally more tiles per second) or pipe-bound?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o hmma_warps hmma_warps.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void ldsm_x4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}

__global__ void kern(int tiles, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];   // one 64-key K | V tile (32 KB)
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t qf[8][4];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk)
#pragma unroll
    for (int j = 0; j < 4; ++j) qf[kk][j] = 0x3c003c00u ^ (lane * 7 + kk + j);
  float o[16][4] = {};
  float m = -1e30f, l = 0.f;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
#pragma unroll 1
  for (int t = 0; t < tiles; ++t) {
    float s[8][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) s[nb][0] = s[nb][1] = s[nb][2] = s[nb][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int nb = 0; nb < 8; nb += 2) {
        uint32_t b[4];
        const int row = nb * 8 + (lane & 7) + ((lane >> 4) << 3), ch = kk * 2 + ((lane >> 3) & 1);
        ldsm_x4(b, base + row * 256 + ((ch ^ (row & 7)) << 4));
        mma16816(s[nb], qf[kk], b);
        mma16816(s[nb + 1], qf[kk], b + 2);
      }
    float mx = m;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) mx = fmaxf(mx, fmaxf(fmaxf(s[nb][0], s[nb][1]), fmaxf(s[nb][2], s[nb][3])));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float corr = exp2f(m - mx);
    m = mx;
    l *= corr;
    uint32_t p[4][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      const float e0 = exp2f(s[nb][0] - mx), e1 = exp2f(s[nb][1] - mx), e2 = exp2f(s[nb][2] - mx),
                  e3 = exp2f(s[nb][3] - mx);
      l += e0 + e1 + e2 + e3;
      p[nb >> 1][(nb & 1) * 2] = pack(e0, e1);
      p[nb >> 1][(nb & 1) * 2 + 1] = pack(e2, e3);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) { o[i][0] *= corr; o[i][1] *= corr; o[i][2] *= corr; o[i][3] *= corr; }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
      for (int db = 0; db < 16; db += 2) {
        uint32_t b[4];
        const int row = ks * 16 + (lane & 15), ch = db + (lane >> 4);
        ldsm_x4_t(b, base + 16384 + row * 256 + ((ch ^ (row & 7)) << 4));
        mma16816(o[db], p[ks], b);
        mma16816(o[db + 1], p[ks], b + 2);
      }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
  float acc = l;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc += o[i][0] + o[i][1] + o[i][2] + o[i][3];
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  if (lane == 0) out[blockIdx.x * 64 + (threadIdx.x >> 5)] = t1 - t0;
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 64 * 8);
  cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  const int tiles = 200;
  for (int warps : {4, 8, 12}) {
    kern<<<148, warps * 32, 32768>>>(tiles, d, sink);
    kern<<<148, warps * 32, 32768>>>(tiles, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    static unsigned long long h[148 * 64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int b = 0; b < 148; ++b)
      for (int w = 0; w < warps; ++w) mx = h[b * 64 + w] > mx ? h[b * 64 + w] : mx;
    const double cyc = (double)mx / tiles;
    printf("warps/SM %2d (%d per sub-partition): %7.0f cycles per tile per warp, %6.0f cycles per tile per SM"
           " (%.2f us per tile-warp at 1.9 GHz)\n",
           warps, warps / 4, cyc, cyc / warps, cyc / 1900.0);
  }
  return 0;
}
