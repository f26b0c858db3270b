// Does cp.async.bulk.prefetch.L2 stage weight bytes in L2 so that a later
// bulk-copy stream of the same bytes runs faster than from HBM?
//   A: cold stream of S MB (148 CTAs, 4 x 32 KB ring each)
//   B: prefetch S MB (one thread per CTA issues 32 KB prefetches), idle, stream
//   C: stream S MB twice back to back (second pass: whatever stayed in L2)
//   D: stream S MB while a concurrent 1-CTA kernel prefetches the NEXT S MB
//      (does a concurrent prefetcher slow the streamer?)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_prefetch l2_prefetch.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int kStages = 4, kChunk = 32768;

__global__ void __launch_bounds__(64, 1) stream_kernel(const uint8_t* buf, size_t per_cta, int policy,
                                                       unsigned long long* sink, int self_pf = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)kStages * kChunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (self_pf) {   // E: this CTA prefetches its own range first, then idles
    for (size_t o = 0; o < per_cta; o += kChunk)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(buf + blockIdx.x * per_cta + o), "r"(kChunk) : "memory");
    const unsigned long long t0 = gt();
    while (gt() - t0 < 40000ull) {}
  }
  atomicMin(&sink[1], gt());
  const uint8_t* src = buf + blockIdx.x * per_cta;
  const long n = (long)(per_cta / kChunk);
  uint64_t pol;
  if (policy) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  unsigned acc = 0;
  for (long i = 0; i < n + kStages; ++i) {
    if (i >= kStages) {
      const int s = (int)((i - kStages) % kStages);
      const uint32_t par = (uint32_t)(((i - kStages) / kStages) & 1);
      asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n"
                   ::"r"(su32(&full[s])), "r"(par) : "memory");
      acc += sm[(size_t)s * kChunk + (i & 127)];
    }
    if (i < n) {
      const int s = (int)(i % kStages);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kChunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                   ::"r"(su32(sm + (size_t)s * kChunk)), "l"(src + (size_t)i * kChunk), "r"(kChunk), "r"(su32(&full[s])), "l"(pol)
                   : "memory");
    }
  }
  if (acc == 0xffffffffu) sink[0] = acc;
  atomicMax(&sink[2], gt());
}

// every CTA (one thread) prefetches its own share, 32 KB per instruction
__global__ void prefetch_kernel(const uint8_t* buf, size_t per_cta) {
  if (threadIdx.x) return;
  const uint8_t* src = buf + blockIdx.x * per_cta;
  for (size_t o = 0; o < per_cta; o += kChunk)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + o), "r"(kChunk) : "memory");
}

// one CTA, 32 lanes, prefetching `bytes` (a concurrent helper)
__global__ void prefetch_one(const uint8_t* buf, size_t bytes) {
  for (size_t o = (size_t)threadIdx.x * kChunk; o < bytes; o += 32 * (size_t)kChunk)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(buf + o), "r"(kChunk) : "memory");
}

__global__ void spin_kernel(int ns) {
  const unsigned long long t0 = gt();
  while (gt() - t0 < (unsigned long long)ns) {}
}

int main() {
  const size_t total = 2ull << 30;
  uint8_t* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 1, total);
  const int G = 148;
  const size_t smem = (size_t)kStages * kChunk + 64;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStream_t s2;
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  size_t off = 0;
  auto fresh = [&](size_t bytes) {   // a region not touched recently (cycle the 2 GB)
    if (off + 2 * bytes > (1ull << 30)) off = 0;
    const uint8_t* p = buf + off;
    off += bytes;
    return p;
  };
  auto timed_stream = [&](const uint8_t* p, size_t bytes, int pol, int self_pf = 0) {
    const size_t per = bytes / G / kChunk * kChunk;
    unsigned long long h[3] = {0ull, ~0ull, 0ull};
    cudaMemcpy(sink, h, sizeof(h), cudaMemcpyHostToDevice);
    stream_kernel<<<G, 64, smem>>>(p, per, pol, sink, self_pf);
    cudaMemcpy(h, sink, sizeof(h), cudaMemcpyDeviceToHost);
    return (double)per * G / ((double)(h[2] - h[1]) * 1e-9) / 1e9;
  };
  // flush L2 with a large read
  auto flush = [&]() { stream_kernel<<<G, 64, smem>>>(buf + (1ull << 30), (512ull << 20) / G / kChunk * kChunk, 1, sink); cudaDeviceSynchronize(); };
  for (int mb : {16, 32, 64, 96}) {
    const size_t bytes = (size_t)mb << 20;
    const size_t per = bytes / G / kChunk * kChunk;
    for (int pol = 0; pol < 2; ++pol) {
      double a = 0, b = 0, c1 = 0, c2 = 0, d = 0, e = 0;
      for (int rep = 0; rep < 3; ++rep) {
        flush();
        a += timed_stream(fresh(bytes), bytes, pol);
        flush();
        const uint8_t* p = fresh(bytes);
        prefetch_kernel<<<G, 32>>>(p, per);
        spin_kernel<<<1, 32>>>(40000);
        cudaDeviceSynchronize();
        b += timed_stream(p, bytes, pol);
        flush();
        p = fresh(bytes);
        c1 += timed_stream(p, bytes, pol);
        c2 += timed_stream(p, bytes, pol);
        flush();
        p = fresh(2 * bytes);
        spin_kernel<<<1, 32>>>(1000);
        prefetch_one<<<1, 32, 0, s2>>>(p + bytes, bytes);
        d += timed_stream(p, bytes, pol);
        cudaDeviceSynchronize();
        flush();
        e += timed_stream(fresh(bytes), bytes, pol, 1);
      }
      printf("%3d MB  %s  cold %7.0f GB/s  prefetched %7.0f  read1 %7.0f read2 %7.0f  cold+concurrent-pf %7.0f  self-prefetched %7.0f\n", mb,
             pol ? "evict_first " : "evict_normal", a / 3, b / 3, c1 / 3, c2 / 3, d / 3, e / 3);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
