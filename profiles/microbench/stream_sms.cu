// HBM streaming rate vs the number of SMs that stream: each CTA pulls its
// contiguous share of a 2 GiB buffer through a ring of `stages` x `chunk`
// bytes with 1-D bulk copies (cp.async.bulk, one mbarrier per slot) and does
// nothing else -- the weight-streaming producer of la_gemm_kernel without
// the MMAs.  Question: can fewer than 148 SMs saturate HBM (so a GEMM with
// fewer, whole tiles per CTA -- no split-K reduction -- loses nothing)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_sms stream_sms.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) stream_kernel(const uint8_t* buf, size_t per_cta, int stages,
                                                       int chunk, unsigned long long* sink, const uint8_t* bsrc = nullptr,
                                                       int bbytes = 0, int consume_ns = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * (chunk + bbytes));
  uint8_t* sb = sm + (size_t)stages * chunk;   // per-stage B slots (GEMM step rows; L2-resident source)
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* src = buf + blockIdx.x * per_cta;
  const long n = (long)(per_cta / chunk);
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  unsigned acc = 0;
  for (long i = 0; i < n + stages; ++i) {
    if (i >= stages) {   // consume chunk i - stages
      const int s = (int)((i - stages) % stages);
      const uint32_t par = (uint32_t)(((i - stages) / stages) & 1);
      asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n"
                   ::"r"(su32(&full[s])), "r"(par) : "memory");
      acc += sm[(size_t)s * chunk + (i & 127)];
      if (consume_ns) {   // the MMA's turnaround before the slot is released
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
        do { asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)consume_ns);
      }
    }
    if (i < n) {
      const int s = (int)(i % stages);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk + bbytes) : "memory");
      if (bbytes)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sb + (size_t)s * bbytes)), "l"(bsrc + (size_t)(i & 63) * 16384), "r"(bbytes), "r"(su32(&full[s]))
                     : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                   ::"r"(su32(sm + (size_t)s * chunk)), "l"(src + (size_t)i * chunk), "r"(chunk), "r"(su32(&full[s])), "l"(pol)
                   : "memory");
    }
  }
  if (acc == 0xffffffffu) sink[0] = acc;
}

int main() {
  const size_t total = 2ull << 30;
  uint8_t* buf;
  uint8_t* bsrc;
  unsigned long long* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&bsrc, 64 * 16384);
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 1, total);
  cudaMemset(bsrc, 1, 64 * 16384);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // {stages, chunk, B bytes per stage, consume ns, SMs}
  const int cfg[][5] = {{6, 32768, 0, 0, 148}, {4, 49152, 0, 0, 148}, {12, 16384, 0, 0, 128},
                        {4, 32768, 8192, 250, 148}, {5, 32768, 8192, 250, 148}, {6, 32768, 2048, 250, 148},
                        {4, 32768, 16384, 250, 148}, {2, 65536, 16384, 400, 148}, {3, 65536, 0, 400, 148},
                        {4, 32768, 8192, 0, 148}, {5, 32768, 8192, 0, 148}, {4, 49152, 8192, 300, 148},
                        {3, 65536, 8192, 400, 148}, {4, 32768, 8192, 250, 96}, {5, 32768, 8192, 250, 96},
                        {4, 32768, 8192, 250, 128}};
  for (auto& c : cfg) {
    const int stages = c[0], chunk = c[1], bb = c[2], cns = c[3], g = c[4];
    const size_t smem = (size_t)stages * (chunk + bb) + 8 * stages;
    if (smem > 227 * 1024) { printf("skip %d x %d\n", stages, chunk); continue; }
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const size_t per = (total / g) / chunk * chunk;
    for (int w = 0; w < 2; ++w) stream_kernel<<<g, 64, smem>>>(buf, per, stages, chunk, sink, bsrc, bb, cns);
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      stream_kernel<<<g, 64, smem>>>(buf, per, stages, chunk, sink, bsrc, bb, cns);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    const double gbs = (double)per * g / (best * 1e-3) / 1e9;
    printf("stages %2d chunk %3d KB  B %5d B  consume %3d ns  ring %4d KB  SMs %3d  %7.1f GB/s  (%.1f per SM)\n",
           stages, chunk / 1024, bb, cns, (int)(smem / 1024), g, gbs, gbs / g);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
