// Step kernels of the temperature sampler (bf16 multi-kernel path).  Logic in
// la_sample.cuh, shared with the fp32 single-CTA decode megakernel.
//
// Per step, after the forward has dumped the rows' logits:
//   la_sample_adjust_kernel   one CTA per row verification may read (row 0 +
//                             every branch row): softmax -> adjusted
//                             distribution (sampling.py:22-66), fp64
//   la_sample_verify_kernel   one CTA: verify_sample (verification.py:74-118)
//                             with the session generator
// K10 (la_step_finish) then consumes d.accepted / d.k / d.winner and draws
// the window refills from the same generator.
#include "la_kernels.h"
#include "la_sample.cuh"

__global__ void __launch_bounds__(1024) la_sample_adjust_kernel(DevDecode* dp) {
  LA_PDL_ENTRY();
  __shared__ LaSampleSmem sm;
  DevDecode& d = *dp;
  if (d.done || d.degenerate) return;
  const int j = blockIdx.x;
  if (j >= la_sample_rows(d)) return;
  const int row = la_sample_row(d, j);
  if (!la_adjust_row(d.logits + (size_t)row * d.V, d.V, d.temperature, d.top_k, d.top_p,
                     d.adj + (size_t)j * d.V, sm) &&
      threadIdx.x == 0)
    d.degenerate = 1;
}

// bf16 path: each row is adjusted by one thread-block cluster of
// LA_ADJ_CLUSTER CTAs, each owning a contiguous vocabulary slice -- with no
// candidates only row 0 exists, and one CTA would leave the GPU idle through
// the ALU-bound radix passes.  Only d.done gates the launch: d.degenerate may
// be raised by another cluster of this grid while it runs.
__global__ void __cluster_dims__(LA_ADJ_CLUSTER, 1, 1) __launch_bounds__(LA_ADJ_THREADS)
    la_sample_adjust_cluster_kernel(DevDecode* dp) {
  LA_PDL_ENTRY();
  __shared__ LaSampleSmem sm;
  DevDecode& d = *dp;
  if (d.done) return;
  const int j = blockIdx.x / LA_ADJ_CLUSTER;
  if (j >= la_sample_rows(d)) return;   // uniform over the cluster
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int V = d.V;
  LaClusterScope sc{(int)((long)V * rank / LA_ADJ_CLUSTER),
                    (int)((long)V * (rank + 1) / LA_ADJ_CLUSTER), rank, LA_ADJ_CLUSTER};
  const bool ok = la_adjust_row_s(d.logits + (size_t)la_sample_row(d, j) * V, sc, V, d.temperature,
                                  d.top_k, d.top_p, d.adj + (size_t)j * V, sm);
  sc.finish();
  if (!ok && rank == 0 && threadIdx.x == 0) d.degenerate = 1;
}

__global__ void __launch_bounds__(1024) la_sample_verify_kernel(DevDecode* dp) {
  LA_PDL_ENTRY();
  __shared__ LaSampleSmem sm;
  DevDecode& d = *dp;
  if (d.done || d.degenerate) return;
  la_verify_sample(d, sm);
}

// parity hook: adjusted_distribution of given probability rows (in place)
__global__ void __launch_bounds__(1024) la_adjust_probs_kernel(double* rows, int V, double temperature,
                                                               int top_k, double top_p, int* degenerate) {
  __shared__ LaSampleSmem sm;
  if (!la_adjust_row(nullptr, V, temperature, top_k, top_p, rows + (size_t)blockIdx.x * V, sm) &&
      threadIdx.x == 0)
    degenerate[blockIdx.x] = 1;
}

// parity hook: the cluster-scope row function on given probability rows
__global__ void __cluster_dims__(LA_ADJ_CLUSTER, 1, 1) __launch_bounds__(LA_ADJ_THREADS)
    la_adjust_probs_cluster_kernel(double* rows, int V, double temperature, int top_k, double top_p,
                                   int* degenerate) {
  __shared__ LaSampleSmem sm;
  const int j = blockIdx.x / LA_ADJ_CLUSTER;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  LaClusterScope sc{(int)((long)V * rank / LA_ADJ_CLUSTER),
                    (int)((long)V * (rank + 1) / LA_ADJ_CLUSTER), rank, LA_ADJ_CLUSTER};
  const bool ok = la_adjust_row_s(nullptr, sc, V, temperature, top_k, top_p, rows + (size_t)j * V, sm);
  sc.finish();
  if (!ok && rank == 0 && threadIdx.x == 0) degenerate[j] = 1;
}

// parity hook: verify_sample on caller distributions already in d.adj
__global__ void __launch_bounds__(1024) la_verify_hook_kernel(DevDecode* dp) {
  __shared__ LaSampleSmem sm;
  la_verify_sample(*dp, sm);
}

LA_TL_DEFINE_SETTER(sample)
