// Kernel declarations shared between translation units.
#pragma once
#include "la_common.cuh"

__global__ void la_pool_seed_kernel(DevDecode* dp, const int* grams, int n, int log_from);
__global__ void la_step_build_kernel(DevDecode* dp, FwdPlan* P);
__global__ void la_pool_test_kernel(DevPool pool, const int* grams, int n_grams, int batch,
                                    const int* leads, int n_leads, int limit, int* out, int* counts,
                                    int* lens, int* overflow);
__global__ void la_step_finish_kernel(DevDecode* dp);
__global__ void la_scatter_amax_kernel(DevDecode* dp, const FwdPlan* P, const int* row_amax);
__global__ void la_merge_amax_kernel(DevDecode* dp, const int* gathered, int world);
__global__ void la_kv_commit_kernel(const DevDecode* dp, uint8_t* kc, uint8_t* vc, int layers,
                                    int slots, int row_bytes);
__global__ void la_kv_pack_kernel(const DevDecode* dp, const uint8_t* kc, const uint8_t* vc,
                                  uint8_t* send, int layers, int slots, int row_bytes);
__global__ void la_kv_unpack_kernel(const DevDecode* dp, const uint8_t* gathered, size_t seg,
                                    uint8_t* kc, uint8_t* vc, int layers, int slots,
                                    int row_bytes);
__global__ void la_sample_adjust_kernel(DevDecode* dp);
__global__ void la_sample_verify_kernel(DevDecode* dp);
#define LA_ADJ_CLUSTER 8      // CTAs per adjusted row (bf16 path)
#define LA_ADJ_THREADS 512
__global__ void la_sample_adjust_cluster_kernel(DevDecode* dp);
__global__ void la_adjust_probs_cluster_kernel(double* rows, int V, double temperature, int top_k,
                                               double top_p, int* degenerate);
__global__ void la_adjust_probs_kernel(double* rows, int V, double temperature, int top_k,
                                       double top_p, int* degenerate);
__global__ void la_verify_hook_kernel(DevDecode* dp);
