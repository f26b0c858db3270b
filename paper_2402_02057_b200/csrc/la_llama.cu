// bf16 Llama path (placeholder until the tcgen05 kernels land).
#include "la_engine.h"
int llama_create(la_engine*) { la_set_error("bf16 path not built yet"); return LA_ERR_UNSUPPORTED; }
void llama_destroy(la_engine*) {}
int llama_prefill(la_engine*, const int*, int, cudaStream_t) { return LA_ERR_UNSUPPORTED; }
int llama_decode_loop(la_engine*, cudaStream_t, int*) { return LA_ERR_UNSUPPORTED; }
int llama_forward_plan(la_engine*, float*, cudaStream_t) { return LA_ERR_UNSUPPORTED; }
int llama_step_forward(la_engine*, cudaStream_t) { return LA_ERR_UNSUPPORTED; }
