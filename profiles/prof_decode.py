"""cfg2-shaped decode for ncu (7B, W15 N5 G15, 512-token prompt): a warm-up
decode, then cudaProfilerStart and one profiled decode of STEPS lookahead
steps with eager launches (ncu cannot see kernels inside conditional graphs).
Use with `ncu --profile-from-start off`.  Inside the profiled region the
order is: prefill (4 chunks x 32 layers), then STEPS steps; per layer the
launches are la_gemm (qkv), la_qkv_epi, la_attn_fused, la_gemm (o),
la_resid_norm, la_gemm (gate/up), la_swiglu_epi, la_gemm (down),
la_resid_norm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LA_LAUNCH_MODE", "eager")
import numpy as np
import torch
import paper_2402_02057_b200 as la
from paper_2402_02057_b200.models import LLAMA2_7B

steps = int(os.environ.get("STEPS", "2"))
m = la.LlamaModel(LLAMA2_7B, dtype="bf16", seed=0, max_context=1088)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, 32000, 512)]
cfg = la.GenerationConfig(window=15, ngram=5, max_candidates=15, max_tokens=steps)
# SAMPLER=temperature: T=1, top_p=0.9 (adds the sampler's adjust / verify kernels)
spec = (la.SamplerSpec("temperature", temperature=1.0, top_p=0.9, seed=0)
        if os.environ.get("SAMPLER") == "temperature" else la.SamplerSpec("greedy"))
la.decode_lookahead(m, prompt, cfg, spec)
torch.cuda.synchronize()
torch.cuda.profiler.start()
la.decode_lookahead(m, prompt, cfg, spec)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
