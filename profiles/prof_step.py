"""Short 7B lookahead decode for ncu: 64-token prompt, a few steps."""
import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2402_02057_b200 as la
from paper_2402_02057_b200.models import LLAMA2_7B
steps = int(os.environ.get("STEPS", "4"))
m = la.LlamaModel(LLAMA2_7B, dtype="bf16", seed=0, max_context=1024)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, 32000, 64)]
cfg = la.GenerationConfig(window=15, ngram=5, max_candidates=15, max_tokens=steps)
la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy"))
torch.cuda.synchronize()
t, met = la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy"))
print("steps", met.steps, m.last_stats)
