"""13B, long prompt: one profiled lookahead step (session API, eager launches)."""
import os, sys
sys.path.insert(0, ".")
os.environ.setdefault("LA_LAUNCH_MODE", "eager")
import numpy as np, torch
import paper_2402_02057_b200 as la
from paper_2402_02057_b200.models import PRESETS
plen = int(os.environ.get("PLEN", "3500"))
m = la.LlamaModel(PRESETS[os.environ.get("PRESET", "llama2-13b")], dtype="bf16", seed=0, max_context=plen + 400)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, m.vocab_size, plen)]
W, N, G = (int(x) for x in os.environ.get("WNG", "15,5,15").split(","))
cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=64)
st = la.start_session(m, prompt, cfg, la.SamplerSpec("greedy"))
for _ in range(3):
    la.lookahead_step(st)
torch.cuda.synchronize()
torch.cuda.profiler.start()
la.lookahead_step(st)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
