import os, sys
sys.path.insert(0, ".")
os.environ["LA_KTIME"] = "1"; os.environ["LA_LAUNCH_MODE"] = "eager"
import numpy as np
import paper_2402_02057_b200 as la
from paper_2402_02057_b200.models import PRESETS
m = la.LlamaModel(PRESETS["llama2-70b"], dtype="bf16", seed=0, max_context=1200)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, m.vocab_size, 512)]
cfg = la.GenerationConfig(window=15, ngram=5, max_candidates=15, max_tokens=16)
print("=== LA", file=sys.stderr)
la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy"))
print("=== GREEDY", file=sys.stderr)
la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), 16)
