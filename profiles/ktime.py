"""Per-kernel warm timings (LA_KTIME, eager launches) of LA and greedy steps under env settings."""
import os, subprocess, sys
code = r'''
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2402_02057_b200 as la
from paper_2402_02057_b200.models import PRESETS
plen = int(os.environ.get("PLEN", "512"))
m = la.LlamaModel(PRESETS[os.environ.get("PRESET", "llama2-7b")], dtype="bf16", seed=0, max_context=plen + 400)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, m.vocab_size, plen)]
cfg = la.GenerationConfig(window=15, ngram=5, max_candidates=15, max_tokens=int(os.environ.get("TOK", "32")))
if os.environ.get("MODE", "la") == "la":
    t, met = la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy"))
    print("ROWS", met.total_queries / met.steps, file=sys.stderr)
else:
    la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), int(os.environ.get("TOK", "32")))
'''
for setting in sys.argv[1:]:
    env = dict(os.environ, LA_KTIME="1", LA_LAUNCH_MODE="eager")
    for kv in setting.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1)
            env[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    lines = [l for l in out.stderr.splitlines() if "attn" in l or "ROWS" in l or "total" in l or "gemm_gu" in l]
    print(setting, "\n  " + "\n  ".join(lines[-6:]) if lines else out.stderr[-800:], flush=True)
