import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2402_02057_b200 as la
from oracle.model_oracle import llama_random_weights
sms = torch.cuda.get_device_properties(0).multi_processor_count
ffn = 64 * (sms + 13)
cfg = dict(dim=256, layers=2, heads=2, kv_heads=2, head_dim=128, ffn=ffn, vocab=1000, rope_theta=10000.0, eps=1e-5)
w = llama_random_weights(cfg, seed=2, std=None)
lc = la.LlamaConfig(dim=256, layers=2, heads=2, kv_heads=2, ffn=ffn, vocab=1000, head_dim=128)
prompt = [int(t) for t in np.random.default_rng(21).integers(0, 1000, 120)]
m = la.LlamaModel(lc, dtype="bf16", weights=w, max_context=512)
ar = la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), 32)
toks, met = la.decode_lookahead(m, prompt, la.GenerationConfig(window=15, ngram=5, max_candidates=15, max_tokens=32), la.SamplerSpec("greedy"))
i = next((i for i in range(32) if ar[i] != toks[i]), None)
print("first diff", i, "steps", met.steps, "accepted per step", [len(s) for s in getattr(met, "accepted_per_step", [])][:5])
if i is not None:
    seq = prompt + ar[:i]
    lg = m.logits(seq[:-1], la.chain_layout(seq[-1], []))[0]
    srt = np.sort(lg)
    print("greedy token", ar[i], "lookahead token", toks[i], "top2", srt[-1], srt[-2], "rel margin", (srt[-1] - srt[-2]) / np.abs(lg).max(),
          "logit(greedy)", lg[ar[i]], "logit(lookahead)", lg[toks[i]])
m.close()
