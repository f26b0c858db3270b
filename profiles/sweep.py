"""W / N / G sweep of the lookahead step (SURVEY 8(d) cfg5 grid, G = W) on one GPU.

    PRESET=llama2-70b TOK=128 python profiles/sweep.py > profiles/<round>_sweep_70b.jsonl

One JSON line per configuration: step time, mean rows per step, the step's
HBM-roofline fraction B(M, ctx) / t / peak, and the ratio to a plain greedy
step measured first on the same model.  Configurations whose step would
exceed the device's 128 query rows ((N-1)(W+G) > 128) are reported as skipped.
Synthetic workload: random-init bf16 weights, prompt default_rng(0), 512 tokens.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2402_02057_b200 as la  # noqa: E402
from paper_2402_02057_b200.models import PRESETS  # noqa: E402
import bench  # noqa: E402

preset = os.environ.get("PRESET", "llama2-7b")
tok = int(os.environ.get("TOK", "128"))
cfg = PRESETS[preset]
m = la.LlamaModel(cfg, dtype="bf16", seed=0, max_context=512 + tok + 64)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, cfg.vocab, 512)]
hbm, _ = bench._peaks()

la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), tok)
la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), tok)
g_ms = m.last_stats["decode_ms"] / m.last_stats["steps"]
g_bytes = bench.algorithmic_step_bytes(cfg, 1, 512 + tok / 2)
print(json.dumps({"preset": preset, "mode": "greedy", "ms_per_step": g_ms, "tokens_per_s": 1e3 / g_ms,
                  "roofline_frac": g_bytes / (g_ms * 1e-3) / 1e9 / hbm}), flush=True)
for W in (5, 7, 10, 15, 20, 31):
    for N in (3, 4, 5, 6):
        G = W
        row = {"preset": preset, "W": W, "N": N, "G": G}
        if (N - 1) * (W + G) > 128:
            row["skipped"] = "more than 128 query rows per step"
            print(json.dumps(row), flush=True)
            continue
        gc = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=tok)
        la.decode_lookahead(m, prompt, gc, la.SamplerSpec("greedy"))
        toks, met = la.decode_lookahead(m, prompt, gc, la.SamplerSpec("greedy"))
        ms = m.last_stats["decode_ms"] / met.steps
        rows = met.total_queries / met.steps
        b = bench.algorithmic_step_bytes(cfg, rows, 512 + tok / 2)
        row.update({"steps": met.steps, "S": met.compression, "mean_rows": rows, "ms_per_step": ms,
                    "step_over_greedy": ms / g_ms, "tokens_per_s": len(toks) / (m.last_stats["decode_ms"] / 1e3),
                    "roofline_frac": b / (ms * 1e-3) / 1e9 / hbm})
        print(json.dumps(row), flush=True)
