"""W/N/G sweep (BASELINE configs[4]): per-step cost vs step compression.

    python bench_sweep.py [--preset llama2-70b] [--new 128] [--prompt 512]

For each (W, N) with G = W and (N-1)(W+G) <= 128 rows (the device row cap),
decodes the synthetic prompt with the random-init model and prints one JSON
line per point: ms per lookahead step, step compression S, tokens/s, the
per-step algorithmic bytes and HBM-roofline fraction, and the plain greedy
step for comparison.  Reuses bench.py's accounting.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="llama2-70b")
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--new", type=int, default=128)
    ap.add_argument("--windows", default="5,7,10,15,20,31")
    ap.add_argument("--ngrams", default="3,4,5,6")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2402_02057_b200 as la
    from paper_2402_02057_b200.models import PRESETS

    cfg = PRESETS[args.preset]
    model = la.LlamaModel(cfg, dtype="bf16", seed=0, max_context=args.prompt + args.new + 64)
    prompt = [int(t) for t in np.random.default_rng(0).integers(0, cfg.vocab, args.prompt)]
    hbm, src = bench._peaks()
    la.decode_autoregressive(model, prompt, la.SamplerSpec("greedy"), 16)
    ar = la.decode_autoregressive(model, prompt, la.SamplerSpec("greedy"), args.new)
    ar_ms = model.last_stats["decode_ms"] / model.last_stats["steps"]
    print(json.dumps({"preset": args.preset, "mode": "greedy", "ms_per_step": ar_ms,
                      "tokens_per_s": 1e3 / ar_ms,
                      "roofline_frac": bench.algorithmic_step_bytes(cfg, 1, args.prompt + args.new / 2)
                      / (ar_ms * 1e-3) / 1e9 / hbm}), flush=True)
    for N in [int(x) for x in args.ngrams.split(",")]:
        for W in [int(x) for x in args.windows.split(",")]:
            G = W
            if (N - 1) * (W + G) > 128:
                continue
            gc = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=args.new)
            la.decode_lookahead(model, prompt, gc, la.SamplerSpec("greedy"))   # warm (graph build)
            toks, met = la.decode_lookahead(model, prompt, gc, la.SamplerSpec("greedy"))
            st = model.last_stats
            ms = st["decode_ms"] / met.steps
            M = met.total_queries / met.steps
            b = bench.algorithmic_step_bytes(cfg, M, args.prompt + met.tokens_generated / 2)
            print(json.dumps({"preset": args.preset, "W": W, "N": N, "G": G, "steps": met.steps,
                              "S": met.compression, "mean_rows": M, "ms_per_step": ms,
                              "step_over_greedy": ms / ar_ms,
                              "tokens_per_s": met.tokens_generated / (st["decode_ms"] * 1e-3),
                              "roofline_frac": b / (ms * 1e-3) / 1e9 / hbm,
                              "tokens_equal_greedy": toks == ar[: len(toks)]}), flush=True)
    model.close()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
