"""A/B step timing under env settings (graph-loop decode, the bench's launch mode).

    python profiles/ab.py "" "LA_NPF=40" "LA_NPF=40,20" ...

Each setting (comma-separated K=V pairs; a bare label is allowed) runs in its
own process: 7B-shaped (PRESET), W15 N5 G15, PLEN-token prompt, TOK new
tokens; prints ms per lookahead step and per greedy step (device decode time
from the engine's CUDA events, warm run).  Settings are run ROUNDS times in
interleaved order so box drift hits every setting alike.
"""
import json
import os
import subprocess
import sys

code = r'''
import os, sys, json
sys.path.insert(0, ".")
import numpy as np
import paper_2402_02057_b200 as la
from paper_2402_02057_b200.models import PRESETS
plen = int(os.environ.get("PLEN", "512")); tok = int(os.environ.get("TOK", "256"))
m = la.LlamaModel(PRESETS[os.environ.get("PRESET", "llama2-7b")], dtype="bf16", seed=0, max_context=plen + tok + 64)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, m.vocab_size, plen)]
W, N, G = (int(x) for x in os.environ.get("WNG", "15,5,15").split(","))
cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=tok)
out = {}
for rep in range(2):
    t, met = la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy"))
la_ms = m.last_stats["decode_ms"] / met.steps
for rep in range(2):
    a = la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), 128)
ar_ms = m.last_stats["decode_ms"] / m.last_stats["steps"]
print("RESULT " + json.dumps({"la": la_ms, "ar": ar_ms, "eq": a == t[:128], "rows": met.total_queries / met.steps}))
'''


def run(setting):
    env = dict(os.environ)
    for kv in setting.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1)
            env[k] = v.replace(";", ",")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    for line in out.stdout.splitlines():
        if line.startswith("RESULT "):
            return json.loads(line[7:])
    return {"err": (out.stderr or out.stdout)[-600:]}


if __name__ == "__main__":
    settings = sys.argv[1:] or [""]
    rounds = int(os.environ.get("ROUNDS", "1"))
    res = {s: [] for s in settings}
    for r in range(rounds):
        for s in settings:
            res[s].append(run(s))
            print(f"[{r}] {s or 'default'}: {res[s][-1]}", flush=True)
    print("== summary (min over rounds)")
    for s, rs in res.items():
        ok = [x for x in rs if "la" in x]
        if ok:
            print(f"{s or 'default':40s} la {min(x['la'] for x in ok):.4f} ms  ar {min(x['ar'] for x in ok):.4f} ms  "
                  f"eq {all(x['eq'] for x in ok)}")
        else:
            print(f"{s or 'default':40s} FAILED {rs[-1]}")
