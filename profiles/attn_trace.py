"""Per-CTA phase stamps of the fused attention kernel (LA_ATTN_TRACE=1).

    python profiles/attn_trace.py [greedy]

Runs a 7B-shaped (PRESET) decode in the graph loop, then reads the stamps of
the LAST attention launch (last layer of the last step): 0 entry, 1 dependency
wait returned, 2 q / mask ready (tile loop starts), 3 first K/V tile landed,
4 all tiles done, 5 every chunk CTA of the group arrived, 6 merge written.
Prints min / median / max per phase in us relative to the first wait return,
split by unit kind (prefix chunk vs step block).
"""
import ctypes as C
import os
import sys

os.environ.setdefault("LA_ATTN_TRACE", "1")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2402_02057_b200 as la  # noqa: E402
from paper_2402_02057_b200.models import PRESETS  # noqa: E402

cfgm = PRESETS[os.environ.get("PRESET", "llama2-7b")]
plen = int(os.environ.get("PLEN", "512"))
m = la.LlamaModel(cfgm, dtype="bf16", seed=0, max_context=plen + 128)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, m.vocab_size, plen)]
greedy = len(sys.argv) > 1 and sys.argv[1] == "greedy"
steps = int(os.environ.get("STEPS", "8"))
W, N, G = (int(x) for x in os.environ.get("WNG", "15,5,15").split(","))
cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=steps)
for _ in range(2):
    if greedy:
        la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), steps)
    else:
        la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy"))
buf = (C.c_uint64 * (8 * 4096))()
rc = m.lib.la_debug_read(m.engine(), 17, buf, C.sizeof(buf))
if rc != 0:
    sys.exit(f"la_debug_read(17) failed: {rc}")
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8).astype(np.float64)
a = a[a[:, 1] > 0]
S1 = int(os.environ.get("ATTN_UNITS", "4"))   # S + 1 chunk units per (KV head, row block)
t0 = a[:, 1].min()
names = ["entry", "wait", "q/mask", "tile0", "tiles", "arrived", "merged"]
for kind, sel in (("prefix", np.arange(len(a)) % S1 != S1 - 1), ("step", np.arange(len(a)) % S1 == S1 - 1)):
    b = a[sel]
    print(f"== {kind} units: {len(b)}")
    for k, n in enumerate(names):
        v = (b[:, k] - t0) / 1e3
        v = v[b[:, k] > 0]
        if len(v):
            print(f"  {n:8s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
