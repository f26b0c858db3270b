"""Per-phase cycles of the fp32 single-CTA decode (cfg1, LA_TINY_PROF=1).

    python profiles/tiny_prof.py

cfg1 workload (the reference TinyTransformer, W5 N3 G5, 32-token prompt, 128
new tokens): lookahead and plain greedy; prints us per step per phase
(cycles / SM clock) -- K1 build, forward, argmax scatter, sampler, K10 finish,
KV commit, loop overhead."""
import ctypes as C
import os
import sys

os.environ.setdefault("LA_TINY_PROF", "1")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2402_02057_b200 as la  # noqa: E402

mhz = float(os.environ.get("SM_MHZ", "1965"))
m = la.TinyTransformer(0, 256, 16, 2, 2, max_context=512, device=0)
prompt = [int(t) for t in np.random.default_rng(1234).integers(0, 256, 32)]
cfg = la.GenerationConfig(window=5, ngram=3, max_candidates=5, max_tokens=128)
names = ["build", "forward", "amax", "sampler", "finish", "commit", "steps", "loop",
         "f.embed", "f.norm1", "f.qkv", "f.attn", "f.o", "f.norm2+mlp1", "f.mlp2", "f.head"]
for label, run in (("lookahead", lambda: la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy"))),
                   ("greedy", lambda: la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), 128))):
    run()
    run()
    buf = (C.c_uint64 * 16)()
    m.lib.la_debug_read(m.engine(), 21, buf, C.sizeof(buf))
    steps = max(1, int(buf[6]))
    tot = sum(int(buf[i]) for i in range(16) if i != 6)
    print(f"== {label}: {steps} steps, {tot / steps / mhz:.1f} us per step, decode_ms {m.last_stats['decode_ms']:.3f}")
    for i, n in enumerate(names):
        if i != 6:
            print(f"  {n:8s} {int(buf[i]) / steps / mhz:8.2f} us/step")
m.close()
