"""In-graph timeline of one 7B lookahead step (LA_TIMELINE=1, LA_GEMM_TRACE=1).

    python profiles/timeline.py [greedy]

Prints, for the last complete decode step, every kernel's dependency-release
time (block 0 passing griddepcontrol.wait) and the gap to the next release
(= that kernel's share of the critical path), summed per kernel kind over the
step; then the per-CTA trace of the last layer's GEMMs (entry / wait returned /
last MMA issued / last piece written / exit, µs relative to the first entry).
"""
import ctypes as C
import os
import sys

os.environ.setdefault("LA_TIMELINE", "1")
os.environ.setdefault("LA_GEMM_TRACE", "1")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2402_02057_b200 as la  # noqa: E402
from paper_2402_02057_b200.models import PRESETS  # noqa: E402

preset = os.environ.get("PRESET", "llama2-7b")
cfgm = PRESETS[preset]
plen = int(os.environ.get("PLEN", "512"))
m = la.LlamaModel(cfgm, dtype="bf16", seed=0, max_context=plen + 128)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, m.vocab_size, plen)]
greedy = len(sys.argv) > 1 and sys.argv[1] == "greedy"
steps = int(os.environ.get("STEPS", "6"))
W, N, G = (int(x) for x in os.environ.get("WNG", "15,5,15").split(","))
cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=steps)
run = (lambda: la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), steps)) if greedy else \
      (lambda: la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy")))
run()
buf = (C.c_uint64 * (1 + 2 * 8192))()
m.lib.la_debug_read(m.engine(), 18, buf, C.sizeof(buf))   # warm-up records
C.memset(buf, 0, C.sizeof(buf))
# reset the device counter by running with a fresh read: the buffer is
# cumulative, so take the records of the LAST step only
run()
m.lib.la_debug_read(m.engine(), 18, buf, C.sizeof(buf))
n = min(int(buf[0]), 8192)
recs = [(int(buf[1 + 2 * i]), int(buf[2 + 2 * i])) for i in range(n)]
recs.sort()
d, H, KVH, F, V = cfgm.dim, cfgm.heads, cfgm.kv_heads, cfgm.ffn, cfgm.vocab


def name(sig):
    grid, block = sig >> 16, sig & 0xFFFF
    if grid == 1:
        return f"k[1x{block}]"
    if block == 192:
        return "gemm"
    if block == 256 and grid == (d // 128) * 16:
        return "resid_norm"
    if block == 128 and grid == (H + 2 * KVH) * 16:
        return "qkv_epi"
    if block == 128 and grid == (F // 64) * 8:
        return "swiglu_epi"
    if block == 128 and grid == ((V + 127) // 128) * 16:
        return "logits_epi"
    if block == 256:
        return f"attn[{grid}]"
    return f"k[{grid}x{block}]"


# step boundaries: the K1 build kernel (1 CTA) starts a step
starts = [i for i in range(len(recs) - 1) if name(recs[i][1]) == "k[1x256]" and name(recs[i + 1][1]) == "resid_norm"]
seg = recs
if len(starts) >= 3:
    seg = recs[starts[-3]:starts[-2] + 1]
print(f"records {n}; step kernels {len(seg) - 1}; step time {(seg[-1][0] - seg[0][0]) / 1e3:.1f} us")
tot = {}
gemm_i = 0
seq = []
for (t0, s), (t1, _) in zip(seg, seg[1:]):
    nm = name(s)
    if nm == "gemm":
        nm = ["gemm_qkv", "gemm_o", "gemm_gu", "gemm_down"][gemm_i % 4] if gemm_i < 4 * cfgm.layers else "gemm_head"
        gemm_i += 1
    tot[nm] = tot.get(nm, 0.0) + (t1 - t0) / 1e3
    seq.append((nm, (t1 - t0) / 1e3))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {k:16s} {v:9.1f} us")
print("step start:", " ".join(f"{k}:{v:.1f}" for k, v in seq[:12]))
print("layer 10:", " ".join(f"{k}:{v:.1f}" for k, v in seq[2 + 9 * 9: 2 + 10 * 9]))
print("step end:", " ".join(f"{k}:{v:.1f}" for k, v in seq[-8:]))
# per-CTA GEMM traces of the last launch of each kind
tr = (C.c_uint64 * (5 * 256 * 8))()
if m.lib.la_debug_read(m.engine(), 5, tr, C.sizeof(tr)) == 0:
    a = np.frombuffer(tr, dtype=np.uint64).reshape(5, 256, 8).astype(np.int64)
    if os.environ.get("DUMP"):
        np.save(os.environ["DUMP"], a)
        np.save(os.environ["DUMP"].replace(".npy", "_tl.npy"), np.array(recs, dtype=np.int64))
    # kernel-boundary latency: last CTA exit of each traced GEMM launch -> the
    # next kernel's dependency release (timeline record right after it)
    ts = np.array([t for t, _ in recs], dtype=np.int64)
    for k, nm in enumerate(["qkv", "o", "gu", "head", "down"]):
        x = a[k]
        x = x[x[:, 0] > 0]
        if not len(x):
            continue
        last_exit = x[:, 3].max()
        j = np.searchsorted(ts, last_exit)
        if j < len(ts):
            print(f"{nm:5s} last exit -> next release {(ts[j] - last_exit) / 1e3:.2f} us ({name(recs[j][1])}); "
                  f"median exit -> last exit {(last_exit - np.median(x[:, 3])) / 1e3:.2f} us")
    for k, nm in enumerate(["qkv", "o", "gu", "head", "down"]):
        x = a[k]
        ok = x[:, 0] > 0
        if not ok.any():
            continue
        x = x[ok]
        base = x[:, 0].min()
        def q(col):
            v = (x[:, col] - base) / 1e3
            return f"{np.min(v):6.2f}/{np.median(v):6.2f}/{np.max(v):6.2f}"
        print(f"{nm:5s} CTAs {len(x)} (min/med/max us) entry {q(0)} wait {q(1)} mma_done {q(2)} "
              f"pieces {q(4)} exit {q(3)}")
        if x[:, 6].min() > 0:
            print(f"      producer at final barrier {q(6)}  drain warp 3 {q(7)}")
# per-unit arrival trace (LA_GEMM_TRACE=2): when the MMA thread saw unit i's
# stage full, relative to the CTA's dependency-wait return
ut = (C.c_uint64 * (5 * 3 * 256 * 32))()
if os.environ.get("LA_GEMM_TRACE") == "2" and m.lib.la_debug_read(m.engine(), 20, ut, C.sizeof(ut)) == 0:
    u = np.frombuffer(ut, dtype=np.uint64).reshape(5, 3, 256, 32).astype(np.int64)
    for k, nm in enumerate(["qkv", "o", "gu", "head", "down"]):
        x = a[k]
        ok = x[:, 0] > 0
        g = int(ok.sum())
        wait = x[ok][:, 1][:, None]
        # the kernel indexes the slices by its own grid: [0][c], [1][c] = [0][grid + c], [2][c] = [0][2 grid + c]
        flat = u[k].reshape(-1, 32)
        full_t, prod_t, mma_t = flat[:g], flat[g:2 * g], flat[2 * g:3 * g]
        def rel(v):
            r = (v - wait) / 1e3
            r[v == 0] = np.nan
            return np.nanmedian(r, axis=0)
        pre = np.nanmedian((prod_t[:, 31] - wait[:, 0]) / 1e3)
        print(f"{nm:5s} preload issued {pre:.2f} us rel. wait; per unit (median us rel. wait):")
        print("   producer issue:", " ".join(f"{v:.2f}" for v in rel(prod_t)[:12]))
        print("   full passed:   ", " ".join(f"{v:.2f}" for v in rel(full_t)[:12]))
        print("   MMAs issued:   ", " ".join(f"{v:.2f}" for v in rel(mma_t)[:12]))
        dr = rel(mma_t)[24:32]
        mdone = np.nanmedian((x[ok][:, 2] - x[ok][:, 1]) / 1e3)
        pr = rel(prod_t)[24:30]
        print("   first drain: tile0 ld-issued/ld-done/stored, tile1 ...:", " ".join(f"{v:.2f}" for v in pr))
        print(f"   drain (warp 4) seg start/end: {' '.join(f'{v:.2f}' for v in dr)}  | MMA thread done {mdone:.2f}")
