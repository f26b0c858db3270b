"""Generate golden vectors from the REFERENCE implementation (test infra only).

Run in the build container (the only place ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

It imports the unmodified reference package from
``/root/reference/pkg/src`` and writes small JSON / NPZ fixtures into
``tests/golden/``.  Those fixtures travel to the GPU box; the reference does
not.  Every fixture records which reference entry point produced it.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import lookahead  # noqa: F401  (the reference package)
    return lookahead


def _dump(name, obj):
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / name).write_text(json.dumps(obj, sort_keys=True, separators=(",", ":")) + "\n")


def _layout_record(L):
    return {
        "tokens": [q.token for q in L.queries],
        "rel": [q.rel_pos for q in L.queries],
        "visible": [sorted(q.visible) for q in L.queries],
        "generators": list(L.generators),
        "branches": [[r.start, r.stop] for r in L.branch_slices],
    }


def gen_layouts(la):
    rng = np.random.default_rng(2024)
    cases = []
    for W, N, c in [(1, 2, 0), (1, 2, 1), (2, 2, 2), (3, 3, 1), (5, 3, 5), (5, 4, 3),
                    (7, 5, 2), (15, 5, 0), (15, 5, 15), (4, 6, 4), (10, 5, 10), (16, 2, 3)]:
        V = 50
        w = la.window_init(W, N, V, rng)
        last = int(rng.integers(0, V))
        sufs = [tuple(int(t) for t in rng.integers(0, V, size=N - 1)) for _ in range(c)]
        L = la.build_layout(w, last, [la.CandidateBranch(suffix=s) for s in sufs])
        cases.append({"W": W, "N": N, "levels": w.levels, "last": last,
                      "suffixes": [list(s) for s in sufs], "layout": _layout_record(L),
                      "matrix": L.visibility_matrix()})
    _dump("layouts.json", {"source": "layout.build_layout (layout.py:128-182)", "cases": cases})


def gen_pool(la):
    rng = np.random.default_rng(77)
    cases = []
    for trial in range(12):
        n = int(rng.integers(2, 6))
        vocab = int(rng.integers(2, 6))
        cap = None if trial % 3 else int(rng.integers(1, 20))
        pool = la.NGramPool(n, capacity=cap)
        ops = []
        for _ in range(int(rng.integers(20, 120))):
            g = [int(t) for t in rng.integers(0, vocab, size=n)]
            pool.insert(g)
            lead = int(rng.integers(0, vocab))
            lim = int(rng.integers(0, 8))
            ops.append({"insert": g, "lookup": [lead, lim],
                        "result": [list(s) for s in pool.lookup(lead, lim)], "len": len(pool)})
        cases.append({"ngram": n, "capacity": cap, "ops": ops})
    # prompt seeding (pool.py:83-90)
    seeds = []
    for prompt, n in [([1, 2, 3, 4], 3), ([1, 2], 3), ([7, 7, 7, 7, 7], 3),
                      ([int(t) for t in rng.integers(0, 4, size=40)], 4)]:
        pool = la.NGramPool(n)
        pool.seed_from_prompt(prompt)
        seeds.append({"prompt": prompt, "ngram": n, "len": len(pool),
                      "lookups": {str(t): [list(s) for s in pool.lookup(t, 100)] for t in range(8)}})
    _dump("pool.json", {"source": "pool.NGramPool (pool.py:17-90)", "cases": cases, "seeding": seeds})


def gen_window(la):
    rng = np.random.default_rng(31)
    cases = []
    for _ in range(40):
        W = int(rng.integers(1, 17))
        N = int(rng.integers(2, 7))
        V = int(rng.integers(2, 300))
        w = la.window_init(W, N, V, rng)
        last = int(rng.integers(0, V))
        new_top = [int(t) for t in rng.integers(0, V, size=W)]
        k = int(rng.integers(1, N + 1))
        seed = int(rng.integers(0, 1000))
        r = np.random.default_rng(seed)
        upd = la.window_update(w, new_top, k, r)
        draws_left = int(r.integers(0, 2**31))
        grams = la.collect_ngrams(w, new_top, last)
        cases.append({"W": W, "N": N, "V": V, "levels": w.levels, "last": last,
                      "new_top": new_top, "k": k, "seed": seed, "updated": upd.levels,
                      "next_draw": draws_left, "ngrams": [list(g) for g in grams]})
    _dump("window.json", {"source": "layout.window_update/collect_ngrams (layout.py:197-252)",
                          "cases": cases})


def gen_verify(la):
    rng = np.random.default_rng(55)
    cases = []
    for _ in range(200):
        V = int(rng.integers(2, 6))
        n_pos = int(rng.integers(1, 5))
        c = int(rng.integers(0, 6))

        def onehotish():
            p = rng.random(V)
            return p / p.sum()

        base = onehotish()
        cands = []
        for _ in range(c):
            suf = [int(t) for t in rng.integers(0, V, size=n_pos)]
            cands.append((tuple(suf), [base] + [onehotish() for _ in range(n_pos)]))
        acc = la.verify_greedy(base, cands)
        cases.append({"V": V, "base": base.tolist(),
                      "cands": [[list(s), [d.tolist() for d in ds]] for s, ds in cands],
                      "accepted": acc})
    _dump("verify.json", {"source": "verification.verify_greedy (verification.py:43-71)",
                          "cases": cases})


def _metrics(m):
    return {"tokens_generated": m.tokens_generated, "steps": m.steps,
            "compression": m.compression,
            "acceptance_histogram": {str(k): v for k, v in m.acceptance_histogram.items()},
            "total_queries": m.total_queries, "mean_queries_per_step": m.mean_queries_per_step}


def _trace_decode(la, model, prompt, cfg, sampler):
    """Per-step outcomes via the reference step API (decoding.py:67-211)."""
    from lookahead.decoding import collect_output
    state = la.start_session(model, prompt, cfg, sampler)
    out, steps, done = [], [], False
    while not done:
        o = la.lookahead_step(state)
        steps.append({"accepted": o.accepted, "new_top": o.new_top,
                      "c": o.candidate_count, "M": o.query_count,
                      "pool": state.records[-1].pool_size})
        done = collect_output(out, o.accepted, cfg.max_tokens, cfg.eos_token)
    return out, steps


def gen_decode(la):
    greedy = la.SamplerSpec(mode="greedy", seed=0)
    runs = []
    # cfg1 (BASELINE configs[0]): TinyTransformer seed 0, V 256 / 32000, W5 N3 G5, 32 + 128
    for V, (W, N, G) in [(256, (5, 3, 5)), (256, (15, 5, 15)), (32000, (5, 3, 5))]:
        model = la.transformer_init(seed=0, vocab_size=V, d_model=16, n_layers=2, n_heads=2)
        prompt = [int(t) for t in np.random.default_rng(1234).integers(0, V, 32)]
        cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=128)
        toks, metrics = la.decode_lookahead(model, prompt, cfg, greedy)
        out, steps = _trace_decode(la, model, prompt, cfg, greedy)
        assert out == toks
        ar = la.decode_autoregressive(model, prompt, greedy, 128)
        runs.append({"model": {"seed": 0, "vocab": V, "d": 16, "L": 2, "H": 2},
                     "prompt": prompt, "W": W, "N": N, "G": G, "max_tokens": 128,
                     "eos": None, "seed_pool": False, "sampler_seed": 0,
                     "tokens": toks, "ar_tokens": ar, "metrics": _metrics(metrics),
                     "steps": steps})
    # the reference test-suite transformers (conftest.py:37-39, test_acceptance.py:49-51)
    for mseed, V in [(11, 12), (3, 16)]:
        model = la.transformer_init(seed=mseed, vocab_size=V, d_model=16, n_layers=2, n_heads=2)
        rng = np.random.default_rng(101)
        for i in range(6):
            prompt = [int(t) for t in rng.integers(0, V, size=int(rng.integers(4, 7)))]
            sampler = la.SamplerSpec(mode="greedy", seed=i)
            ar = la.decode_autoregressive(model, prompt, sampler, 16)
            for W, N, G in [(1, 2, 0), (5, 3, 5), (15, 5, 15)]:
                for eos in (None, ar[5]):
                    cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G,
                                              max_tokens=16, eos_token=eos,
                                              seed_pool_from_prompt=True)
                    toks, metrics = la.decode_lookahead(model, prompt, cfg, sampler)
                    out, steps = _trace_decode(la, model, prompt, cfg, sampler)
                    assert out == toks
                    runs.append({"model": {"seed": mseed, "vocab": V, "d": 16, "L": 2, "H": 2},
                                 "prompt": prompt, "W": W, "N": N, "G": G, "max_tokens": 16,
                                 "eos": eos, "seed_pool": True, "sampler_seed": i,
                                 "tokens": toks,
                                 "ar_tokens": la.decode_autoregressive(model, prompt, sampler,
                                                                       16, eos),
                                 "metrics": _metrics(metrics), "steps": steps})
    _dump("decode_tiny.json", {"source": "decoding.decode_lookahead / decode_autoregressive "
                                         "(decoding.py:96-116,235-255)", "runs": runs})


def gen_forward(la):
    """Per-query log-probabilities of ModelInterface.forward (models.py:80-89)."""
    arrays = {}
    meta = []
    rng = np.random.default_rng(9)
    cases = [((11, 12), 5, 3, 2, 6), ((0, 256), 5, 3, 5, 31), ((0, 256), 15, 5, 15, 100),
             ((3, 16), 1, 2, 1, 3)]
    for idx, ((mseed, V), W, N, c, plen) in enumerate(cases):
        model = la.transformer_init(seed=mseed, vocab_size=V, d_model=16, n_layers=2, n_heads=2)
        w = la.window_init(W, N, V, rng)
        prefix = [int(t) for t in rng.integers(0, V, size=plen)]
        last = int(rng.integers(0, V))
        sufs = [tuple(int(t) for t in rng.integers(0, V, size=N - 1)) for _ in range(c)]
        L = la.build_layout(w, last, [la.CandidateBranch(suffix=s) for s in sufs])
        d = model.forward(prefix, L)
        arrays[f"case{idx}"] = np.log(np.stack(d))
        meta.append({"model": [mseed, V], "W": W, "N": N, "levels": w.levels, "last": last,
                     "suffixes": [list(s) for s in sufs], "prefix": prefix,
                     "layout": _layout_record(L)})
    # hand-built layouts of tests/test_models.py:122-163 (two chains off query 0)
    model = la.transformer_init(seed=11, vocab_size=12, d_model=16, n_layers=2, n_heads=2)
    qs = [la.QueryToken(token=1, rel_pos=0)]
    for start in (1, 4):
        for k in range(3):
            qs.append(la.QueryToken(token=int(rng.integers(0, 12)), rel_pos=k + 1,
                                    visible=(0,) + tuple(range(start, start + k))))
    L = la.StepLayout(queries=qs)
    arrays["hand0"] = np.log(np.stack(model.forward([0], L)))
    meta.append({"model": [11, 12], "prefix": [0], "layout": _layout_record(L), "hand": True})
    L = la.chain_layout(7, [1, 2, 3])
    arrays["hand1"] = np.log(np.stack(model.forward([4, 5], L)))
    meta.append({"model": [11, 12], "prefix": [4, 5], "layout": _layout_record(L), "hand": True})
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "forward_tiny.npz", **arrays)
    _dump("forward_tiny.json", {"source": "models.ModelInterface.forward (models.py:80-89)",
                                "cases": meta})


def gen_lp(la):
    from lookahead.parallel import partition_layout
    rng = np.random.default_rng(66)
    plans = []
    for W, N, c, D in [(15, 5, 15, 1), (15, 5, 15, 2), (15, 5, 15, 4), (15, 5, 15, 8),
                       (5, 3, 5, 2), (5, 3, 2, 4), (7, 2, 3, 3), (4, 6, 4, 4), (15, 5, 7, 8)]:
        w = la.window_init(W, N, 10, rng)
        sufs = [tuple(int(t) for t in rng.integers(0, 10, size=N - 1)) for _ in range(c)]
        L = la.build_layout(w, 0, [la.CandidateBranch(suffix=s) for s in sufs])
        ps = partition_layout(L, W, N, D)
        plans.append({"W": W, "N": N, "c": c, "D": D,
                      "plans": [{"columns": [p.columns.start, p.columns.stop],
                                 "candidates": p.candidates, "owned": p.owned_queries,
                                 "redundant": p.redundant_queries} for p in ps]})
    runs = []
    model = la.transformer_init(seed=3, vocab_size=16, d_model=16, n_layers=2, n_heads=2)
    for W, N, G, D in [(5, 3, 5, 2), (5, 3, 5, 4), (15, 5, 15, 2), (15, 5, 15, 4), (15, 5, 15, 8)]:
        prompt = [int(t) for t in np.random.default_rng(W * 10 + D).integers(0, 16, 6)]
        cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=24,
                                  seed_pool_from_prompt=True)
        sampler = la.SamplerSpec(mode="greedy", seed=D)
        toks, metrics, comm = la.decode_lookahead_devices(model, prompt, cfg, sampler, D)
        runs.append({"model": [3, 16], "prompt": prompt, "W": W, "N": N, "G": G, "D": D,
                     "sampler_seed": D, "max_tokens": 24, "tokens": toks,
                     "metrics": _metrics(metrics),
                     "comm": {"tokens_synchronized": comm.tokens_synchronized,
                              "sync_events": comm.sync_events}})
    _dump("lp.json", {"source": "parallel.partition_layout / decode_lookahead_devices "
                                "(parallel.py:64-192)", "plans": plans, "runs": runs})


def gen_jacobi(la):
    # decode_jacobi (decoding.py:119-149) on the TinyTransformer of config 1;
    # the rng is passed in the state the caller left it, so each case records
    # the seed of a fresh default_rng
    model = la.transformer_init(seed=0, vocab_size=256, d_model=16, n_layers=2, n_heads=2)
    cases = []
    for k, m in enumerate([1, 2, 3, 8, 16, 31, 64]):
        prompt = [int(t) for t in np.random.default_rng(700 + k).integers(0, 256, 5 + 3 * k)]
        seed = 900 + k
        toks, traj, iters = la.decode_jacobi(model, prompt, m, np.random.default_rng(seed))
        cases.append({"model": [0, 256], "prompt": prompt, "m": m, "rng_seed": seed,
                      "tokens": toks, "iterates": traj.iterates, "iterations": iters})
    _dump("jacobi.json", {"source": "decoding.decode_jacobi (decoding.py:119-149)", "cases": cases})


def gen_sampling(la):
    """Temperature sampler: adjusted distributions (sampling.py:22-66),
    verify_sample (verification.py:74-118) and whole sampled decodes
    (decoding.py:96-116,160-204) on the config-1 TinyTransformer."""
    from lookahead.sampling import adjusted_distribution
    from lookahead.verification import verify_sample
    rng = np.random.default_rng(77)
    adjust = []
    for i in range(60):
        V = int(rng.integers(2, 40))
        p = rng.random(V) ** 3
        if i % 4 == 1:                       # ties: quantised probabilities
            p = np.round(p * 4) / 4 + 1e-3
        if i % 7 == 3:                       # zeros
            p[rng.integers(0, V, size=max(1, V // 3))] = 0.0
        p = p / p.sum()
        T = [1.0, 0.5, 0.7, 1.5, 2.0][i % 5]
        k = [None, 1, 2, 5, 17, 100][i % 6]
        tp = [None, 0.9, 0.5, 0.99, 0.01, 1.0, 0.3][i % 7]
        spec = la.SamplerSpec(mode="temperature", temperature=T, top_k=k, top_p=tp, seed=0)
        adjust.append({"probs": p.tolist(), "T": T, "top_k": k, "top_p": tp,
                       "out": adjusted_distribution(p, spec).tolist()})
    verify = []
    for i in range(120):
        V = int(rng.integers(2, 7))
        S = int(rng.integers(1, 5))
        c = int(rng.integers(0, 6))

        def dist():
            q = rng.random(V) ** 2
            if rng.random() < 0.2:
                q[int(rng.integers(0, V))] = 0.0
            q[int(rng.integers(0, V))] += 0.05
            return q / q.sum()

        base = dist()
        cands = []
        for _ in range(c):
            suf = [int(t) for t in rng.integers(0, V, size=S)]
            cands.append((tuple(suf), [base] + [dist() for _ in range(S)]))
        seed = 1000 + i
        acc = verify_sample(base, cands, np.random.default_rng(seed))
        verify.append({"V": V, "base": base.tolist(), "seed": seed,
                       "cands": [[list(s), [d.tolist() for d in ds]] for s, ds in cands],
                       "accepted": acc})
    decode = []
    model = la.transformer_init(seed=0, vocab_size=256, d_model=16, n_layers=2, n_heads=2)
    prompt = [int(t) for t in np.random.default_rng(1234).integers(0, 256, 32)]
    for j, (T, k, tp) in enumerate([(1.0, None, None), (0.7, None, None), (0.5, 20, None),
                                    (1.0, None, 0.9), (0.8, 50, 0.95), (1.3, None, None)]):
        spec = la.SamplerSpec(mode="temperature", temperature=T, top_k=k, top_p=tp, seed=j)
        for W, N, G in [(5, 3, 5), (15, 5, 15), (1, 2, 0)]:
            cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=48)
            toks, metrics = la.decode_lookahead(model, prompt, cfg, spec)
            out, steps = _trace_decode(la, model, prompt, cfg, spec)
            assert out == toks
            decode.append({"prompt": prompt, "W": W, "N": N, "G": G, "max_tokens": 48,
                           "T": T, "top_k": k, "top_p": tp, "seed": j, "tokens": toks,
                           "metrics": _metrics(metrics), "steps": steps})
    ar = []
    for j, (T, k, tp) in enumerate([(1.0, None, None), (0.6, 10, 0.9), (2.0, None, 0.8)]):
        spec = la.SamplerSpec(mode="temperature", temperature=T, top_k=k, top_p=tp, seed=40 + j)
        ar.append({"prompt": prompt, "T": T, "top_k": k, "top_p": tp, "seed": 40 + j,
                   "max_tokens": 64, "tokens": la.decode_autoregressive(model, prompt, spec, 64)})
    _dump("sampling.json", {"source": "sampling.adjusted_distribution, verification.verify_sample, "
                                      "decoding.decode_lookahead / decode_autoregressive "
                                      "(temperature SamplerSpec)",
                            "model": [0, 256], "adjust": adjust, "verify": verify,
                            "decode": decode, "ar": ar})


def gen_cli(la):
    """Reports of the reference CLI (cli.py:174-297) on the config-1 transformer,
    run with relative paths from a scratch directory so the config echo is
    location independent; the GPU test re-runs the same argv on our CLI."""
    import shutil
    import tempfile
    from lookahead import cli
    prompts = "hello lookahead\nthe quick brown fox jumps\nabcabcabcabc\n"
    cases = [
        ["decode", "--mode", "lookahead", "-W", "5", "-N", "3", "--max-tokens", "40"],
        ["decode", "--mode", "autoregressive", "--max-tokens", "24", "--format", "csv"],
        ["decode", "--mode", "jacobi", "--max-tokens", "16"],
        ["decode", "--mode", "lookahead", "-W", "4", "-N", "4", "-G", "2", "--max-tokens", "32",
         "--pool-from-prompt", "--temperature", "0.8", "--top-p", "0.9", "--seed", "3"],
        ["bench", "-W", "5", "-N", "3", "--max-tokens", "20", "--pool-from-prompt"],
        ["simulate", "--devices", "2", "-W", "6", "-N", "3", "--max-tokens", "24"],
        ["decode", "--mode", "lookahead", "-W", "5", "-N", "3", "--max-tokens", "40",
         "--pool-capacity", "6", "--pool-from-prompt"],
    ]
    out = []
    d = tempfile.mkdtemp()
    cwd = os.getcwd()
    try:
        os.chdir(d)
        for argv in cases:
            for f in os.listdir("."):
                os.remove(f)
            Path("prompts.txt").write_text(prompts)
            full = argv + ["--model", "transformer", "--prompts", "prompts.txt", "--out", "report.json"]
            assert cli.main(full) == 0
            files = {f: Path(f).read_text() for f in sorted(os.listdir(".")) if f != "prompts.txt"}
            out.append({"argv": full, "files": files})
    finally:
        os.chdir(cwd)
        shutil.rmtree(d)
    _dump("cli.json", {"source": "cli.main (cli.py:174-330), --model transformer", "prompts": prompts,
                       "cases": out})


def main():
    la = _ref()
    if len(sys.argv) > 1:   # regenerate selected fixtures only, e.g. `make_golden.py jacobi`
        for name in sys.argv[1:]:
            globals()["gen_" + name](la)
        print("golden vectors written to", OUT)
        return
    gen_layouts(la)
    gen_pool(la)
    gen_window(la)
    gen_verify(la)
    gen_forward(la)
    gen_lp(la)
    gen_decode(la)
    gen_jacobi(la)
    gen_sampling(la)
    gen_cli(la)
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
