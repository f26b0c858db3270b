"""Step-level API (reference decoding.py:67-93,152-232): start_session +
lookahead_step + collect_output on the device reproduce the reference's own
per-step trace (tests/golden/decode_tiny.json, sampling.json) -- accepted
tokens, new_top, candidate / query counts, pool size, and the caller pool."""

import numpy as np
import pytest

from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

la = pytest.importorskip("paper_2402_02057_b200")


@pytest.fixture(scope="module")
def models():
    cache = {}

    def get(seed, V):
        if (seed, V) not in cache:
            cache[(seed, V)] = la.TinyTransformer(seed, V, 16, 2, 2, max_context=1024)
        return cache[(seed, V)]

    yield get
    for m in cache.values():
        m.close()


def _run_steps(m, prompt, cfg, spec, pool=None):
    state = la.start_session(m, prompt, cfg, spec, pool=pool)
    out, steps, done = [], [], False
    while not done:
        o = la.lookahead_step(state)
        steps.append({"accepted": o.accepted, "new_top": o.new_top, "c": o.candidate_count,
                      "M": o.query_count, "pool": state.records[-1].pool_size})
        done = la.collect_output(out, o.accepted, cfg.max_tokens, cfg.eos_token)
    return out, steps, state


def test_greedy_session_matches_reference_trace(models):
    for run in load_golden("decode_tiny.json")["runs"]:
        m = models(run["model"]["seed"], run["model"]["vocab"])
        cfg = la.GenerationConfig(window=run["W"], ngram=run["N"], max_candidates=run["G"],
                                  max_tokens=run["max_tokens"], eos_token=run["eos"],
                                  seed_pool_from_prompt=run["seed_pool"])
        out, steps, state = _run_steps(m, run["prompt"], cfg,
                                       la.SamplerSpec("greedy", seed=run["sampler_seed"]))
        assert out == run["tokens"]
        assert steps == run["steps"], (run["W"], run["N"], run["G"])
        assert state.prefix[len(run["prompt"]):][: len(out)] == out


def test_sampled_session_matches_reference_trace(models):
    m = models(0, 256)
    for c in load_golden("sampling.json")["decode"]:
        cfg = la.GenerationConfig(window=c["W"], ngram=c["N"], max_candidates=c["G"],
                                  max_tokens=c["max_tokens"])
        spec = la.SamplerSpec("temperature", temperature=c["T"], top_k=c["top_k"],
                              top_p=c["top_p"], seed=c["seed"])
        out, steps, _ = _run_steps(m, c["prompt"], cfg, spec)
        assert out == c["tokens"]
        assert steps == c["steps"]


def test_session_state_and_pool_mirror(models):
    """DecodeState fields: the caller pool is mutated like the reference's,
    the window reads back in Window2D form, ``rng`` advances like the
    reference session's generator, and a whole decode in between does not
    disturb the session (sessions own their engine)."""
    from oracle import lookahead_oracle as lo
    m = models(0, 256)
    prompt = [int(t) for t in np.random.default_rng(4).integers(0, 256, 20)]
    cfg = la.GenerationConfig(window=4, ngram=3, max_candidates=4, max_tokens=30,
                              seed_pool_from_prompt=True)
    pool = la.NGramPool(3)
    pool.insert([1, 2, 3])
    state = la.start_session(m, prompt, cfg, la.SamplerSpec("greedy", seed=2), pool=pool)
    assert len(pool) == 1 + len(set(tuple(prompt[i:i + 3]) for i in range(18)) - {(1, 2, 3)})
    w0 = np.random.default_rng(2).integers(0, 256, size=(3 - 1) * 4 - 1).tolist()
    assert state.window.levels == [w0[:3], w0[3:]]
    out = []
    g = np.random.default_rng(2)
    g.integers(0, 256, size=(3 - 1) * 4 - 1)
    first = True
    while True:
        o = la.lookahead_step(state)
        for _ in range(lo.window_draws(4, 3, len(o.accepted))):
            g.integers(0, 256)
        assert state.rng.bit_generator.state == g.bit_generator.state
        if first:
            la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), 4)
            first = False
        if la.collect_output(out, o.accepted, 30, None):
            break
    # oracle: same caller pool, same decode
    opool = lo.OraclePool(3)
    opool.insert((1, 2, 3))
    from oracle.model_oracle import TinyTransformerOracle
    run = lo.decode_lookahead(TinyTransformerOracle(0, 256), prompt, 4, 3, 4, 30, seed=2,
                              seed_pool=True, pool=opool)
    assert out == run.tokens
    assert len(pool) == len(opool)
    for t in range(256):
        assert pool.lookup(t, 4) == opool.lookup(t, 4)


def test_interleaved_sessions_are_independent(models):
    """Two DecodeStates on one model, stepped alternately (the reference keeps
    no per-model session state): each reproduces its own whole decode, and a
    temperature session's ``rng`` ends where the reference generator does."""
    m = models(0, 256)
    p1 = [int(t) for t in np.random.default_rng(5).integers(0, 256, 16)]
    p2 = [int(t) for t in np.random.default_rng(6).integers(0, 256, 24)]
    c1 = la.GenerationConfig(window=5, ngram=3, max_candidates=5, max_tokens=24)
    c2 = la.GenerationConfig(window=4, ngram=4, max_candidates=3, max_tokens=20,
                             seed_pool_from_prompt=True)
    s2 = la.SamplerSpec("temperature", temperature=0.8, top_p=0.9, seed=11)
    w1, _ = la.decode_lookahead(m, p1, c1, la.SamplerSpec("greedy", seed=1))
    w2, _ = la.decode_lookahead(m, p2, c2, s2)
    a = la.start_session(m, p1, c1, la.SamplerSpec("greedy", seed=1))
    b = la.start_session(m, p2, c2, s2)
    oa, ob, da, db = [], [], False, False
    while not (da and db):
        if not da:
            da = la.collect_output(oa, la.lookahead_step(a).accepted, 24, None)
        if not db:
            db = la.collect_output(ob, la.lookahead_step(b).accepted, 20, None)
    assert oa == w1 and ob == w2
    # the sampled session's generator: the reference state after the same decode
    from oracle import sampling_oracle as so
    from oracle.model_oracle import TinyTransformerOracle
    ref = so.decode_lookahead_sampled(TinyTransformerOracle(0, 256), p2, 4, 4, 3, 20, 0.8, None, 0.9,
                                      seed=11, seed_pool=True)
    assert ob == ref.tokens
    assert b.rng.bit_generator.state == ref.rng_state


def test_bf16_session_equals_whole_decode():
    from oracle.model_oracle import llama_random_weights
    cfg_m = dict(dim=256, layers=2, heads=4, kv_heads=2, head_dim=128, ffn=512, vocab=1000,
                 rope_theta=10000.0, eps=1e-5)
    w = llama_random_weights(cfg_m, seed=1, std=None)
    lc = la.LlamaConfig(dim=256, layers=2, heads=4, kv_heads=2, ffn=512, vocab=1000, head_dim=128,
                        rope_theta=10000.0, norm_eps=1e-5)
    m = la.LlamaModel(lc, dtype="bf16", weights=w, max_context=1024)
    try:
        prompt = [int(t) for t in np.random.default_rng(11).integers(0, 1000, 64)]
        cfg = la.GenerationConfig(window=5, ngram=3, max_candidates=5, max_tokens=40,
                                  seed_pool_from_prompt=True)
        for spec in (la.SamplerSpec("greedy", seed=1),
                     la.SamplerSpec("temperature", temperature=0.9, top_k=40, seed=7)):
            whole, met = la.decode_lookahead(m, prompt, cfg, spec)
            out, steps, state = _run_steps(m, prompt, cfg, spec)
            assert out == whole
            assert len(steps) == met.steps
    finally:
        m.close()


@pytest.mark.parametrize("cap", [1, 2, 5, 13, 40])
def test_lru_capped_pool_matches_oracle(models, cap):
    """NGramPool(capacity=...) global LRU eviction (pool.py:41-61) on the device
    pool: per-step candidate counts and pool sizes, the decode, and the
    caller pool afterwards equal the oracle's (itself pinned to the
    reference's capped-pool golden streams)."""
    from oracle import lookahead_oracle as lo
    from oracle.model_oracle import TinyTransformerOracle
    for (mseed, V), (W, N, G) in [((11, 12), (5, 3, 5)), ((3, 16), (7, 4, 7)), ((0, 256), (15, 5, 15))]:
        m = models(mseed, V)
        orc = TinyTransformerOracle(mseed, V)
        prompt = [int(t) for t in np.random.default_rng(cap + V).integers(0, V, 12)]
        cfg = la.GenerationConfig(window=W, ngram=N, max_candidates=G, max_tokens=40,
                                  seed_pool_from_prompt=True)
        opool = lo.OraclePool(N, capacity=cap)
        run = lo.decode_lookahead(orc, prompt, W, N, G, 40, seed=cap, seed_pool=True, pool=opool)
        pool = la.NGramPool(N, capacity=cap)
        toks, met = la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy", seed=cap), pool=pool)
        assert toks == run.tokens
        assert met.steps == len(run.steps)
        assert met.total_queries == sum(s.query_count for s in run.steps)
        assert len(pool) == len(opool) <= cap
        for t in range(V):
            assert pool.lookup(t, G) == opool.lookup(t, G), (mseed, t)
        # per step, through a session
        out, steps, state = _run_steps(m, prompt, cfg, la.SamplerSpec("greedy", seed=cap),
                                       pool=la.NGramPool(N, capacity=cap))
        assert [(s["c"], s["pool"], len(s["accepted"])) for s in steps] == \
            [(s.candidate_count, s.pool_size, len(s.accepted)) for s in run.steps]
