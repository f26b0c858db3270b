"""GPU parity of the temperature sampler (la_sample.cuh) against golden
vectors of the reference (sampling.py:22-85, verification.py:74-118,
decoding.py:96-116,160-204) and, on the bf16 path, its defining properties."""

import ctypes as C

import numpy as np
import pytest

from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

la = pytest.importorskip("paper_2402_02057_b200")
from paper_2402_02057_b200 import _lib  # noqa: E402


@pytest.fixture(scope="module")
def tiny():
    m = la.TinyTransformer(0, 256, 16, 2, 2, max_context=1024)
    yield m
    m.close()


def _spec(c, seed=None):
    return la.SamplerSpec("temperature", temperature=c["T"], top_k=c["top_k"], top_p=c["top_p"],
                          seed=c["seed"] if seed is None else seed)


@pytest.mark.parametrize("cluster", ["0", "1"])
def test_adjusted_distribution_on_device(tiny, cluster, monkeypatch):
    """fp64 on both sides: same support, values within a few ulps (pow / sum
    order); one CTA per row (fp32 path) and the cluster-split row (bf16 path)."""
    monkeypatch.setenv("LA_ADJ_HOOK_CLUSTER", cluster)
    for c in load_golden("sampling.json")["adjust"]:
        p = np.ascontiguousarray(np.array(c["probs"], dtype=np.float64)[None])
        out = np.zeros_like(p)
        smp = _lib.make_sampler(c["T"], c["top_k"], c["top_p"], np.random.default_rng(0))
        _lib.check(tiny.lib.la_adjust_distributions(tiny.engine(), p.ctypes.data, 1, p.shape[1],
                                                    C.byref(smp), out.ctypes.data, tiny.stream()))
        ref = np.array(c["out"])
        assert ((out[0] > 0) == (ref > 0)).all(), c
        np.testing.assert_allclose(out[0], ref, rtol=1e-12, atol=1e-300)


def test_verify_sample_on_device(tiny):
    for c in load_golden("sampling.json")["verify"]:
        V = c["V"]
        sufs = [s for s, _ in c["cands"]]
        S = len(sufs[0]) if sufs else 1
        rows = [c["base"]] + [d for _, ds in c["cands"] for d in ds[1:]]
        dists = np.ascontiguousarray(np.array(rows, dtype=np.float64))
        suf = np.ascontiguousarray(np.array(sufs if sufs else [[0]], dtype=np.int32))
        out = np.zeros(S + 2, dtype=np.int32)
        n = C.c_int32(0)
        smp = _lib.make_sampler(1.0, None, None, np.random.default_rng(c["seed"]))
        P32 = C.POINTER(C.c_int32)
        _lib.check(tiny.lib.la_verify_sample_dists(
            tiny.engine(), dists.ctypes.data, V, S, len(sufs), suf.ctypes.data_as(P32),
            C.byref(smp), out.ctypes.data_as(P32), C.byref(n), tiny.stream()))
        assert out[: n.value].tolist() == c["accepted"], c


def test_sampled_lookahead_matches_reference(tiny):
    """Token-exact against the reference's fp64 run: fp32 logits change a
    verification outcome only if a uniform draw lands within ~1e-6 of a
    probability boundary."""
    g = load_golden("sampling.json")
    for c in g["decode"]:
        cfg = la.GenerationConfig(window=c["W"], ngram=c["N"], max_candidates=c["G"],
                                  max_tokens=c["max_tokens"])
        toks, met = la.decode_lookahead(tiny, c["prompt"], cfg, _spec(c))
        assert toks == c["tokens"], (c["W"], c["N"], c["T"], c["top_k"], c["top_p"])
        assert met.steps == c["metrics"]["steps"]
        assert met.total_queries == c["metrics"]["total_queries"]


def test_sampled_autoregressive_matches_reference(tiny):
    for c in load_golden("sampling.json")["ar"]:
        toks = la.decode_autoregressive(tiny, c["prompt"], _spec(c), c["max_tokens"])
        assert toks == c["tokens"]


def test_sampler_errors(tiny):
    p = [1, 2, 3]
    cfg = la.GenerationConfig(window=3, ngram=3, max_candidates=3, max_tokens=8)
    with pytest.raises(ValueError):
        la.SamplerSpec("temperature", temperature=0.0)
    # top_k=1 under temperature == greedy (sampling.py:41-42)
    greedy = la.decode_lookahead(tiny, p, cfg, la.SamplerSpec("greedy"))[0]
    assert la.decode_lookahead(tiny, p, cfg, la.SamplerSpec("temperature", top_k=1, seed=5))[0] == greedy
    # LP with a temperature sampler: the reference defines the LP outcome as
    # identical to the single-device decode (parallel.py:145-151)
    spec = la.SamplerSpec("temperature", temperature=0.9, seed=4)
    single, met1 = la.decode_lookahead(tiny, p, cfg, spec)
    lp, met2, comm = la.decode_lookahead_devices(tiny, p, cfg, spec, 2)
    assert lp == single and met2.steps == met1.steps
    assert comm.sync_events > 0


# ----------------------------------------------------------- bf16 path
@pytest.fixture(scope="module")
def llama():
    from oracle.model_oracle import llama_random_weights
    cfg = dict(dim=256, layers=2, heads=4, kv_heads=2, head_dim=128, ffn=512, vocab=1000,
               rope_theta=10000.0, eps=1e-5)
    w = llama_random_weights(cfg, seed=1, std=None)
    lc = la.LlamaConfig(dim=256, layers=2, heads=4, kv_heads=2, ffn=512, vocab=1000, head_dim=128,
                        rope_theta=10000.0, norm_eps=1e-5)
    m = la.LlamaModel(lc, dtype="bf16", weights=w, max_context=1024)
    yield m
    m.close()


def test_bf16_top_k1_is_greedy_and_seeded_runs_repeat(llama):
    prompt = [int(t) for t in np.random.default_rng(11).integers(0, 1000, 64)]
    ar = la.decode_autoregressive(llama, prompt, la.SamplerSpec("greedy"), 32)
    cfg = la.GenerationConfig(window=5, ngram=3, max_candidates=5, max_tokens=32,
                              seed_pool_from_prompt=True)
    assert la.decode_lookahead(llama, prompt, cfg, la.SamplerSpec("temperature", top_k=1))[0] == ar
    assert la.decode_autoregressive(llama, prompt, la.SamplerSpec("temperature", top_k=1), 32) == ar
    s = la.SamplerSpec("temperature", temperature=1.0, top_p=0.9, seed=3)
    a = la.decode_lookahead(llama, prompt, cfg, s)[0]
    assert a == la.decode_lookahead(llama, prompt, cfg, s)[0]
    assert len(a) == 32 and all(0 <= t < 1000 for t in a)


def test_bf16_sampled_first_token_law(llama):
    """Distribution preservation (verification.py:121-150): the first token of
    a sampled lookahead decode follows the adjusted base distribution."""
    prompt = [int(t) for t in np.random.default_rng(5).integers(0, 1000, 24)]
    prompt = prompt + prompt[:8]            # give the pool candidates for the first step
    layout = la.StepLayout(queries=[la.QueryToken(prompt[-1], 0, ())])
    probs = np.asarray(llama.forward(prompt[:-1], layout)[0], dtype=np.float64)
    from oracle.sampling_oracle import adjusted_distribution
    T, k = 0.7, 8
    want = adjusted_distribution(probs / probs.sum(), T, k, None)
    cfg = la.GenerationConfig(window=4, ngram=3, max_candidates=4, max_tokens=1,
                              seed_pool_from_prompt=True)
    n = 400
    counts = np.zeros(1000)
    for seed in range(n):
        t = la.decode_lookahead(llama, prompt, cfg,
                                la.SamplerSpec("temperature", temperature=T, top_k=k, seed=seed))[0]
        counts[t[0]] += 1
    assert counts[want == 0].sum() == 0
    tv = 0.5 * np.abs(counts / n - want).sum()
    assert tv < 0.12, tv


def _verify(m, base, cands, seed):
    """device verify_sample; cands = [(suffix, [d_1 .. d_S])] (base shared)."""
    V = len(base)
    S = len(cands[0][0]) if cands else 1
    rows = [base] + [d for _, ds in cands for d in ds]
    dists = np.ascontiguousarray(np.array(rows, dtype=np.float64))
    suf = np.ascontiguousarray(np.array([s for s, _ in cands] if cands else [[0]], dtype=np.int32))
    out = np.zeros(S + 2, dtype=np.int32)
    n = C.c_int32(0)
    smp = _lib.make_sampler(1.0, None, None, np.random.default_rng(seed))
    P32 = C.POINTER(C.c_int32)
    _lib.check(m.lib.la_verify_sample_dists(m.engine(), dists.ctypes.data, V, S, len(cands),
                                            suf.ctypes.data_as(P32), C.byref(smp),
                                            out.ctypes.data_as(P32), C.byref(n), m.stream()))
    return out[: n.value].tolist()


def test_verify_sample_law_on_device(tiny):
    """test_verification.py:103-132 / test_acceptance.py:113-127: the first
    emitted token follows the base law whatever the speculations."""
    cases = [
        (np.array([0.4, 0.3, 0.2, 0.1]), []),                                        # no candidates
        (np.array([0.4, 0.3, 0.2, 0.1]), [((2,), [np.full(4, 0.25)])]),              # single candidate
        (np.array([0.5, 0.3, 0.2]), [((1,), [np.array([0.5, 0.3, 0.2])])] * 2),      # duplicates
        (np.array([0.1, 0.2, 0.3, 0.4]), [((3, 1), [np.full(4, 0.25)] * 2), ((0, 2), [np.full(4, 0.25)] * 2),
                                          ((3, 3), [np.full(4, 0.25)] * 2)]),
    ]
    runs = 30000
    for base, cands in cases:
        counts = np.zeros(len(base))
        for seed in range(runs):
            counts[_verify(tiny, base, cands, seed)[0]] += 1
        tv = 0.5 * np.abs(counts / runs - base).sum()
        assert tv < 0.01, (cands, tv)


def test_verify_sample_edge_cases_on_device(tiny):
    oh = lambda i: np.eye(3)[i]  # noqa: E731
    # one-hot distributions accept every speculation, any seed (test_verification.py:92-101)
    for seed in range(25):
        assert _verify(tiny, oh(2), [((2, 0), [oh(0), oh(1)])], seed) == [2, 0, 1]
    # deterministic given the generator state (:134-139)
    base = np.array([0.4, 0.3, 0.2, 0.1])
    c = [((2,), [np.full(4, 0.25)])]
    assert _verify(tiny, base, c, 42) == _verify(tiny, base, c, 42)
    # zero-mass base raises DegenerateDistributionError (:141-144)
    dead = np.zeros(2)
    with pytest.raises(la.DegenerateDistributionError):
        _verify(tiny, dead, [((1,), [dead])], 0)


@pytest.mark.parametrize("cluster", ["0", "1"])
def test_adjusted_distribution_wide_vocab(tiny, cluster, monkeypatch):
    """V = 32000 rows (slices of 4000 per cluster CTA) incl. ties, vs the oracle."""
    from oracle.sampling_oracle import adjusted_distribution
    monkeypatch.setenv("LA_ADJ_HOOK_CLUSTER", cluster)
    rng = np.random.default_rng(9)
    for T, k, tp in [(1.0, 50, None), (0.7, None, 0.9), (1.3, 1000, 0.5), (0.5, 7, 0.99)]:
        p = rng.random(32000) ** 4
        p[::97] = p[5]                       # a block of exact ties
        p /= p.sum()
        x = np.ascontiguousarray(p[None])
        out = np.zeros_like(x)
        smp = _lib.make_sampler(T, k, tp, np.random.default_rng(0))
        _lib.check(tiny.lib.la_adjust_distributions(tiny.engine(), x.ctypes.data, 1, 32000,
                                                    C.byref(smp), out.ctypes.data, tiny.stream()))
        ref = adjusted_distribution(p, T, k, tp)
        assert ((out[0] > 0) == (ref > 0)).all(), (T, k, tp)
        np.testing.assert_allclose(out[0], ref, rtol=1e-11, atol=1e-300)
