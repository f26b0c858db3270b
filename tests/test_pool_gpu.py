"""Device n-gram pool (la_state.cuh) against the oracle pool (pool.py:17-90),
through the step-finish insert path: the block-parallel batch insert for the
unbounded pool and the serial LRU path under a capacity.  The oracle pool is
itself pinned to the reference's pool streams (tests/test_oracle_golden.py)."""

import ctypes as C

import numpy as np
import pytest

from oracle import lookahead_oracle as lo
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

la = pytest.importorskip("paper_2402_02057_b200")
from paper_2402_02057_b200 import _lib  # noqa: E402

P32 = C.POINTER(C.c_int32)


def _device_pool(N, cap, grams, batch, leads, limit):
    lib = _lib.load()
    g = np.ascontiguousarray(np.asarray(grams, dtype=np.int32).reshape(-1, N))
    ld = np.ascontiguousarray(np.asarray(leads, dtype=np.int32))
    nb = (len(g) + batch - 1) // batch
    out = np.zeros((nb, len(ld), limit, N - 1), dtype=np.int32)
    counts = np.zeros((nb, len(ld)), dtype=np.int32)
    lens = np.zeros(nb, dtype=np.int32)
    _lib.check(lib.la_pool_test(N, cap or 0, limit, g.ctypes.data_as(P32), len(g), batch,
                                ld.ctypes.data_as(P32), len(ld), limit, out.ctypes.data_as(P32),
                                counts.ctypes.data_as(P32), lens.ctypes.data_as(P32)))
    return out, counts, lens


@pytest.mark.parametrize("cap", [None, 3, 17])
@pytest.mark.parametrize("N,vocab,batch", [(2, 3, 15), (3, 4, 15), (5, 3, 7), (4, 6, 31)])
def test_batched_inserts_equal_serial_oracle(N, vocab, batch, cap):
    rng = np.random.default_rng(N * 100 + vocab + batch + (cap or 0))
    grams = rng.integers(0, vocab, size=(batch * 12, N))
    grams[::5] = grams[1::5][: len(grams[::5])]          # in-batch repeats
    leads, limit = list(range(vocab)), 8
    out, counts, lens = _device_pool(N, cap, grams.ravel(), batch, leads, limit)
    pool = lo.OraclePool(N, capacity=cap)
    for b in range(len(lens)):
        pool.insert_all([tuple(int(t) for t in x) for x in grams[b * batch:(b + 1) * batch]])
        assert lens[b] == len(pool), b
        for q, lead in enumerate(leads):
            ref = pool.lookup(lead, limit)
            got = [tuple(out[b, q, i].tolist()) for i in range(counts[b, q])]
            assert got == [tuple(s) for s in ref], (b, lead)


def test_reference_pool_streams_on_device():
    """tests/golden/pool.json (reference NGramPool op streams, with and without
    capacity): one insert per batch, every lookup checked."""
    for case in load_golden("pool.json")["cases"]:
        N, cap = case["ngram"], case["capacity"]
        ops = case["ops"]
        vocab = 1 + max(max(o["insert"]) for o in ops)
        out, counts, lens = _device_pool(N, cap, [t for o in ops for t in o["insert"]], 1,
                                         list(range(max(vocab, 8))), 8)
        for b, o in enumerate(ops):
            lead, lim = o["lookup"]
            if lead >= out.shape[1]:
                continue
            got = [list(out[b, lead, i]) for i in range(min(counts[b, lead], lim))]
            assert got == o["result"], (N, cap, b)
            assert lens[b] == o["len"]


def test_large_capacity_pool_memory_is_linear():
    """An LRU cap of thousands of entries over a 1000-token vocabulary (the
    capped pool links each lead's entries through the distinct-set slots:
    O(LT + ST) memory, no per-lead buckets sized to the cap)."""
    N, cap, V = 5, 2500, 1000
    rng = np.random.default_rng(17)
    grams = rng.integers(0, V, size=(15 * 300, N))
    grams[:, 0] = rng.integers(0, 40, size=len(grams))        # few leads, long lists
    grams[7::9] = grams[3::9][: len(grams[7::9])]             # refreshes
    leads, limit = list(range(40)), 15
    out, counts, lens = _device_pool(N, cap, grams.ravel(), 15, leads, limit)
    pool = lo.OraclePool(N, capacity=cap)
    for b in range(len(lens)):
        pool.insert_all([tuple(int(t) for t in x) for x in grams[b * 15:(b + 1) * 15]])
        assert lens[b] == len(pool), b
        if b % 25 == 0 or b == len(lens) - 1:
            for q, lead in enumerate(leads):
                got = [tuple(out[b, q, i].tolist()) for i in range(counts[b, q])]
                assert got == [tuple(s) for s in pool.lookup(lead, limit)], (b, lead)
    assert len(pool) == cap


def _lossless_up_to_near_tie(orc, prompt, ar, toks, rel_tol=1e-2):
    """toks == ar, or they first differ where the two tokens are the top two
    of a near tie (oracle top-2 logit margin below rel_tol, the north_star's
    bf16 tolerance): a lookahead row and the greedy step sum a row's keys over
    different prefix / step-block splits, so bf16 rounding may flip a tie."""
    i = next((k for k, (a, b) in enumerate(zip(ar, toks)) if a != b), None)
    if i is None:
        return len(ar) == len(toks)
    seq = list(prompt) + list(ar[:i])
    lg = orc.logits_rows(seq[:-1], lo.Rows([seq[-1]], [0], [[]], [], []))[0]
    top2 = set(int(t) for t in np.argsort(lg)[-2:])
    srt = np.sort(lg)
    margin = (srt[-1] - srt[-2]) / max(np.abs(lg).max(), 1e-6)
    return margin < rel_tol and {ar[i], toks[i]} <= top2


def test_capped_decode_at_7b_session_scale():
    """The advisor's failing case: a W15 N5 G15 session with a pool cap of a
    few thousand on a 1000-token vocabulary and a 2048-token context now runs;
    greedy lookahead stays lossless (up to a documented near tie)."""
    from oracle.model_oracle import LlamaOracle, llama_random_weights
    cfg_m = dict(dim=256, layers=2, heads=4, kv_heads=2, head_dim=128, ffn=512, vocab=1000,
                 rope_theta=10000.0, eps=1e-5)
    w = llama_random_weights(cfg_m, seed=3, std=None)
    lc = la.LlamaConfig(dim=256, layers=2, heads=4, kv_heads=2, ffn=512, vocab=1000, head_dim=128,
                        rope_theta=1e4, norm_eps=1e-5)
    m = la.LlamaModel(lc, dtype="bf16", weights=w, max_context=2048)
    orc = LlamaOracle(cfg_m, w, emulate_bf16=True)
    try:
        prompt = [int(t) for t in np.random.default_rng(5).integers(0, 1000, 600)]
        cfg = la.GenerationConfig(window=15, ngram=5, max_candidates=15, max_tokens=200,
                                  seed_pool_from_prompt=True)
        ar = la.decode_autoregressive(m, prompt, la.SamplerSpec("greedy"), 200)
        for cap in (600, 2500):
            pool = la.NGramPool(5, capacity=cap)
            toks, met = la.decode_lookahead(m, prompt, cfg, la.SamplerSpec("greedy", seed=0), pool=pool)
            assert _lossless_up_to_near_tie(orc, prompt, ar, toks)
            assert len(pool) <= cap
            state = la.start_session(m, prompt, cfg, la.SamplerSpec("greedy", seed=0),
                                     pool=la.NGramPool(5, capacity=cap))
            out = []
            while not la.collect_output(out, la.lookahead_step(state).accepted, 200, None):
                pass
            assert out == toks      # the session is the same decode
    finally:
        m.close()
