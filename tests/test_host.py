"""CPU tests of the host-side logic of the drop-in package: API types and
their validation, the host pool container, layout -> chain conversion
(LayoutError semantics), RNG stream sizing, run metrics and the LP row plan
-- each against the reference's golden vectors / known answers."""

import numpy as np
import pytest

import paper_2402_02057_b200 as la
from paper_2402_02057_b200.decoding import window_rng_draws, window_rng_stream
from paper_2402_02057_b200.layout import layout_chains
from paper_2402_02057_b200.parallel import shard_rows
from oracle import lookahead_oracle as lo
from oracle.model_oracle import TinyTransformerOracle
from tests.conftest import load_golden


# ------------------------------------------------------------- types
def test_generation_config_defaults_and_errors():
    c = la.GenerationConfig()
    assert (c.window, c.ngram, c.max_candidates, c.max_tokens) == (15, 5, 15, 64)
    assert la.GenerationConfig(window=7).max_candidates == 7           # G defaults to W
    for kw, msg in [({"window": 0}, "W must be"), ({"ngram": 1}, "N must be"),
                    ({"max_candidates": -1}, "G must be"), ({"max_tokens": 0}, "positive")]:
        with pytest.raises(ValueError, match=msg):
            la.GenerationConfig(**kw)


def test_sampler_spec_validation():
    la.SamplerSpec("greedy")
    for kw in [{"mode": "beam"}, {"temperature": 0}, {"top_k": 0}, {"top_p": 0.0}, {"top_p": 1.5}]:
        with pytest.raises(ValueError):
            la.SamplerSpec(**kw)


def test_step_record_requires_progress():
    with pytest.raises(ValueError):
        la.StepRecord(0, 0, 1, 0)


def test_flops_proxy_and_compression():
    assert la.flops_proxy(15, 5, 15) == 120      # paper §5.5 / reference test_acceptance.py:161-165
    assert la.flops_proxy(10, 5, 10) == 80
    assert la.flops_proxy(7, 5, 7) == 56
    assert la.compression_ratio(10, 4) == 2.5
    with pytest.raises(ValueError):
        la.compression_ratio(1, 0)


# -------------------------------------------------------------- pool
def test_host_pool_matches_reference_golden():
    g = load_golden("pool.json")
    for case in g["cases"]:
        p = la.NGramPool(case["ngram"], capacity=case["capacity"])
        for op in case["ops"]:
            p.insert(op["insert"])
            lead, lim = op["lookup"]
            assert [list(s) for s in p.lookup(lead, lim)] == op["result"]
            assert len(p) == op["len"]
    for s in g["seeding"]:
        p = la.NGramPool(s["ngram"])
        p.seed_from_prompt(s["prompt"])
        assert len(p) == s["len"]
        for t, res in s["lookups"].items():
            assert [list(x) for x in p.lookup(int(t), 100)] == res


def test_host_pool_errors():
    with pytest.raises(ValueError):
        la.NGramPool(1)
    with pytest.raises(ValueError):
        la.NGramPool(3, capacity=0)
    with pytest.raises(ValueError):
        la.NGramPool(3).insert((1, 2))


# ----------------------------------------------------------- layouts
def _layout(rec):
    return la.StepLayout(queries=[la.QueryToken(t, r, tuple(v)) for t, r, v in
                                  zip(rec["tokens"], rec["rel"], rec["visible"])])


def test_layout_chains_of_reference_layouts():
    g = load_golden("layouts.json")
    for case in g["cases"]:
        rows = lo.build_rows([t for r in case["levels"] for t in r], case["W"], case["N"],
                             case["last"], [tuple(s) for s in case["suffixes"]])
        ids, rel, chain = layout_chains(_layout(case["layout"]))
        assert list(ids) == rows.ids and list(rel) == rows.rel
        for i in range(len(rows)):
            assert list(chain[i, : rel[i]]) == rows.chains[i]


@pytest.mark.parametrize("queries", [
    # forward reference (reference tests/test_models.py:167-176)
    [la.QueryToken(0, 0), la.QueryToken(1, 1, (0, 2)), la.QueryToken(2, 2, (0, 1))],
    # chain gap (:178-186)
    [la.QueryToken(0, 0), la.QueryToken(1, 2, (0,))],
    # two tokens at one rel_pos (:188-199)
    [la.QueryToken(0, 0), la.QueryToken(1, 1, (0,)), la.QueryToken(2, 1, (0,)),
     la.QueryToken(3, 2, (0, 1, 2))],
    # query 0 not at rel 0
    [la.QueryToken(0, 1)],
])
def test_layout_errors(queries):
    with pytest.raises(la.LayoutError):
        layout_chains(la.StepLayout(queries=queries))


def test_chain_layout_conditioning():
    # reference tests/test_models.py:201-203
    ids, rel, chain = layout_chains(la.chain_layout(7, [1, 2, 3]))
    assert list(ids) == [7, 1, 2, 3] and list(chain[3, :3]) == [0, 1, 2]


# ------------------------------------------------------ rng + metrics
def test_rng_stream_covers_every_refill():
    g = load_golden("decode_tiny.json")
    run = g["runs"][1]                                   # W15 N5 G15, 128 tokens
    W, N = run["W"], run["N"]
    need = (N - 1) * W - 1 + sum(lo.window_draws(W, N, len(s["accepted"])) for s in run["steps"])
    assert window_rng_draws(W, N, run["max_tokens"]) >= need
    s = window_rng_stream(0, 256, W, N, run["max_tokens"])
    rng = np.random.default_rng(0)
    assert list(s[: (N - 1) * W - 1]) == lo.window_init(W, N, 256, rng)


def test_run_metrics_from_records():
    g = load_golden("decode_tiny.json")
    for run in g["runs"][:6]:
        recs = [la.StepRecord(len(s["accepted"]), s["c"], s["M"], s["pool"]) for s in run["steps"]]
        m = la.RunMetrics.from_records(len(run["tokens"]), recs, run["N"])
        ref = run["metrics"]
        assert m.steps == ref["steps"] and m.total_queries == ref["total_queries"]
        assert {str(k): v for k, v in m.acceptance_histogram.items()} == ref["acceptance_histogram"]
        assert abs(m.compression - ref["compression"]) < 1e-12


# ------------------------------------------------------- LP row plan
def test_shard_rows_matches_reference_partition():
    g = load_golden("lp.json")
    for case in g["plans"]:
        W, N, c, D = case["W"], case["N"], case["c"], case["D"]
        owned_all = []
        for rank, ref in enumerate(case["plans"]):
            comp, own = shard_rows(W, N, c, rank, D)
            assert sorted(own) == sorted(ref["owned"])
            assert comp == sorted(set(ref["owned"]) | set(ref["redundant"]))
            owned_all += own
        assert sorted(owned_all) == list(range((N - 1) * (W + c)))


def test_comm_accounting_matches_reference():
    g = load_golden("lp.json")
    for run in g["runs"]:
        o = lo.decode_lookahead(TinyTransformerOracle(*run["model"]), run["prompt"], run["W"],
                                run["N"], run["G"], run["max_tokens"], None, run["sampler_seed"],
                                True)
        assert o.tokens == run["tokens"]
        tot = la.CommStats()
        for st in o.steps:
            tot.add(la.step_comm(run["W"], run["N"], run["D"], st.candidate_count))
        assert tot.tokens_synchronized == run["comm"]["tokens_synchronized"]
        assert tot.sync_events == run["comm"]["sync_events"]
