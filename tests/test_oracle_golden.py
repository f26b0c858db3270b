"""Pin the CPU oracle to golden vectors produced by the reference itself
(``oracle/make_golden.py``) and to the reference test-suite's known answers.
CPU only."""

import numpy as np
import pytest

from oracle import lookahead_oracle as lo
from oracle.model_oracle import TinyTransformerOracle, bf16_round
from tests.conftest import GOLDEN, load_golden


def _levels_to_flat(levels):
    return [t for row in levels for t in row]


def _flat_to_levels(flat, W, N):
    out = [flat[: W - 1]]
    for l in range(1, N - 1):
        s = W - 1 + (l - 1) * W
        out.append(flat[s : s + W])
    return out


def _visible_from_chain(rows, i):
    # the reference's visible set = chain rows minus the implicit query 0
    # when query 0 is listed (build_layout lists 0 explicitly for non-q0 rows)
    return sorted(rows.chains[i])


def test_layouts_match_reference():
    g = load_golden("layouts.json")
    for case in g["cases"]:
        W, N = case["W"], case["N"]
        rows = lo.build_rows(_levels_to_flat(case["levels"]), W, N, case["last"],
                             [tuple(s) for s in case["suffixes"]])
        ref = case["layout"]
        assert rows.ids == ref["tokens"]
        assert rows.rel == ref["rel"]
        assert rows.generators == ref["generators"]
        for i in range(len(rows)):
            assert _visible_from_chain(rows, i) == ref["visible"][i], (W, N, i)
        assert [[b, b + N - 1] for b in rows.branch_base] == ref["branches"]
        assert len(rows) == (N - 1) * (W + len(case["suffixes"]))   # appendix A.1


def test_visibility_matrix_known_answer():
    # tests/test_layout.py:138-153 (W3 N3, one candidate)
    rows = lo.build_rows([21, 22, 11, 12, 13], 3, 3, 9, [(1, 2)])
    lines = []
    for i in range(len(rows)):
        seen = set(rows.chains[i])
        lines.append("".join("#" if j == i else "1" if j in seen else "."
                             for j in range(len(rows))))
    assert lines == ["#.......", "1#......", "11#.....", "1..#....", "11..#...",
                     "111..#..", "1.....#.", "1.....1#"]


def test_pool_matches_reference():
    g = load_golden("pool.json")
    for case in g["cases"]:
        p = lo.OraclePool(case["ngram"], capacity=case["capacity"])
        for op in case["ops"]:
            p.insert(op["insert"])
            lead, lim = op["lookup"]
            assert [list(s) for s in p.lookup(lead, lim)] == op["result"]
            assert len(p) == op["len"]
    for s in g["seeding"]:
        p = lo.OraclePool(s["ngram"])
        p.seed_from_prompt(s["prompt"])
        assert len(p) == s["len"]
        for t, res in s["lookups"].items():
            assert [list(x) for x in p.lookup(int(t), 100)] == res


def test_window_update_and_ngrams_match_reference():
    g = load_golden("window.json")
    for c in g["cases"]:
        W, N = c["W"], c["N"]
        flat = _levels_to_flat(c["levels"])
        grams = lo.collect_ngrams(flat, W, N, c["new_top"], c["last"])
        assert [list(x) for x in grams] == c["ngrams"]
        rng = np.random.default_rng(c["seed"])
        upd = lo.window_update(flat, W, N, c["V"], c["new_top"], c["k"], rng)
        assert _flat_to_levels(upd, W, N) == c["updated"]
        assert int(rng.integers(0, 2**31)) == c["next_draw"]


def test_rng_stream_pregeneration_equivalent():
    """the window's scalar draws equal one pre-generated array."""
    g = load_golden("window.json")
    for c in g["cases"]:
        W, N, V = c["W"], c["N"], c["V"]
        flat = _levels_to_flat(c["levels"])
        n = lo.window_draws(W, N, c["k"])
        stream = np.random.default_rng(c["seed"]).integers(0, V, size=n + 1)
        upd = lo.window_update(flat, W, N, V, c["new_top"], c["k"], np.random.default_rng(c["seed"]))
        # refills are the vacated cells, level-ascending then column-ascending
        s = c["k"] - 1
        refills = []
        idx = 0
        for level in range(N - 1):
            first = 2 if level == 0 else 1
            for col in range(first, W + 1):
                if col + s > W:
                    refills.append(upd[idx])
                idx += 1
        assert refills == [int(t) for t in stream[:n]]


def test_verify_greedy_matches_reference():
    g = load_golden("verify.json")
    for c in g["cases"]:
        cands = c["cands"]
        sufs = [tuple(s) for s, _ in cands]
        if not sufs:
            rows = lo.Rows([0], [0], [[]], [], [])
            acc, _ = lo.verify_greedy_rows(lambda r: int(np.argmax(c["base"])), rows, sufs)
            assert acc == c["accepted"]
            continue
        n_pos = len(sufs[0])
        # rows: 0 = base, branch b rows = dists 1..n_pos
        table = {0: int(np.argmax(c["base"]))}
        bases = []
        r = 1
        for _, ds in cands:
            bases.append(r)
            for k in range(1, n_pos + 1):
                table[r] = int(np.argmax(ds[k]))
                r += 1
        rows = lo.Rows([0] * r, [0] * r, [[]] * r, [], bases)
        acc, _ = lo.verify_greedy_rows(lambda x: table[x], rows, sufs)
        assert acc == c["accepted"]


@pytest.mark.parametrize("mseed,V", [(11, 12), (0, 256), (3, 16)])
def test_tiny_transformer_weights_and_forward(mseed, V):
    g = load_golden("forward_tiny.json")
    arr = np.load(GOLDEN / "forward_tiny.npz")
    m = TinyTransformerOracle(mseed, V)
    hits = 0
    for idx, case in enumerate(g["cases"]):
        if case["model"] != [mseed, V] or case.get("hand"):
            continue
        rows = lo.build_rows(_levels_to_flat(case["levels"]), case["W"], case["N"],
                             case["last"], [tuple(s) for s in case["suffixes"]])
        ref = arr[f"case{idx}"]
        for i in range(len(rows)):
            seq = case["prefix"] + [rows.ids[c] for c in rows.chains[i]] + [rows.ids[i]]
            np.testing.assert_array_equal(np.log(m.probs_seq(seq)), ref[i])
        hits += 1
    assert hits >= 1


def test_decode_matches_reference():
    g = load_golden("decode_tiny.json")
    models = {}
    for run in g["runs"]:
        mk = (run["model"]["seed"], run["model"]["vocab"])
        if mk[1] == 32000:
            continue  # covered on the GPU; the fp64 oracle is slow at V=32000
        if mk not in models:
            models[mk] = TinyTransformerOracle(*mk)
        res = lo.decode_lookahead(models[mk], run["prompt"], run["W"], run["N"], run["G"],
                                  run["max_tokens"], run["eos"], run["sampler_seed"],
                                  run["seed_pool"])
        assert res.tokens == run["tokens"]
        m = res.metrics()
        assert m["steps"] == run["metrics"]["steps"]
        assert {str(k): v for k, v in m["acceptance_histogram"].items()} == \
            run["metrics"]["acceptance_histogram"]
        assert m["total_queries"] == run["metrics"]["total_queries"]
        for st, ref in zip(res.steps, run["steps"]):
            assert st.accepted == ref["accepted"]
            assert st.new_top == ref["new_top"]
            assert (st.candidate_count, st.query_count, st.pool_size) == \
                (ref["c"], ref["M"], ref["pool"])
        if run["eos"] is None:
            assert lo.decode_autoregressive(models[mk], run["prompt"], run["max_tokens"]) == \
                run["ar_tokens"]


def test_lp_partition_matches_reference():
    g = load_golden("lp.json")
    for case in g["plans"]:
        ps = lo.lp_partition(case["W"], case["N"], case["D"], case["c"])
        for p, ref in zip(ps, case["plans"]):
            assert [p["columns"][0], p["columns"][-1] + 1] == ref["columns"]
            assert p["candidates"] == ref["candidates"]
            assert p["owned"] == ref["owned"]
            assert p["redundant"] == ref["redundant"]


def test_bf16_round_is_rne():
    x = np.array([1.0, 1.00390625, 1.01171875, -3.3, 65504.0], dtype=np.float32)
    import torch
    ref = torch.tensor(x).to(torch.bfloat16).to(torch.float32).numpy()
    np.testing.assert_array_equal(bf16_round(x), ref)


def test_jacobi_matches_reference():
    """Oracle restatement of decode_jacobi pinned to the reference's iterates."""
    g = load_golden("jacobi.json")
    models = {}
    for case in g["cases"]:
        if case["m"] > 16:
            continue   # longer chains are covered on the GPU (fp64 oracle recompute is slow)
        mk = tuple(case["model"])
        if mk not in models:
            models[mk] = TinyTransformerOracle(*mk)
        toks, iterates, iters = lo.decode_jacobi(models[mk], case["prompt"], case["m"],
                                                 np.random.default_rng(case["rng_seed"]))
        assert toks == case["tokens"]
        assert iterates == case["iterates"]
        assert iters == case["iterations"]
