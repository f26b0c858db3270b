"""Pin the sampling oracle (``oracle/sampling_oracle.py``) to numpy's PCG64
stream and to golden vectors produced by the reference's temperature sampler
(``oracle/make_golden.py sampling``).  CPU only."""

import numpy as np
import pytest

from oracle import sampling_oracle as so
from oracle.model_oracle import TinyTransformerOracle
from tests.conftest import load_golden


@pytest.mark.parametrize("seed", [0, 1, 7, 12345, 2**40 + 3])
def test_pcg64_matches_numpy(seed):
    ref = np.random.default_rng(seed)
    me = so.Pcg64.from_numpy(np.random.default_rng(seed))
    pick = np.random.default_rng(seed + 1)
    for i in range(400):
        op = int(pick.integers(0, 4))
        if op == 0:
            assert me.random() == ref.random()
        else:
            V = [2, 3, 256, 32000, 2**31 - 1, 7][int(pick.integers(0, 6))]
            if op == 3:   # array form (window_init) == consecutive scalars
                n = int(pick.integers(1, 9))
                assert [me.integers(V) for _ in range(n)] == ref.integers(0, V, size=n).tolist()
            else:
                assert me.integers(V) == int(ref.integers(0, V))
    s = ref.bit_generator.state
    assert (me.state, me.inc, me.has_uint32, me.uinteger) == (
        s["state"]["state"], s["state"]["inc"], s["has_uint32"], s["uinteger"])


def test_adjusted_distribution_matches_reference():
    for c in load_golden("sampling.json")["adjust"]:
        got = so.adjusted_distribution(np.array(c["probs"]), c["T"], c["top_k"], c["top_p"])
        np.testing.assert_array_equal(got, np.array(c["out"]))


def test_verify_sample_matches_reference():
    for c in load_golden("sampling.json")["verify"]:
        base = np.array(c["base"])
        sufs = [tuple(s) for s, _ in c["cands"]]
        dists = [[np.array(d) for d in ds] for _, ds in c["cands"]]
        rng = so.Pcg64.from_numpy(np.random.default_rng(c["seed"]))
        acc, _ = so.verify_sample(base, sufs, dists, rng)
        assert acc == c["accepted"]


def test_sampled_decodes_match_reference():
    g = load_golden("sampling.json")
    m = TinyTransformerOracle(0, 256)
    for c in g["decode"][:6]:
        run = so.decode_lookahead_sampled(m, c["prompt"], c["W"], c["N"], c["G"], c["max_tokens"],
                                          c["T"], c["top_k"], c["top_p"], seed=c["seed"])
        assert run.tokens == c["tokens"]
        assert [s.accepted for s in run.steps] == [s["accepted"] for s in c["steps"]]
        assert [s.new_top for s in run.steps] == [s["new_top"] for s in c["steps"]]
    for c in g["ar"][:2]:
        assert so.decode_autoregressive_sampled(m, c["prompt"], c["max_tokens"], c["T"],
                                                c["top_k"], c["top_p"], seed=c["seed"]) == c["tokens"]


def test_device_generator_host_build_matches_numpy():
    """la_pcg64_draws runs la_sample.cuh's PCG64 on the host (no GPU)."""
    import ctypes as C
    from paper_2402_02057_b200 import _lib
    lib = _lib.load()
    for seed in (0, 3, 99):
        ref = np.random.default_rng(seed)
        ref.integers(0, 256, size=7)          # leave a buffered upper half behind
        smp = _lib.make_sampler(1.0, None, None, ref)
        out = np.zeros(64, dtype=np.float64)
        _lib.check(lib.la_pcg64_draws(C.byref(smp), 1, 256, 64, out.ctypes.data))
        assert out.astype(int).tolist() == ref.integers(0, 256, size=64).tolist()
        smp = _lib.make_sampler(1.0, None, None, ref)
        _lib.check(lib.la_pcg64_draws(C.byref(smp), 0, 0, 64, out.ctypes.data))
        assert out.tolist() == [ref.random() for _ in range(64)]
        smp = _lib.make_sampler(1.0, None, None, ref)
        _lib.check(lib.la_pcg64_draws(C.byref(smp), 1, 32000, 64, out.ctypes.data))
        assert out.astype(int).tolist() == [int(ref.integers(0, 32000)) for _ in range(64)]
