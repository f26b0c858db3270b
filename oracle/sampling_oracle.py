"""CPU oracle for SAMPLING verification (TEST INFRASTRUCTURE ONLY).

Restates the reference's temperature sampler and distribution-preserving
verification (paths relative to ``/root/reference/pkg/src/lookahead``):

* ``adjusted_distribution`` -- ``sampling.py:22-66`` (temperature power,
  top-k, top-p nucleus over the (-p, id) order, renormalise);
* ``draw`` -- ``sampling.py:69-74`` (inverse CDF, searchsorted right);
* ``verify_sample`` -- ``verification.py:74-118``;
* ``decode_lookahead_sampled`` / ``decode_autoregressive_sampled`` --
  ``decoding.py:96-116,160-204`` with a temperature ``SamplerSpec``.

The randomness is numpy's ``default_rng(seed)`` (PCG64).  ``Pcg64`` below
restates the bit generator and the two Generator methods the reference
calls -- ``random()`` (53-bit double) and ``integers(0, V)`` (32-bit
Lemire rejection with the bit generator's buffered upper half) -- in plain
Python integers.  It is the specification of the device generator
(``la_sample.cuh``) and is pinned against numpy itself in the tests.
"""

from __future__ import annotations

import numpy as np

M128 = (1 << 128) - 1
M64 = (1 << 64) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645   # PCG_DEFAULT_MULTIPLIER_128


class Pcg64:
    """numpy.random.PCG64 + Generator.random / integers(0, V) (scalar)."""

    def __init__(self, state: int, inc: int, has_uint32: int = 0, uinteger: int = 0):
        self.state, self.inc = state & M128, inc & M128
        self.has_uint32, self.uinteger = int(has_uint32), int(uinteger) & 0xFFFFFFFF

    @classmethod
    def from_numpy(cls, rng: np.random.Generator) -> "Pcg64":
        s = rng.bit_generator.state
        return cls(s["state"]["state"], s["state"]["inc"], s["has_uint32"], s["uinteger"])

    def next64(self) -> int:
        # step, then XSL-RR output of the new state
        self.state = (self.state * PCG_MULT + self.inc) & M128
        hi, lo = self.state >> 64, self.state & M64
        x, rot = hi ^ lo, hi >> 58
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next32(self) -> int:
        if self.has_uint32:
            self.has_uint32 = 0
            return self.uinteger
        v = self.next64()
        self.has_uint32, self.uinteger = 1, v >> 32
        return v & 0xFFFFFFFF

    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def integers(self, high: int) -> int:
        """integers(0, high) for 1 < high <= 2**32 - 1 (Lemire, 32-bit path)."""
        rng = high - 1
        if rng == 0:
            return 0
        excl = rng + 1
        m = self.next32() * excl
        left = m & 0xFFFFFFFF
        if left < excl:
            thr = (0xFFFFFFFF - rng) % excl
            while left < thr:
                m = self.next32() * excl
                left = m & 0xFFFFFFFF
        return m >> 32


class DegenerateDistribution(ValueError):
    """types.DegenerateDistributionError."""


def adjusted_distribution(probs, temperature: float = 1.0, top_k=None, top_p=None) -> np.ndarray:
    """``sampling.py:22-66`` (temperature mode)."""
    p = np.asarray(probs, dtype=np.float64)
    p = np.power(p, 1.0 / temperature) if temperature != 1.0 else p.copy()
    order = np.lexsort((np.arange(p.size), -p))
    if top_k is not None and top_k < p.size:
        q = np.zeros_like(p)
        q[order[:top_k]] = p[order[:top_k]]
        p = q
    if top_p is not None and top_p < 1.0:
        cum = np.cumsum(p[order])
        if cum[-1] <= 0.0:
            raise DegenerateDistribution("no probability mass before nucleus truncation")
        cut = min(int(np.searchsorted(cum, top_p * cum[-1], side="left")), p.size - 1)
        q = np.zeros_like(p)
        q[order[:cut + 1]] = p[order[:cut + 1]]
        p = q
    t = p.sum()
    if t <= 0.0:
        raise DegenerateDistribution("all probability mass truncated away")
    return p / t


def draw(p: np.ndarray, rng: Pcg64) -> int:
    """``sampling.py:69-74``."""
    u = rng.random()
    cum = np.cumsum(p)
    return min(int(np.searchsorted(cum, u * cum[-1], side="right")), p.shape[0] - 1)


def verify_sample(base: np.ndarray, suffixes, dists, rng: Pcg64) -> tuple[list[int], int]:
    """``verification.py:74-118``; ``dists[j]`` = [base, d_1 .. d_{N-1}] of
    candidate j.  Returns (accepted tokens, first surviving candidate or -1)."""
    if not suffixes:
        return [draw(base, rng)], -1
    alive = list(range(len(suffixes)))
    S = len(suffixes[0])
    out: list[int] = []
    for i in range(S):
        p = np.array(dists[alive[0]][i], dtype=np.float64)
        ok = False
        j = 0
        while j < len(alive):
            s = suffixes[alive[j]][i]
            r = rng.random()
            if p[s] > 0.0 and r <= p[s]:
                out.append(int(s))
                ok = True
                alive = [b for b in alive[j:] if suffixes[b][i] == s]
                break
            p[s] = 0.0
            t = p.sum()
            if t <= 0.0:
                raise DegenerateDistribution("verification renormalized to zero mass")
            p = p / t
            j += 1
        if not ok:
            out.append(draw(p, rng))
            return out, (alive[0] if i > 0 else -1)
    out.append(draw(dists[alive[0]][S], rng))
    return out, alive[0]


def _softmax64(logits) -> np.ndarray:
    x = np.asarray(logits, dtype=np.float64)
    e = np.exp(x - x.max())
    return e / e.sum()


def decode_lookahead_sampled(model, prompt, W: int, N: int, G: int | None, max_tokens: int,
                             temperature: float = 1.0, top_k=None, top_p=None, eos=None,
                             seed: int = 0, seed_pool: bool = False):
    """``decoding.py:235-255`` with a temperature SamplerSpec: greedy
    generators, sampling verification, window refills from the same rng."""
    from .lookahead_oracle import (OraclePool, OracleRun, StepLog, build_rows, collect_ngrams,
                                   fold_output, window_cells, window_update)
    if not len(prompt):
        raise ValueError("prompt must be nonempty")
    G = W if G is None else G
    V = model.vocab_size
    pool = OraclePool(N)
    if seed_pool:
        pool.seed_from_prompt([int(t) for t in prompt])
    npr = np.random.default_rng(seed)
    window = [int(t) for t in npr.integers(0, V, size=window_cells(W, N))]
    rng = Pcg64.from_numpy(npr)
    adj = lambda l: adjusted_distribution(_softmax64(l), temperature, top_k, top_p)  # noqa: E731
    prefix = [int(t) for t in prompt]
    out: list[int] = []
    steps: list[StepLog] = []
    done = False
    while not done:
        last = prefix[-1]
        sufs = pool.lookup(last, G)
        rows = build_rows(window, W, N, last, sufs)
        lg = model.logits_rows(prefix[:-1], rows)
        new_top = [int(np.argmax(lg[g])) for g in rows.generators]
        base = adj(lg[0])
        dists = [[base] + [adj(lg[rows.branch_base[b] + k]) for k in range(N - 1)]
                 for b in range(len(sufs))]
        acc, win = verify_sample(base, sufs, dists, rng)
        pool.insert_all(collect_ngrams(window, W, N, new_top, last))
        wb = list(window)
        window = window_update(window, W, N, V, new_top, len(acc), _NumpyFacade(rng))
        prefix.extend(acc)
        steps.append(StepLog(acc, new_top, len(sufs), len(rows), len(pool), win, wb))
        done = fold_output(out, acc, max_tokens, eos)
    run = OracleRun(out, steps, N)
    run.rng_state = {"bit_generator": "PCG64", "state": {"state": rng.state, "inc": rng.inc},
                     "has_uint32": rng.has_uint32, "uinteger": rng.uinteger}
    return run


def decode_autoregressive_sampled(model, prompt, max_tokens: int, temperature: float = 1.0,
                                  top_k=None, top_p=None, eos=None, seed: int = 0) -> list[int]:
    """``decoding.py:96-116`` + ``sample_token`` (``sampling.py:77-85``)."""
    from .lookahead_oracle import Rows
    if not len(prompt):
        raise ValueError("prompt must be nonempty")
    rng = Pcg64.from_numpy(np.random.default_rng(seed))
    prefix = [int(t) for t in prompt]
    out: list[int] = []
    while len(out) < max_tokens:
        lg = model.logits_rows(prefix[:-1], Rows([prefix[-1]], [0], [[]], [], []))[0]
        tok = draw(adjusted_distribution(_softmax64(lg), temperature, top_k, top_p), rng)
        out.append(tok)
        prefix.append(tok)
        if eos is not None and tok == eos:
            break
    return out


class _NumpyFacade:
    """``rng.integers(0, V)`` on a Pcg64 (what window_update calls)."""

    def __init__(self, g: Pcg64):
        self.g = g

    def integers(self, low: int, high: int) -> int:
        return low + self.g.integers(high - low)
