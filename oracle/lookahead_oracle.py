"""CPU oracle for the greedy lookahead step (TEST INFRASTRUCTURE ONLY).

A numpy / plain-Python restatement of the reference's hot path, written on
the flat row geometry the device uses so that per-step device outputs can be
compared field by field.  Every function cites the reference code it
restates (paths relative to ``/root/reference/pkg/src/lookahead``).

Flat geometry:

* the 2-D window is one int array of (N-1)*W - 1 cells: level 0 holds
  columns 2..W, every later level columns 1..W (``layout.py:83-114``);
* window cell ``f`` is step row ``f + 1``; row 0 is query 0;
* branch ``b`` offset ``k`` (1..N-1) is row ``(N-1)*W + b*(N-1) + k - 1``.
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np


# ---------------------------------------------------------------- pool
class OraclePool:
    """Restates ``NGramPool`` (``pool.py:17-90``): per-lead recency buckets,
    dedup with refresh, optional global LRU capacity."""

    def __init__(self, ngram: int, capacity: int | None = None):
        if ngram < 2:
            raise ValueError("n-gram size must be >= 2")
        self.ngram = ngram
        self.capacity = capacity
        self._order: "OrderedDict[tuple, None]" = OrderedDict()   # global, oldest first
        self._lead: dict[int, "OrderedDict[tuple, None]"] = {}      # per lead, oldest first

    def __len__(self) -> int:
        return len(self._order)

    def insert(self, gram) -> None:                                  # pool.py:41-61
        g = tuple(int(t) for t in gram)
        if len(g) != self.ngram:
            raise ValueError("wrong n-gram length")
        lead, suf = g[0], g[1:]
        if g in self._order:
            self._order.move_to_end(g)
            self._lead[lead].move_to_end(suf)
            return
        if self.capacity is not None and len(self._order) >= self.capacity:
            old, _ = self._order.popitem(last=False)
            bucket = self._lead[old[0]]
            del bucket[old[1:]]
            if not bucket:
                del self._lead[old[0]]
        self._order[g] = None
        self._lead.setdefault(lead, OrderedDict())[suf] = None

    def insert_all(self, grams) -> None:                             # pool.py:63-67
        for g in grams:
            self.insert(g)

    def lookup(self, last: int, limit: int) -> list[tuple]:          # pool.py:69-81
        if limit <= 0:
            return []
        bucket = self._lead.get(int(last))
        if not bucket:
            return []
        return list(reversed(bucket))[:limit]

    def seed_from_prompt(self, prompt) -> None:                      # pool.py:83-90
        n = self.ngram
        for i in range(len(prompt) - n + 1):
            self.insert(prompt[i:i + n])

    def entries_oldest_first(self) -> list[tuple]:
        return list(self._order)


# ------------------------------------------------------------ geometry
def window_cells(W: int, N: int) -> int:
    return (N - 1) * W - 1


def cell_level_col(f: int, W: int) -> tuple[int, int]:
    if f < W - 1:
        return 0, f + 2
    f2 = f - (W - 1)
    return 1 + f2 // W, 1 + f2 % W


def cell_index(level: int, col: int, W: int) -> int:
    return col - 2 if level == 0 else (W - 1) + (level - 1) * W + (col - 1)


def window_init(W: int, N: int, V: int, rng: np.random.Generator) -> list[int]:
    """``layout.py:117-125``: level by level, uniform draws."""
    out: list[int] = []
    for level in range(N - 1):
        n = W - 1 if level == 0 else W
        out.extend(int(t) for t in rng.integers(0, V, size=n))
    return out


@dataclass
class Rows:
    """One step's query rows (``layout.py:128-182`` restated on flat rows)."""

    ids: list[int]
    rel: list[int]
    chains: list[list[int]]          # visible row per rel_pos 0..rel-1 (chain order)
    generators: list[int]            # row producing new_top of column j=1..W
    branch_base: list[int]           # first row of each branch
    W: int = 0
    N: int = 0

    def __len__(self) -> int:
        return len(self.ids)


def build_rows(window: list[int], W: int, N: int, last: int, suffixes) -> Rows:
    ids = [int(last)]
    rel = [0]
    chains: list[list[int]] = [[]]
    for f, tok in enumerate(window):
        level, col = cell_level_col(f, W)
        ids.append(int(tok))
        r = col + level - 1
        rel.append(r)
        if level == 0:                     # oldest row: q0 + level-0 cells left of col
            chains.append(list(range(0, col - 1)))
        else:                              # q0 + level-0 cols 2..col + same column below
            ch = list(range(0, col))
            ch += [cell_index(m, col, W) + 1 for m in range(1, level)]
            chains.append(ch)
    bases = []
    for s in suffixes:
        if len(s) != N - 1:
            raise ValueError("candidate suffix must have N-1 tokens")
        base = len(ids)
        bases.append(base)
        for k, tok in enumerate(s, start=1):
            ids.append(int(tok))
            rel.append(k)
            chains.append([0] + list(range(base, base + k - 1)))
    top = N - 2
    gens = []
    for col in range(1, W + 1):
        if top == 0 and col == 1:
            gens.append(0)
        else:
            gens.append(cell_index(top, col, W) + 1)
    return Rows(ids, rel, chains, gens, bases, W, N)


def collect_ngrams(window: list[int], W: int, N: int, new_top, last: int) -> list[tuple]:
    """``layout.py:197-216``: one n-gram per column from the OLD window."""
    grams = []
    for col in range(1, W + 1):
        g = [int(last)] if col == 1 else [window[cell_index(0, col, W)]]
        g += [window[cell_index(level, col, W)] for level in range(1, N - 1)]
        g.append(int(new_top[col - 1]))
        grams.append(tuple(g))
    return grams


def window_update(window: list[int], W: int, N: int, V: int, new_top, k: int,
                  rng: np.random.Generator) -> list[int]:
    """``layout.py:219-252``: drop level 0, append new_top, shift by k-1,
    refill vacated cells level-ascending / column-ascending."""
    if not 1 <= k <= N:
        raise ValueError("accepted count out of range")
    s = k - 1
    sources = []
    for level in range(1, N - 1):
        sources.append([window[cell_index(level, c, W)] for c in range(1, W + 1)])
    sources.append([int(t) for t in new_top])
    out: list[int] = []
    for level, src in enumerate(sources):
        first = 2 if level == 0 else 1
        for col in range(first, W + 1):
            c = col + s
            out.append(src[c - 1] if c <= W else int(rng.integers(0, V)))
    return out


def window_draws(W: int, N: int, k: int) -> int:
    """RNG draws one window_update consumes."""
    s = k - 1
    return min(s, W - 1) + (N - 2) * min(s, W)


# -------------------------------------------------------- verification
def greedy_argmax(x: np.ndarray) -> int:
    """``sampling.py:17-19``: lowest index attaining the maximum."""
    return int(np.argmax(x))


def verify_greedy_rows(argmax_of_row, rows: Rows, suffixes) -> tuple[list[int], int]:
    """``verification.py:43-71`` on per-row argmax ids.

    Returns (accepted tokens, first surviving branch or -1)."""
    if not suffixes:
        return [argmax_of_row(0)], -1
    n_pos = len(suffixes[0])
    alive = list(range(len(suffixes)))
    out: list[int] = []
    for i in range(n_pos):
        lead = alive[0]
        row = 0 if i == 0 else rows.branch_base[lead] + i - 1
        target = argmax_of_row(row)
        keep = [b for b in alive if suffixes[b][i] == target]
        out.append(target)
        if not keep:
            return out, -1
        alive = keep
    lead = alive[0]
    out.append(argmax_of_row(rows.branch_base[lead] + n_pos - 1))
    return out, lead


# --------------------------------------------------------- decode loop
@dataclass
class StepLog:
    accepted: list[int]
    new_top: list[int]
    candidate_count: int
    query_count: int
    pool_size: int
    winner: int
    window_before: list[int] = field(default_factory=list)


@dataclass
class OracleRun:
    tokens: list[int]
    steps: list[StepLog]
    ngram: int

    def metrics(self) -> dict:
        """``analytics.py:142-156`` (RunMetrics.from_records)."""
        hist = {k: 0 for k in range(1, self.ngram + 1)}
        for s in self.steps:
            hist[len(s.accepted)] += 1
        tq = sum(s.query_count for s in self.steps)
        n = len(self.steps)
        return dict(tokens_generated=len(self.tokens), steps=n,
                    compression=len(self.tokens) / n, acceptance_histogram=hist,
                    total_queries=tq, mean_queries_per_step=tq / n)


def fold_output(out: list[int], accepted, max_tokens: int, eos) -> bool:
    """``decoding.py:214-232``."""
    for t in accepted:
        out.append(int(t))
        if eos is not None and t == eos:
            return True
        if len(out) >= max_tokens:
            return True
    return False


def decode_lookahead(model, prompt, W: int, N: int, G: int | None, max_tokens: int,
                     eos=None, seed: int = 0, seed_pool: bool = False,
                     pool: OraclePool | None = None) -> OracleRun:
    """``decoding.py:235-255`` + ``start_session`` ``:67-93`` +
    ``lookahead_step`` ``:207-211`` (greedy)."""
    if not len(prompt):
        raise ValueError("prompt must be nonempty")
    G = W if G is None else G
    V = model.vocab_size
    pool = OraclePool(N) if pool is None else pool
    if seed_pool:
        pool.seed_from_prompt([int(t) for t in prompt])
    rng = np.random.default_rng(seed)
    window = window_init(W, N, V, rng)
    prefix = [int(t) for t in prompt]
    out: list[int] = []
    steps: list[StepLog] = []
    done = False
    while not done:
        last = prefix[-1]
        sufs = pool.lookup(last, G)
        rows = build_rows(window, W, N, last, sufs)
        am = model.argmax_rows(prefix[:-1], rows)
        new_top = [am[g] for g in rows.generators]
        acc, win = verify_greedy_rows(lambda r: am[r], rows, sufs)
        pool.insert_all(collect_ngrams(window, W, N, new_top, last))
        wb = list(window)
        window = window_update(window, W, N, V, new_top, len(acc), rng)
        prefix.extend(acc)
        steps.append(StepLog(acc, new_top, len(sufs), len(rows), len(pool), win, wb))
        done = fold_output(out, acc, max_tokens, eos)
    return OracleRun(out, steps, N)


def decode_autoregressive(model, prompt, max_tokens: int, eos=None) -> list[int]:
    """``decoding.py:96-116`` (greedy: no RNG use)."""
    if not len(prompt):
        raise ValueError("prompt must be nonempty")
    prefix = [int(t) for t in prompt]
    out: list[int] = []
    while len(out) < max_tokens:
        rows = Rows([prefix[-1]], [0], [[]], [], [])
        tok = model.argmax_rows(prefix[:-1], rows)[0]
        out.append(tok)
        prefix.append(tok)
        if eos is not None and tok == eos:
            break
    return out


def decode_jacobi(model, prompt, m: int, rng: np.random.Generator):
    """``decoding.py:119-149``: random initial guess from ``rng``, then
    parallel fixed-point iteration over the triangular chain layout
    (``layout.py:185-194``: token i sees query 0 and the tokens before it).
    Returns (tokens, iterates incl. the guess, iterations)."""
    if not len(prompt):
        raise ValueError("prompt must be nonempty")
    if m < 1:
        raise ValueError("generation length m must be >= 1")
    prefix = [int(t) for t in prompt]
    current = [int(t) for t in rng.integers(0, model.vocab_size, size=m)]
    iterates = [list(current)]
    iterations = 0
    new = current
    for _ in range(m):
        rows = Rows([prefix[-1]] + current, list(range(m + 1)),
                    [list(range(i)) for i in range(m + 1)], [], [])
        new = model.argmax_rows(prefix[:-1], rows)[:m]
        iterations += 1
        iterates.append(list(new))
        if new == current:
            break
        current = new
    return new, iterates, iterations


# ------------------------------------------------ lookahead parallelism
def lp_partition(W: int, N: int, D: int, n_cand: int) -> list[dict]:
    """``parallel.py:64-116``: contiguous column ranges (sizes differ by <=1),
    candidates round-robin, redundant q0 + level-0 cells left of the range."""
    if not 1 <= D <= W:
        raise ValueError("device count must lie in [1, W]")
    base, extra = divmod(W, D)
    plans = []
    start = 1
    for d in range(D):
        size = base + (1 if d < extra else 0)
        cols = list(range(start, start + size))
        start += size
        owned = [cell_index(l, c, W) + 1 for l in range(N - 1) for c in cols
                 if not (l == 0 and c == 1)]
        redundant = [cell_index(0, c, W) + 1 for c in range(2, cols[0])]
        if d == 0:
            owned.insert(0, 0)
        else:
            redundant.insert(0, 0)
        plans.append(dict(device=d, columns=cols, candidates=[], owned=owned,
                          redundant=redundant))
    for i in range(n_cand):
        p = plans[i % D]
        p["candidates"].append(i)
        b0 = (N - 1) * W + i * (N - 1)
        p["owned"].extend(range(b0, b0 + N - 1))
    return plans


def lp_tokens_synchronized(W: int, N: int, D: int, n_cand: int) -> int:
    """``parallel.py:164,168``: per-step token accounting."""
    per = 0
    for p in lp_partition(W, N, D, n_cand):
        per += len(p["columns"]) + len(p["candidates"]) * N
    return per * (D - 1)
