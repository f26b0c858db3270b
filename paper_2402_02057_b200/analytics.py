"""Run metrics returned by the decode API (reference analytics.py:90-156)."""

from __future__ import annotations

from dataclasses import dataclass
from collections.abc import Sequence

from .types import StepRecord


def compression_ratio(tokens: int, steps: int) -> float:
    """Step compression S = generated tokens / decoding steps (Eq. 6)."""
    if steps < 1:
        raise ValueError("step count must be >= 1")
    return tokens / steps


def flops_proxy(window: int, ngram: int, max_candidates: int) -> int:
    """(W + G)(N - 1): extra input tokens per step (paper §5.5)."""
    if window < 1 or ngram < 2 or max_candidates < 0:
        raise ValueError("need W >= 1, N >= 2, G >= 0")
    return (window + max_candidates) * (ngram - 1)


@dataclass
class RunMetrics:
    tokens_generated: int
    steps: int
    compression: float
    acceptance_histogram: dict[int, int]
    total_queries: int
    mean_queries_per_step: float

    @classmethod
    def from_records(cls, tokens_generated: int, records: Sequence[StepRecord],
                     ngram: int) -> "RunMetrics":
        # histogram keys 1..N over *untruncated* accepted counts; compression over
        # the *truncated* token count (reference decoding.py:191-198,254-255)
        hist = dict.fromkeys(range(1, ngram + 1), 0)
        queries = 0
        for r in records:
            hist[r.accepted_count] += 1
            queries += r.query_count
        n = len(records)
        return cls(tokens_generated=tokens_generated, steps=n,
                   compression=compression_ratio(tokens_generated, n),
                   acceptance_histogram=hist, total_queries=queries,
                   mean_queries_per_step=queries / n)
