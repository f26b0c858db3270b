"""Host container for an n-gram pool passed into / out of a decode.

The decode itself runs on the GPU-resident pool (``csrc/la_state.cuh``).
This class only carries a caller's pool across the API boundary with the
reference's observable semantics (``pool.py:17-90``): per-lead recency,
dedup-with-refresh, ``len()`` = distinct n-grams.  After a decode the engine's
insert log is replayed into it, exactly as the reference mutates a
caller-supplied pool.
"""

from __future__ import annotations

from collections import OrderedDict
from collections.abc import Iterable, Sequence


class NGramPool:
    def __init__(self, ngram: int, capacity: int | None = None):
        if ngram < 2:
            raise ValueError("n-gram size must be >= 2")
        if capacity is not None and capacity < 1:
            raise ValueError("capacity must be a positive integer")
        self.ngram = ngram
        self.capacity = capacity
        self.insertion_counter = 0
        self._recency: "OrderedDict[tuple[int, ...], int]" = OrderedDict()  # full n-gram -> stamp

    def __len__(self) -> int:
        return len(self._recency)

    def insert(self, gram: Sequence[int]) -> None:
        key = tuple(int(t) for t in gram)
        if len(key) != self.ngram:
            raise ValueError(f"expected {self.ngram}-gram, got {len(key)} tokens")
        self.insertion_counter += 1
        if key in self._recency:
            self._recency.move_to_end(key)
        elif self.capacity is not None and len(self._recency) >= self.capacity:
            self._recency.popitem(last=False)
        self._recency[key] = self.insertion_counter

    def insert_all(self, grams: Iterable[Sequence[int]]) -> None:
        for g in grams:
            self.insert(g)

    def lookup(self, last_token: int, limit: int) -> list[tuple[int, ...]]:
        if limit <= 0:
            return []
        lead = int(last_token)
        hits: list[tuple[int, ...]] = []
        for key in reversed(self._recency):
            if key[0] == lead:
                hits.append(key[1:])
                if len(hits) == limit:
                    break
        return hits

    def seed_from_prompt(self, prompt: Sequence[int]) -> None:
        n = self.ngram
        for start in range(0, len(prompt) - n + 1):
            self.insert(prompt[start:start + n])

    def entries_oldest_first(self) -> list[tuple[int, ...]]:
        return list(self._recency)
