"""Step-layout value types for the ``ModelInterface.forward`` parity hook.

The decode hot path builds its layouts on the device (K1, ``la_state.cuh``
``la_step_build``).  These host types exist so a caller -- including the
reference's own orchestration -- can hand an explicit layout to a B200 model
(``models.B200Model.forward``), mirroring reference ``layout.py:33-80,185-194``.
Any object with ``.queries`` whose items carry ``token``, ``rel_pos`` and
``visible`` is accepted, so reference ``StepLayout`` objects work unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from collections.abc import Sequence

import numpy as np

from .types import LayoutError


@dataclass(frozen=True)
class QueryToken:
    token: int
    rel_pos: int
    visible: tuple[int, ...] = ()


@dataclass
class StepLayout:
    queries: list[QueryToken]
    window_cells: dict[tuple[int, int], int] = field(default_factory=dict)
    branch_slices: list[range] = field(default_factory=list)
    generators: tuple[int, ...] = ()

    def __len__(self) -> int:
        return len(self.queries)


@dataclass(frozen=True)
class CandidateBranch:
    suffix: tuple[int, ...]
    source: tuple[int, ...] = ()


def chain_layout(last_token: int, tokens: Sequence[int]) -> StepLayout:
    """Triangular chain: token i sees query 0 and every earlier token."""
    qs = [QueryToken(int(last_token), 0)]
    qs += [QueryToken(int(t), i, tuple(range(i))) for i, t in enumerate(tokens, start=1)]
    return StepLayout(queries=qs)


def layout_chains(layout) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(ids, rel, chain[M, max_rel]) of a layout, validated like the
    reference's ``conditioning_chain`` (models.py:33-64).

    chain[i, r] is the query index providing relative position r to query i.
    The device evaluates each query on top of the K/V of those queries, so the
    layout must also be chain-closed: a visible query's own chain must spell
    the same tokens as the prefix of the viewer's chain (always true for
    build_layout / chain_layout / partitioned layouts)."""
    qs = list(layout.queries)
    M = len(qs)
    if M == 0:
        raise LayoutError("empty layout")
    if qs[0].rel_pos != 0:
        raise LayoutError("query 0 must sit at relative position 0")
    ids = np.array([int(q.token) for q in qs], dtype=np.int32)
    rel = np.array([int(q.rel_pos) for q in qs], dtype=np.int32)
    width = max(1, int(rel.max()))
    chain = np.full((M, width), -1, dtype=np.int32)
    for i in range(1, M):
        q = qs[i]
        by_rel = {0: 0}
        tok_at = {0: int(qs[0].token)}
        for v in set(q.visible):
            if not 0 <= v < M or v == i:
                raise LayoutError(f"query {i} has out-of-range visible index {v}")
            r = int(qs[v].rel_pos)
            if r >= q.rel_pos:
                raise LayoutError(f"query {i} (rel_pos {q.rel_pos}) sees query {v} at rel_pos {r}")
            if r in tok_at and tok_at[r] != int(qs[v].token):
                raise LayoutError(f"query {i} sees two tokens at rel_pos {r}")
            tok_at[r] = int(qs[v].token)
            if r != 0 and (r not in by_rel or v < by_rel[r]):
                by_rel[r] = v
        for r in range(q.rel_pos):
            if r not in tok_at:
                raise LayoutError(f"query {i} has no visible token at rel_pos {r}")
            chain[i, r] = by_rel[r]
    # chain closure: the K/V a row reuses must come from the same token chain
    def tokens_of(i):
        return [int(ids[chain[i, r]]) for r in range(rel[i])] + [int(ids[i])]
    for i in range(M):
        mine = tokens_of(i)
        for r in range(1, rel[i]):
            v = chain[i, r]
            if tokens_of(v) != mine[: r + 1]:
                raise LayoutError(
                    f"query {i}: visible query {v} is not chain-closed (its own chain differs)")
    return ids, rel, chain
