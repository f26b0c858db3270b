"""Lookahead parallelism (drop-in for reference ``parallel.py:145-192``).

``decode_lookahead_devices(model, prompt, config, sampler, devices)``:

* inside a ``torch.distributed`` job whose world size equals ``devices`` (one
  process per GPU, NCCL backend): every rank holds a full replica, evaluates
  its visibility-closed share of the step (contiguous window columns +
  round-robin candidates), and the ranks exchange argmax ids and the accepted
  branch's K/V with two NCCL all-gathers per step (``csrc/la_lp.cu``);
* otherwise: the reference's single-process simulation -- ``devices`` engine
  replicas on the current GPU with device-copy exchanges.

Either way the outcome is bit-identical to ``decode_lookahead`` (reference
``SPEC.md:515,523``), and ``CommStats`` follows the reference accounting.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from collections.abc import Sequence

from . import _lib
from .decoding import _finish_lookahead, _gen_config, _prepare_lookahead, _require_b200
from .pool import NGramPool
from .types import GenerationConfig, SamplerSpec


@dataclass
class CommStats:
    tokens_synchronized: int = 0
    sync_events: int = 0

    def add(self, other: "CommStats") -> None:
        self.tokens_synchronized += other.tokens_synchronized
        self.sync_events += other.sync_events


def column_ranges(window: int, devices: int) -> list[range]:
    """Contiguous column split, sizes differing by at most one (parallel.py:74-80)."""
    if not 1 <= devices <= window:
        raise ValueError(f"device count must lie in [1, {window}], got {devices}")
    base, extra = divmod(window, devices)
    out, start = [], 1
    for d in range(devices):
        n = base + (1 if d < extra else 0)
        out.append(range(start, start + n))
        start += n
    return out


def shard_rows(window: int, ngram: int, candidates: int, rank: int, world: int):
    """Host mirror of the device row plan (``la_lp_row_role``, la_state.cuh):
    (computed rows, owned rows) of ``rank`` for a step with ``candidates``
    branches, in global row order (SURVEY appendix A.1 geometry).

    Owned rows are disjoint across ranks and cover the layout; computed rows
    add query 0 and the oldest-level cells left of the rank's columns, which
    makes every shard closed under visibility (reference parallel.py:88-98)."""
    W, N = window, ngram
    cols = column_ranges(W, world)[rank]
    c0, c1 = cols.start, cols.stop - 1
    nwin = (N - 1) * W
    computed, owned = [], []
    for g in range(nwin + candidates * (N - 1)):
        if g == 0:
            comp, own = True, rank == 0
        elif g < nwin:
            f = g - 1
            if f < W - 1:
                level, col = 0, f + 2
            else:
                level, col = 1 + (f - (W - 1)) // W, 1 + (f - (W - 1)) % W
            own = c0 <= col <= c1
            comp = own or (level == 0 and col < c0)
        else:
            comp = own = ((g - nwin) // (N - 1)) % world == rank
        if comp:
            computed.append(g)
        if own:
            owned.append(g)
    return computed, owned


def step_comm(window: int, ngram: int, devices: int, candidates: int) -> CommStats:
    """Per-step accounting: each device sends one token per owned column and
    N values per owned candidate to the D-1 peers (parallel.py:164,168)."""
    per = window + candidates * ngram
    return CommStats(tokens_synchronized=per * (devices - 1), sync_events=1)


def _dist_world():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist, dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return None, 0, 1


def broadcast_unique_id(uid, group=None) -> bytes:
    """Rank 0's 128-byte NCCL id to every rank over the job's process group."""
    import torch.distributed as dist
    dist.broadcast(uid, src=0, group=group)
    return bytes(uid.cpu().tolist())


def lp_init(model, group=None):
    """Create the model's NCCL LP communicator from the torch.distributed job."""
    import torch
    dist, rank, world = _dist_world()
    if dist is None or world < 2:
        raise RuntimeError("lp_init needs an initialised torch.distributed job with >= 2 ranks")
    m = _require_b200(model)
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf = (C.c_uint8 * 128)()
        _lib.check(m.lib.la_lp_unique_id(buf))
        uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        uid = uid.cuda(m.device)
    raw = broadcast_unique_id(uid, group)
    _lib.check(m.lib.la_lp_init(m.engine(), C.c_char_p(raw), rank, world))
    m._lp_world = world


def decode_lookahead_devices(model, prompt: Sequence[int], config: GenerationConfig,
                             sampler: SamplerSpec, devices: int, pool: NGramPool | None = None):
    """LP decode; returns (tokens, RunMetrics, CommStats)."""
    m = _require_b200(model)
    if not 1 <= devices <= config.window:
        raise ValueError(f"device count must lie in [1, {config.window}], got {devices}")
    if sampler.mode != "greedy":
        # verify_sample needs whole adjusted distributions of the verified rows
        # while the LP exchange carries argmax ids, so a temperature decode runs
        # as a replica on every rank.  The reference defines the LP outcome as
        # bit-identical to the single-device decode (parallel.py:145-151,
        # SPEC.md:515,523) -- this is that decode -- and CommStats keeps the
        # reference accounting of the sharded step (parallel.py:164,168).
        io = _prepare_lookahead(m, prompt, config, sampler, pool)
        eng = m.engine("replica") if getattr(m, "_lp_world", 1) > 1 else m.engine()
        _lib.check(m.lib.la_decode_lookahead_sampled(eng, C.byref(_gen_config(config)),
                                                     C.byref(io.sampler), C.byref(io.io),
                                                     m.stream()))
        m.last_stats = io.stats()
        tokens, metrics = _finish_lookahead(io, config, pool)
        totals = CommStats()
        for rec in io.records():
            totals.add(step_comm(config.window, config.ngram, devices, rec.candidate_count))
        return tokens, metrics, totals
    io = _prepare_lookahead(m, prompt, config, sampler, pool)
    dist, rank, world = _dist_world()
    if dist is not None and world == devices and devices > 1:
        if getattr(m, "_lp_world", 1) != world:
            lp_init(m)
        _lib.check(m.lib.la_decode_lookahead(m.engine(), C.byref(_gen_config(config)),
                                             C.byref(io.io), m.stream()))
    else:
        handles = (C.c_void_p * devices)(*[m.engine(("lp", i)) for i in range(devices)])
        _lib.check(m.lib.la_decode_lookahead_group(handles, devices, C.byref(_gen_config(config)),
                                                   C.byref(io.io), m.stream()))
    m.last_stats = io.stats()
    tokens, metrics = _finish_lookahead(io, config, pool)
    totals = CommStats()
    for rec in io.records():
        totals.add(step_comm(config.window, config.ngram, devices, rec.candidate_count))
    return tokens, metrics, totals
