"""Decode API (drop-in for reference ``decoding.py:96-116,235-255``).

``decode_lookahead`` uploads the prompt, the window's RNG stream and any
caller pool once, runs every lookahead step on the GPU (device-resident
window, n-gram pool, KV cache; no token returns to the host inside the
loop), then reads the tokens, per-step records and pool log once.

Both samplers of the reference run on the device.  Greedy: argmax ids, the
window's random stream pre-generated on the host.  Temperature
(``SamplerSpec(mode="temperature")``): the host draws only the initial window
from ``default_rng(seed)`` exactly like ``start_session`` and hands the
generator state to the device, which consumes the identical PCG64 stream for
verify_sample's trials / draws and the window refills (``la_sample.cuh``).
"""

from __future__ import annotations

import ctypes as C
import weakref
from collections.abc import Sequence

import numpy as np

from . import _lib
from .analytics import RunMetrics
from .models import B200Model
from .pool import NGramPool
from .types import (GenerationConfig, JacobiTrajectory, SamplerSpec, StepOutcome, StepRecord,
                    Window2D)


def window_rng_draws(window: int, ngram: int, max_tokens: int) -> int:
    """Length of the pre-generated window stream:
    (N-1)W-1 initial cells plus, per step with shift s <= N-1,
    min(s, W-1) + (N-2) min(s, W) refills; at most max_tokens steps."""
    s = ngram - 1
    per_step = min(s, window - 1) + (ngram - 2) * min(s, window)
    return (ngram - 1) * window - 1 + max_tokens * per_step


def window_rng_stream(seed: int, vocab: int, window: int, ngram: int, max_tokens: int) -> np.ndarray:
    """``default_rng(seed).integers(0, V, size=R)``: the reference draws the
    window's cells from one generator (layout.py:117-125, 243-250), and array
    and scalar ``integers`` calls consume the same stream."""
    n = window_rng_draws(window, ngram, max_tokens)
    return np.random.default_rng(seed).integers(0, vocab, size=max(n, 1)).astype(np.int32)


def _require_b200(model) -> B200Model:
    if not isinstance(model, B200Model):
        raise TypeError("the B200 decode path needs a paper_2402_02057_b200 model "
                        f"(got {type(model).__name__})")
    return model


def _device_sampler(sampler: SamplerSpec, rng: np.random.Generator) -> _lib.la_sampler:
    return _lib.make_sampler(sampler.temperature, sampler.top_k, sampler.top_p, rng)


def _prompt(prompt) -> np.ndarray:
    if not len(prompt):
        raise ValueError("prompt must be nonempty")
    return np.ascontiguousarray(np.asarray([int(t) for t in prompt], dtype=np.int32))


class _IO:
    """Owns the host buffers behind one la_decode_io struct."""

    def __init__(self, prompt: np.ndarray, max_tokens: int, rng: np.ndarray | None = None,
                 pool_init: np.ndarray | None = None, ngram: int = 2, log_cap: int = 0):
        P32 = C.POINTER(C.c_int32)
        self.prompt = prompt
        self.rng = rng
        self.sampler = None
        self.pool_init = pool_init
        self.out = np.zeros(max_tokens, dtype=np.int32)
        self.rec = np.zeros((max_tokens + 1, 4), dtype=np.int32)
        self.log = np.zeros((max(log_cap, 1), ngram), dtype=np.int32)
        io = _lib.la_decode_io()
        io.prompt = prompt.ctypes.data_as(P32)
        io.n_prompt = len(prompt)
        if rng is not None:
            io.rng_stream = rng.ctypes.data_as(P32)
            io.rng_len = len(rng)
        if pool_init is not None and len(pool_init):
            io.pool_init = pool_init.ctypes.data_as(P32)
            io.pool_init_n = len(pool_init)
        io.out_tokens = self.out.ctypes.data_as(P32)
        io.out_cap = max_tokens
        io.step_records = self.rec.ctypes.data_as(P32)
        io.rec_cap = self.rec.shape[0]
        io.pool_log = self.log.ctypes.data_as(P32)
        io.pool_log_cap = self.log.shape[0]
        self.io = io

    def tokens(self) -> list[int]:
        return [int(t) for t in self.out[: self.io.n_out]]

    def records(self) -> list[StepRecord]:
        return [StepRecord(*map(int, r)) for r in self.rec[: self.io.n_steps]]

    def stats(self) -> dict:
        return dict(prefill_ms=float(self.io.prefill_ms), decode_ms=float(self.io.decode_ms),
                    launches=int(self.io.launches), steps=int(self.io.n_steps),
                    tokens=int(self.io.n_out))


def _gen_config(config: GenerationConfig) -> _lib.la_gen_config:
    eos = -1 if config.eos_token is None else int(config.eos_token)
    return _lib.la_gen_config(config.window, config.ngram, config.max_candidates,
                              config.max_tokens, eos, 1 if config.seed_pool_from_prompt else 0)


def _prepare_lookahead(model, prompt, config, sampler, pool):
    p = _prompt(prompt)
    if pool is not None and pool.ngram != config.ngram:
        raise ValueError("pool n-gram size does not match the generation config")
    init = None
    if pool is not None and len(pool):
        init = np.ascontiguousarray(np.asarray(pool.entries_oldest_first(), dtype=np.int32))
    dev_sampler = None
    if sampler.mode == "greedy":
        rng = window_rng_stream(sampler.seed, model.vocab_size, config.window, config.ngram,
                                config.max_tokens)
    else:
        # start_session (decoding.py:83-84): window_init's draws, then the
        # generator continues on the device
        gen = np.random.default_rng(sampler.seed)
        ncell = max((config.ngram - 1) * config.window - 1, 0)
        cells = gen.integers(0, model.vocab_size, size=ncell).astype(np.int32)
        rng = np.ascontiguousarray(cells if ncell else np.zeros(1, dtype=np.int32))
        dev_sampler = _device_sampler(sampler, gen)
    n_seed = max(0, len(p) - config.ngram + 1) if config.seed_pool_from_prompt else 0
    log_cap = n_seed + config.max_tokens * config.window + 1
    io = _IO(p, config.max_tokens, rng, init, config.ngram, log_cap)
    io.io.pool_capacity = 0 if pool is None or pool.capacity is None else int(pool.capacity)
    io.sampler = dev_sampler
    return io


def _finish_lookahead(io: _IO, config: GenerationConfig, pool: NGramPool | None):
    if pool is not None:
        n = min(io.io.pool_log_n, io.log.shape[0])
        pool.insert_all(io.log[:n].tolist())
    tokens = io.tokens()
    metrics = RunMetrics.from_records(len(tokens), io.records(), config.ngram)
    return tokens, metrics


def decode_lookahead(model, prompt: Sequence[int], config: GenerationConfig,
                     sampler: SamplerSpec, pool: NGramPool | None = None):
    """Lookahead decode on the GPU; returns (tokens, RunMetrics).

    Greedy: token-for-token equal to ``decode_autoregressive`` on the same
    model (exactness guarantee, reference decoding.py:235-241).  Temperature:
    distribution-preserving verification (verification.py:74-118) on the
    same random stream as the reference session seeded with ``sampler.seed``."""
    m = _require_b200(model)
    io = _prepare_lookahead(m, prompt, config, sampler, pool)
    if io.sampler is None:
        rc = m.lib.la_decode_lookahead(m.engine(), C.byref(_gen_config(config)),
                                       C.byref(io.io), m.stream())
    else:
        rc = m.lib.la_decode_lookahead_sampled(m.engine(), C.byref(_gen_config(config)),
                                               C.byref(io.sampler), C.byref(io.io), m.stream())
    _lib.check(rc)
    m.last_stats = io.stats()
    return _finish_lookahead(io, config, pool)


def decode_autoregressive(model, prompt: Sequence[int], sampler: SamplerSpec, max_tokens: int,
                          eos_token: int | None = None) -> list[int]:
    """One token per forward (reference decoding.py:96-116): argmax, or one
    ``sample_token`` draw from ``default_rng(sampler.seed)`` per token."""
    m = _require_b200(model)
    p = _prompt(prompt)
    if max_tokens < 1:
        return []      # the reference loop `while len(out) < max_tokens` never runs
    io = _IO(p, max_tokens)
    eos = -1 if eos_token is None else int(eos_token)
    if sampler.mode == "greedy":
        rc = m.lib.la_decode_autoregressive(m.engine(), max_tokens, eos, C.byref(io.io),
                                            m.stream())
    else:
        smp = _device_sampler(sampler, np.random.default_rng(sampler.seed))
        rc = m.lib.la_decode_autoregressive_sampled(m.engine(), max_tokens, eos, C.byref(smp),
                                                    C.byref(io.io), m.stream())
    _lib.check(rc)
    m.last_stats = io.stats()
    return io.tokens()


def decode_jacobi(model, prompt: Sequence[int], m: int,
                  rng: np.random.Generator) -> tuple[list[int], JacobiTrajectory, int]:
    """Solve an m-token greedy continuation by parallel fixed-point iteration
    (reference decoding.py:119-149).  The initial guess is drawn from ``rng``
    exactly like the reference (``rng.integers(0, V, size=m)``); every
    iteration is one device forward of the triangular chain layout
    (layout.py:185-194) with the per-row argmax taken on the GPU, so the
    fixed point equals greedy autoregressive decoding in <= m iterations."""
    mdl = _require_b200(model)
    if not len(prompt):
        raise ValueError("prompt must be nonempty")
    if m < 1:
        raise ValueError("generation length m must be >= 1")
    p = _prompt(prompt)
    init = np.ascontiguousarray(rng.integers(0, mdl.vocab_size, size=m).astype(np.int32))
    out = np.zeros(m, dtype=np.int32)
    iterates = np.zeros((m, m), dtype=np.int32)
    n_it = C.c_int32(0)
    P32 = C.POINTER(C.c_int32)
    _lib.check(mdl.lib.la_decode_jacobi(mdl.engine(), p.ctypes.data_as(P32), len(p), int(m),
                                        init.ctypes.data_as(P32), out.ctypes.data_as(P32),
                                        iterates.ctypes.data_as(P32), C.byref(n_it), mdl.stream()))
    traj = [[int(t) for t in init]] + [[int(t) for t in iterates[i]] for i in range(n_it.value)]
    return [int(t) for t in out], JacobiTrajectory(traj), int(n_it.value)


# ------------------------------------------------------------ step sessions
_SESSION_SEQ = 0


class DecodeState:
    """Per-session state (reference decoding.py:53-64).  The window, pool and
    KV cache live on the device between steps, in an engine of the session's
    own (sessions on one model are independent, as in the reference);
    ``prefix``, ``records``, the caller-visible ``pool`` and ``rng`` (the
    generator the device consumes) are kept in step on the host, ``window``
    is read back on access."""

    def __init__(self, model, prefix, pool, config, sampler, rng, key="main"):
        self.model = model
        self._key = key
        self.prefix = prefix
        self.pool = pool
        self.config = config
        self.sampler = sampler
        self.rng = rng              # host generator after window_init (the device continues it)
        self.records: list[StepRecord] = []
        self._log_n = 0

    def _engine(self):
        return self.model.engine(self._key)

    @property
    def window(self) -> Window2D:
        m, W, N = self.model, self.config.window, self.config.ngram
        cells = np.zeros(max((N - 1) * W - 1, 1), dtype=np.int32)
        _lib.check(m.lib.la_session_read(self._engine(), 0, 0, (N - 1) * W - 1,
                                         cells.ctypes.data_as(C.POINTER(C.c_int32))))
        levels = [cells[: W - 1].tolist()] + [cells[W - 1 + l * W: W - 1 + (l + 1) * W].tolist()
                                              for l in range(N - 2)]
        return Window2D(W, N, m.vocab_size, levels)

    def _sync_pool(self, log_n: int) -> None:
        n = log_n - self._log_n
        if n > 0:
            buf = np.zeros((n, self.config.ngram), dtype=np.int32)
            _lib.check(self.model.lib.la_session_read(self._engine(), 1, self._log_n, n,
                                                      buf.ctypes.data_as(C.POINTER(C.c_int32))))
            self.pool.insert_all(buf.tolist())
        self._log_n = log_n

    def _sync_rng(self) -> None:
        """The reference session's generator advances with every window refill
        and verify_sample draw (layout.py:243-250, verification.py:74-118):
        mirror the device generator into ``rng``."""
        w = np.zeros(10, dtype=np.int32)
        _lib.check(self.model.lib.la_session_read(self._engine(), 2, 0, 10,
                                                  w.ctypes.data_as(C.POINTER(C.c_int32))))
        u = w.view(np.uint32).astype(object)
        q = [int(u[2 * i]) | (int(u[2 * i + 1]) << 32) for i in range(4)]
        self.rng.bit_generator.state = {
            "bit_generator": "PCG64",
            "state": {"state": (q[0] << 64) | q[1], "inc": (q[2] << 64) | q[3]},
            "has_uint32": int(w[8]), "uinteger": int(u[9])}


def start_session(model, prompt: Sequence[int], config: GenerationConfig, sampler: SamplerSpec,
                  pool: NGramPool | None = None) -> DecodeState:
    """Initialise window, pool and generator for step-by-step decoding
    (reference decoding.py:67-93); the prompt is prefilled on the device."""
    m = _require_b200(model)
    p = _prompt(prompt)
    if pool is None:
        pool = NGramPool(config.ngram)
    elif pool.ngram != config.ngram:
        raise ValueError("pool n-gram size does not match the generation config")
    init = None
    if len(pool):
        init = np.ascontiguousarray(np.asarray(pool.entries_oldest_first(), dtype=np.int32))
    rng = np.random.default_rng(sampler.seed)
    ncell = (config.ngram - 1) * config.window - 1
    cells = rng.integers(0, m.vocab_size, size=ncell).astype(np.int32)   # window_init
    stream = np.ascontiguousarray(cells if ncell else np.zeros(1, dtype=np.int32))
    n_seed = max(0, len(p) - config.ngram + 1) if config.seed_pool_from_prompt else 0
    io = _IO(p, 1, stream, init, config.ngram, 1)
    io.io.pool_capacity = 0 if pool.capacity is None else int(pool.capacity)
    smp = _lib.make_sampler(sampler.temperature, sampler.top_k, sampler.top_p, rng)
    # every session gets an engine of its own (KV cache, window, pool), released
    # with the state object
    global _SESSION_SEQ
    _SESSION_SEQ += 1
    key = ("session", _SESSION_SEQ)
    try:
        _lib.check(m.lib.la_session_start(m.engine(key), C.byref(_gen_config(config)),
                                          1 if sampler.mode == "greedy" else 0, C.byref(smp),
                                          C.byref(io.io), m.stream()))
    except Exception:
        m.release_engine(key)
        raise
    state = DecodeState(m, [int(t) for t in p], pool, config, sampler, rng, key)
    weakref.finalize(state, m.release_engine, key)
    # a caller pool's replay is not a new insert; prompt seeding is (pool.py:83-90)
    state._log_n = 0
    state._sync_pool(n_seed)
    return state


def lookahead_step(state: DecodeState) -> StepOutcome:
    """One generate-and-verify step on the device (reference decoding.py:207-211)."""
    m = state.model
    out = _lib.la_step_outcome()
    _lib.check(m.lib.la_session_step(state._engine(), C.byref(out), m.stream()))
    accepted = [int(out.accepted[i]) for i in range(out.n_accepted)]
    state._sync_pool(int(out.pool_log_n))
    state._sync_rng()
    state.prefix.extend(accepted)
    state.records.append(StepRecord(out.n_accepted, int(out.candidate_count),
                                    int(out.query_count), int(out.pool_size)))
    return StepOutcome(accepted, [int(out.new_top[i]) for i in range(out.n_new_top)],
                       int(out.candidate_count), int(out.query_count))


def collect_output(out: list[int], accepted: Sequence[int], max_tokens: int,
                   eos_token: int | None) -> bool:
    """Fold one step's tokens into the output (reference decoding.py:214-232)."""
    for token in accepted:
        out.append(int(token))
        if eos_token is not None and token == eos_token:
            return True
        if len(out) >= max_tokens:
            return True
    return False
