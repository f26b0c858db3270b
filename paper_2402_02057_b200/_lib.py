"""ctypes binding of the C ABI (``include/lookahead_b200.h``).

The library is built in-tree (``python -m paper_2402_02057_b200._build``).
There is no fallback: if the library is missing or a call fails, an
exception is raised.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .types import DegenerateDistributionError, LayoutError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "liblookahead_b200.so"

ABI_VERSION = 2   # la_abi_version() of the library this binding matches

LA_OK = 0
LA_ERR_INVALID_CONFIG = -1
LA_ERR_LAYOUT = -2
LA_ERR_CUDA = -3
LA_ERR_NCCL = -4
LA_ERR_CAPACITY = -5
LA_ERR_UNSUPPORTED = -6
LA_ERR_DEGENERATE = -7

ARCH_GPT_F32 = 0
ARCH_LLAMA_F32 = 1
ARCH_LLAMA_BF16 = 2

# every symbol the header declares (checked by tests/test_cabi.py)
EXPORTS = (
    "la_last_error", "la_abi_version", "la_weight_count", "la_weight_name", "la_create",
    "la_destroy", "la_decode_lookahead", "la_decode_autoregressive", "la_forward_layout",
    "la_lp_unique_id", "la_lp_init", "la_decode_lookahead_group", "la_debug_read",
    "la_gemm_timing_enable", "la_gemm_timing_reset", "la_gemm_timing_read", "la_forward_timing_read", "la_packed_bytes",
    "la_decode_jacobi", "la_decode_lookahead_sampled", "la_decode_autoregressive_sampled",
    "la_adjust_distributions", "la_verify_sample_dists", "la_pcg64_draws",
    "la_session_start", "la_session_step", "la_session_read", "la_pool_test",
    "la_pack_weight",
)


class CudaEngineError(RuntimeError):
    """A CUDA / NCCL failure inside the engine."""


class la_model_desc(C.Structure):
    _fields_ = [("arch", C.c_int32), ("vocab", C.c_int32), ("dim", C.c_int32),
                ("layers", C.c_int32), ("heads", C.c_int32), ("kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("ffn", C.c_int32), ("rope_theta", C.c_float),
                ("norm_eps", C.c_float), ("max_context", C.c_int32)]


class la_gen_config(C.Structure):
    _fields_ = [("window", C.c_int32), ("ngram", C.c_int32), ("max_candidates", C.c_int32),
                ("max_tokens", C.c_int32), ("eos_token", C.c_int32),
                ("seed_pool_from_prompt", C.c_int32)]


_P32 = C.POINTER(C.c_int32)


class la_sampler(C.Structure):
    _fields_ = [("temperature", C.c_double), ("top_k", C.c_int32), ("top_p", C.c_double),
                ("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64),
                ("inc_lo", C.c_uint64), ("has_uint32", C.c_int32), ("uinteger", C.c_uint32)]


class la_step_outcome(C.Structure):
    _fields_ = [("accepted", C.c_int32 * 9), ("n_accepted", C.c_int32),
                ("new_top", C.c_int32 * 64), ("n_new_top", C.c_int32),
                ("candidate_count", C.c_int32), ("query_count", C.c_int32),
                ("pool_size", C.c_int32), ("pool_log_n", C.c_int32)]


def make_sampler(temperature: float, top_k, top_p, rng) -> la_sampler:
    """la_sampler from a SamplerSpec's knobs and a numpy Generator (PCG64) in
    its current state."""
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("the device generator restates numpy's PCG64 (default_rng)")
    m64 = (1 << 64) - 1
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    return la_sampler(float(temperature), 0 if top_k is None else int(top_k),
                      1.0 if top_p is None else float(top_p), s >> 64, s & m64, inc >> 64,
                      inc & m64, int(st["has_uint32"]), int(st["uinteger"]))


class la_decode_io(C.Structure):
    _fields_ = [("prompt", _P32), ("n_prompt", C.c_int32),
                ("rng_stream", _P32), ("rng_len", C.c_int32),
                ("pool_init", _P32), ("pool_init_n", C.c_int32),
                ("out_tokens", _P32), ("out_cap", C.c_int32), ("n_out", C.c_int32),
                ("step_records", _P32), ("rec_cap", C.c_int32), ("n_steps", C.c_int32),
                ("pool_log", _P32), ("pool_log_cap", C.c_int32), ("pool_log_n", C.c_int32),
                ("prefill_ms", C.c_float), ("decode_ms", C.c_float), ("launches", C.c_int32),
                ("pool_capacity", C.c_int32)]


_lib = None


def load(path: str | os.PathLike | None = None):
    """Load the library (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    # LA_LIB_PATH: another build of the same ABI (profiling A/B runs)
    p = Path(path or os.environ.get("LA_LIB_PATH") or LIB_PATH)
    if not p.exists():
        raise RuntimeError(
            f"CUDA library {p} is missing: build it with `python -m paper_2402_02057_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    lib.la_last_error.restype = C.c_char_p
    lib.la_abi_version.restype = C.c_int32
    if lib.la_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{p}: ABI version {lib.la_abi_version()}, this binding needs {ABI_VERSION} "
                           "(rebuild with `python -m paper_2402_02057_b200._build`)")
    lib.la_weight_count.argtypes = [C.POINTER(la_model_desc)]
    lib.la_weight_count.restype = C.c_int32
    lib.la_weight_name.argtypes = [C.POINTER(la_model_desc), C.c_int32]
    lib.la_weight_name.restype = C.c_char_p
    lib.la_create.argtypes = [C.POINTER(la_model_desc), C.POINTER(C.c_void_p), C.c_int32,
                              C.c_int32, C.POINTER(C.c_void_p)]
    lib.la_destroy.argtypes = [C.c_void_p]
    lib.la_decode_lookahead.argtypes = [C.c_void_p, C.POINTER(la_gen_config),
                                        C.POINTER(la_decode_io), C.c_void_p]
    lib.la_decode_autoregressive.argtypes = [C.c_void_p, C.c_int32, C.c_int32,
                                             C.POINTER(la_decode_io), C.c_void_p]
    lib.la_forward_layout.argtypes = [C.c_void_p, _P32, C.c_int32, C.c_int32, _P32, _P32, _P32,
                                      C.c_int32, C.POINTER(C.c_float), C.c_void_p]
    lib.la_lp_unique_id.argtypes = [C.c_void_p]
    lib.la_lp_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]
    lib.la_decode_lookahead_group.argtypes = [C.POINTER(C.c_void_p), C.c_int32,
                                              C.POINTER(la_gen_config), C.POINTER(la_decode_io),
                                              C.c_void_p]
    lib.la_debug_read.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64]
    lib.la_packed_bytes.argtypes = [C.c_int32, C.c_int32]
    lib.la_packed_bytes.restype = C.c_int64
    lib.la_pack_weight.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                   C.c_int32, C.c_void_p]
    SP = C.POINTER(la_sampler)
    lib.la_decode_lookahead_sampled.argtypes = [C.c_void_p, C.POINTER(la_gen_config), SP,
                                                C.POINTER(la_decode_io), C.c_void_p]
    lib.la_decode_autoregressive_sampled.argtypes = [C.c_void_p, C.c_int32, C.c_int32, SP,
                                                     C.POINTER(la_decode_io), C.c_void_p]
    lib.la_adjust_distributions.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, SP,
                                            C.c_void_p, C.c_void_p]
    lib.la_verify_sample_dists.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                           C.c_int32, _P32, SP, _P32, _P32, C.c_void_p]
    lib.la_pcg64_draws.argtypes = [SP, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
    lib.la_session_start.argtypes = [C.c_void_p, C.POINTER(la_gen_config), C.c_int32, SP,
                                     C.POINTER(la_decode_io), C.c_void_p]
    lib.la_session_step.argtypes = [C.c_void_p, C.POINTER(la_step_outcome), C.c_void_p]
    lib.la_session_read.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, _P32]
    lib.la_pool_test.argtypes = [C.c_int32, C.c_int32, C.c_int32, _P32, C.c_int32, C.c_int32, _P32,
                                 C.c_int32, C.c_int32, _P32, _P32, _P32]
    lib.la_gemm_timing_enable.argtypes = [C.c_void_p, C.c_int32]
    lib.la_gemm_timing_reset.argtypes = [C.c_void_p]
    lib.la_gemm_timing_read.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    for name in EXPORTS:
        getattr(lib, name).restype = getattr(lib, name).restype or C.c_int32
    lib.la_last_error.restype = C.c_char_p
    lib.la_weight_name.restype = C.c_char_p
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C status code to the reference's exception classes."""
    if rc == LA_OK:
        return
    msg = (load().la_last_error() or b"").decode(errors="replace")
    if rc == LA_ERR_LAYOUT:
        raise LayoutError(msg)
    if rc in (LA_ERR_INVALID_CONFIG,):
        raise ValueError(msg)
    if rc == LA_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == LA_ERR_DEGENERATE:
        raise DegenerateDistributionError(msg)
    if rc == LA_ERR_CAPACITY:
        raise ValueError(f"capacity: {msg}")
    raise CudaEngineError(f"engine error {rc}: {msg}")


def i32_array(values):
    n = len(values)
    arr = (C.c_int32 * max(n, 1))(*[int(v) for v in values])
    return arr
