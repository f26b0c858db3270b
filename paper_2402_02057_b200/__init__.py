"""B200-native greedy lookahead decoding (arXiv 2402.02057).

Drop-in for the reference package's decode path: same names, argument
meaning and error behaviour; the step runs as sm_100a CUDA kernels behind a
C ABI (``include/lookahead_b200.h``).
"""

__version__ = "0.1.0"

from .analytics import RunMetrics, compression_ratio, flops_proxy
from .decoding import (DecodeState, collect_output, decode_autoregressive, decode_jacobi,
                       decode_lookahead, lookahead_step, start_session, window_rng_stream)
from .layout import CandidateBranch, QueryToken, StepLayout, chain_layout
from .models import (CODELLAMA_7B, LLAMA2_13B, LLAMA2_70B, LLAMA2_7B, PRESETS, B200Model,
                     LlamaConfig, LlamaModel, TinyTransformer)
from .parallel import CommStats, column_ranges, decode_lookahead_devices, lp_init, step_comm
from .pool import NGramPool
from .types import (DegenerateDistributionError, GenerationConfig, JacobiTrajectory, LayoutError,
                    SamplerSpec, StepOutcome, StepRecord, Window2D)


def transformer_init(seed, vocab_size, d_model=16, n_layers=2, n_heads=2, **kw):
    """Reference-compatible constructor (models.py:274-284) on the B200 path."""
    return TinyTransformer(seed, vocab_size, d_model, n_layers, n_heads, **kw)


def greedy_token(probs) -> int:
    """Lowest index attaining the maximum (reference sampling.py:17-19)."""
    import numpy as np
    return int(np.argmax(probs))


__all__ = [
    "DecodeState", "StepOutcome", "Window2D", "collect_output", "lookahead_step", "start_session",
    "B200Model", "CODELLAMA_7B", "CandidateBranch", "CommStats", "DegenerateDistributionError",
    "GenerationConfig", "JacobiTrajectory", "LLAMA2_13B", "LLAMA2_70B", "LLAMA2_7B", "LayoutError", "LlamaConfig",
    "LlamaModel", "NGramPool", "PRESETS", "QueryToken", "RunMetrics", "SamplerSpec",
    "StepLayout", "StepRecord", "TinyTransformer", "chain_layout", "column_ranges",
    "compression_ratio", "decode_autoregressive", "decode_jacobi", "decode_lookahead",
    "decode_lookahead_devices", "flops_proxy", "greedy_token", "lp_init", "step_comm",
    "transformer_init", "window_rng_stream",
]
