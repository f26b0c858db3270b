"""B200 models behind the reference's model plugin boundary.

``B200Model`` satisfies the reference ``ModelInterface`` contract
(``models.py:67-93``: ``vocab_size``, ``forward(prefix, layout)`` returning
one float64 distribution per query, ``next_distribution(sequence)``), so the
reference's own orchestration can drive it, while ``decode_lookahead`` in this
package runs the whole step on the device through the C ABI.

Weights live in torch device tensors owned by the model; the C engine
borrows their pointers (``la_create``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace
from collections.abc import Sequence

import numpy as np

from . import _lib
from .layout import layout_chains


def _torch():
    import torch
    return torch


class B200Model:
    """Base class: a model whose forward runs in the CUDA C-ABI engine."""

    arch: int = -1

    def __init__(self, desc: dict, named: dict, device: int = 0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("B200 models need a CUDA device (there is no CPU fallback)")
        self.lib = _lib.load()
        self.device = int(device)
        self.vocab_size = int(desc["vocab"])
        self.desc = _lib.la_model_desc(
            self.arch, desc["vocab"], desc["dim"], desc["layers"], desc["heads"],
            desc["kv_heads"], desc["head_dim"], desc["ffn"], float(desc.get("rope_theta", 1e4)),
            float(desc.get("norm_eps", 1e-5)), int(desc["max_context"]))
        n = self.lib.la_weight_count(C.byref(self.desc))
        names = [self.lib.la_weight_name(C.byref(self.desc), i).decode() for i in range(n)]
        missing = [k for k in names if k not in named]
        if missing:
            raise ValueError(f"missing weights: {missing[:5]}")
        self._tensors = [named[k] for k in names]
        self._names = names
        self._engines: dict = {}
        self.last_stats: dict = {}

    # -------------------------------------------------------------- engines
    def engine(self, key="main"):
        h = self._engines.get(key)
        if h is None:
            ptrs = (C.c_void_p * len(self._tensors))(*[t.data_ptr() for t in self._tensors])
            out = C.c_void_p()
            _lib.check(self.lib.la_create(C.byref(self.desc), ptrs, len(self._tensors),
                                          self.device, C.byref(out)))
            h = out.value
            self._engines[key] = h
        return h

    def release_engine(self, key) -> None:
        """Destroy one engine (a finished step session's); no-op if absent."""
        h = self._engines.pop(key, None)
        if h is not None:
            self.lib.la_destroy(h)

    def close(self) -> None:
        for h in list(self._engines.values()):
            self.lib.la_destroy(h)
        self._engines.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stream(self):
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def max_context(self) -> int:
        return int(self.desc.max_context)

    # ------------------------------------------------ ModelInterface surface
    def _check_token(self, t: int) -> None:
        if not 0 <= int(t) < self.vocab_size:
            raise ValueError(f"token {int(t)} outside vocabulary of size {self.vocab_size}")

    def logits(self, prefix: Sequence[int], layout) -> np.ndarray:
        """fp32 logits [n_queries, V] of ``layout`` after ``prefix``."""
        for t in prefix:
            self._check_token(t)
        for q in layout.queries:
            self._check_token(q.token)
        ids, rel, chain = layout_chains(layout)
        M = len(ids)
        out = np.empty((M, self.vocab_size), dtype=np.float32)
        pre = _lib.i32_array(prefix)
        chain_c = np.ascontiguousarray(chain, dtype=np.int32)
        P32 = C.POINTER(C.c_int32)
        _lib.check(self.lib.la_forward_layout(
            self.engine(), pre, len(prefix), M, ids.ctypes.data_as(P32), rel.ctypes.data_as(P32),
            chain_c.ctypes.data_as(P32), chain_c.shape[1],
            out.ctypes.data_as(C.POINTER(C.c_float)), self.stream()))
        return out

    def forward(self, prefix: Sequence[int], layout) -> list[np.ndarray]:
        """One next-token distribution per query, in query order (float64)."""
        lg = self.logits(prefix, layout).astype(np.float64)
        lg -= lg.max(axis=1, keepdims=True)
        p = np.exp(lg)
        p /= p.sum(axis=1, keepdims=True)
        return [p[i] for i in range(p.shape[0])]

    def next_distribution(self, sequence: Sequence[int]) -> np.ndarray:
        from .layout import chain_layout
        seq = [int(t) for t in sequence]
        return self.forward(seq[:-1], chain_layout(seq[-1], []))[0]


# ------------------------------------------------------------ tiny GPT model
class TinyTransformer(B200Model):
    """The reference TinyTransformer (models.py:189-271) on the fp32 SIMT path.

    Weights are drawn from ``numpy.random.default_rng(seed)`` in the
    reference's order (models.py:219-242), so a reference model and this one
    built from the same arguments hold identical weights."""

    arch = _lib.ARCH_GPT_F32

    def __init__(self, seed: int, vocab_size: int, d_model: int = 16, n_layers: int = 2,
                 n_heads: int = 2, *, max_context: int = 4096, device: int = 0):
        if min(vocab_size, d_model, n_layers, n_heads) < 1:
            raise ValueError("all dimensions must be positive")
        if d_model % n_heads != 0:
            raise ValueError("d_model must be divisible by n_heads")
        torch = _torch()
        self.seed = seed
        self.d_model, self.n_layers, self.n_heads = d_model, n_layers, n_heads
        rng = np.random.default_rng(seed)
        sd = 1.0 / np.sqrt(d_model)
        ff = 4 * d_model
        host = {"embed": rng.normal(0.0, sd, size=(vocab_size, d_model))}
        for i in range(n_layers):
            for nm in ("wq", "wk", "wv", "wo"):
                host[f"{i}.{nm}"] = rng.normal(0.0, sd, size=(d_model, d_model)).T
            host[f"{i}.ln1_g"], host[f"{i}.ln1_b"] = np.ones(d_model), np.zeros(d_model)
            host[f"{i}.w1"] = rng.normal(0.0, sd, size=(d_model, ff)).T
            host[f"{i}.b1"] = np.zeros(ff)
            host[f"{i}.w2"] = rng.normal(0.0, 1.0 / np.sqrt(ff), size=(ff, d_model)).T
            host[f"{i}.b2"] = np.zeros(d_model)
            host[f"{i}.ln2_g"], host[f"{i}.ln2_b"] = np.ones(d_model), np.zeros(d_model)
        host["lnf_g"], host["lnf_b"] = np.ones(d_model), np.zeros(d_model)
        host["unembed"] = rng.normal(0.0, sd, size=(d_model, vocab_size)).T
        dev = torch.device("cuda", device)
        named = {k: torch.tensor(np.ascontiguousarray(v, dtype=np.float32), device=dev)
                 for k, v in host.items()}
        desc = dict(vocab=vocab_size, dim=d_model, layers=n_layers, heads=n_heads,
                    kv_heads=n_heads, head_dim=d_model // n_heads, ffn=ff,
                    max_context=max_context)
        super().__init__(desc, named, device)


# --------------------------------------------------------------- Llama family
@dataclass(frozen=True)
class LlamaConfig:
    dim: int
    layers: int
    heads: int
    kv_heads: int
    ffn: int
    vocab: int = 32000
    head_dim: int = 128
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    def as_desc(self, max_context: int) -> dict:
        return dict(vocab=self.vocab, dim=self.dim, layers=self.layers, heads=self.heads,
                    kv_heads=self.kv_heads, head_dim=self.head_dim, ffn=self.ffn,
                    rope_theta=self.rope_theta, norm_eps=self.norm_eps, max_context=max_context)

    def with_(self, **kw) -> "LlamaConfig":
        return replace(self, **kw)


LLAMA2_7B = LlamaConfig(dim=4096, layers=32, heads=32, kv_heads=32, ffn=11008)
CODELLAMA_7B = LlamaConfig(dim=4096, layers=32, heads=32, kv_heads=32, ffn=11008,
                           vocab=32016, rope_theta=1e6)
LLAMA2_13B = LlamaConfig(dim=5120, layers=40, heads=40, kv_heads=40, ffn=13824)
LLAMA2_70B = LlamaConfig(dim=8192, layers=80, heads=64, kv_heads=8, ffn=28672)
PRESETS = {"llama2-7b": LLAMA2_7B, "codellama-7b": CODELLAMA_7B, "llama2-13b": LLAMA2_13B,
           "llama2-70b": LLAMA2_70B}


def llama_weight_shapes(cfg: LlamaConfig) -> dict:
    d, hd = cfg.dim, cfg.head_dim
    shapes = {"embed": (cfg.vocab, d), "lm_head": (cfg.vocab, d), "final_norm": (d,)}
    for i in range(cfg.layers):
        shapes.update({f"{i}.wq": (cfg.heads * hd, d), f"{i}.wk": (cfg.kv_heads * hd, d),
                       f"{i}.wv": (cfg.kv_heads * hd, d), f"{i}.wo": (d, cfg.heads * hd),
                       f"{i}.w_gate": (cfg.ffn, d), f"{i}.w_up": (cfg.ffn, d),
                       f"{i}.w_down": (d, cfg.ffn), f"{i}.attn_norm": (d,),
                       f"{i}.mlp_norm": (d,)})
    return shapes


class LlamaModel(B200Model):
    """Llama-2-shaped decoder (RMSNorm, rotate-half RoPE, SwiGLU, GQA).

    ``dtype="bf16"``: the tcgen05 multi-kernel path (configs 2-5).  Projection
    matrices live in the packed LA-tile layout (``la_pack_weight``): q/k/v
    stacked, gate/up interleaved per 64 rows, each 128x64 block one
    contiguous 16 KB swizzled image so the GEMM streams HBM sequentially.
    ``dtype="f32"``: the fp32 SIMT single-CTA path (small parity models).
    ``weights``: optional name -> array/tensor dict in HF layout ([out][in]:
    ``embed, lm_head, final_norm, i.wq, i.wk, i.wv, i.wo, i.w_gate, i.w_up,
    i.w_down, i.attn_norm, i.mlp_norm``), converted on the device; otherwise
    random-init N(0, 0.02^2) matrices and unit norm gains from a seeded CUDA
    generator (BASELINE: synthetic weights of the named shape)."""

    def __init__(self, cfg: LlamaConfig, *, dtype: str = "bf16", weights: dict | None = None,
                 seed: int = 0, max_context: int = 2048, device: int = 0, init_std: float = 0.02):
        torch = _torch()
        if dtype not in ("bf16", "f32"):
            raise ValueError("dtype must be 'bf16' or 'f32'")
        self.cfg = cfg
        self.dtype = dtype
        self.arch = _lib.ARCH_LLAMA_BF16 if dtype == "bf16" else _lib.ARCH_LLAMA_F32
        dev = torch.device("cuda", device)
        self._gen = None
        self._seed = seed
        self._std = init_std
        self._dev = dev
        if dtype == "f32":
            named = {}
            for name, shape in llama_weight_shapes(cfg).items():
                named[name] = self._tensor(weights, name, shape, torch.float32)
        else:
            named = self._packed_bf16(cfg, weights)
        super().__init__(cfg.as_desc(max_context), named, device)

    # ---------------------------------------------------------- weights
    def _rand(self, shape, dtype):
        torch = _torch()
        if self._gen is None:
            self._gen = torch.Generator(device=self._dev)
            self._gen.manual_seed(self._seed)
        return torch.empty(shape, dtype=dtype, device=self._dev).normal_(0.0, self._std,
                                                                        generator=self._gen)

    def _tensor(self, weights, name, shape, dtype):
        torch = _torch()
        if weights is not None:
            src = weights[name]
            t = src if isinstance(src, torch.Tensor) else torch.from_numpy(np.asarray(src))
            return t.to(device=self._dev, dtype=dtype).contiguous()
        if len(shape) == 1:
            return torch.ones(shape, dtype=torch.float32, device=self._dev)
        return self._rand(shape, dtype)

    def _packed_bf16(self, cfg: LlamaConfig, weights: dict | None) -> dict:
        torch = _torch()
        lib = _lib.load()
        bf = torch.bfloat16
        d, hd, H, KVH, F, V = cfg.dim, cfg.head_dim, cfg.heads, cfg.kv_heads, cfg.ffn, cfg.vocab
        stream = C.c_void_p(torch.cuda.current_stream(self._dev).cuda_stream)

        def packed(rows, K):
            n = lib.la_packed_bytes(rows, K)
            if n < 0:
                raise ValueError(f"cannot pack a [{rows}][{K}] matrix (K % 64 != 0)")
            return torch.zeros(n // 2, dtype=bf, device=self._dev)

        def pack_into(dst, name, rows, K, mode=0, off=0):
            src = self._tensor(weights, name, (rows, K), bf)
            _lib.check(lib.la_pack_weight(C.c_void_p(src.data_ptr()), rows, K,
                                          C.c_void_p(dst.data_ptr()), mode, off, stream))
            del src

        named = {"embed": self._tensor(weights, "embed", (V, d), bf),
                 "final_norm": self._tensor(weights, "final_norm", (d,), torch.float32)}
        if weights is None:
            # synthetic: draw the packed tiles directly (same distribution)
            def fill(rows, K):
                t = packed(rows, K)
                t.normal_(0.0, self._std, generator=self._gen_or_new())
                return t
            named["lm_head_tiles"] = fill(V, d)
            for i in range(cfg.layers):
                named[f"{i}.wqkv_tiles"] = fill((H + 2 * KVH) * hd, d)
                named[f"{i}.wo_tiles"] = fill(d, H * hd)
                named[f"{i}.wgu_tiles"] = fill(2 * F, d)
                named[f"{i}.wd_tiles"] = fill(d, F)
                named[f"{i}.attn_norm"] = torch.ones(d, dtype=torch.float32, device=self._dev)
                named[f"{i}.mlp_norm"] = torch.ones(d, dtype=torch.float32, device=self._dev)
            return named
        lm = packed(V, d)
        pack_into(lm, "lm_head", V, d)
        named["lm_head_tiles"] = lm
        for i in range(cfg.layers):
            qkv = packed((H + 2 * KVH) * hd, d)
            pack_into(qkv, f"{i}.wq", H * hd, d, 0, 0)
            pack_into(qkv, f"{i}.wk", KVH * hd, d, 0, H * hd)
            pack_into(qkv, f"{i}.wv", KVH * hd, d, 0, (H + KVH) * hd)
            wo = packed(d, H * hd)
            pack_into(wo, f"{i}.wo", d, H * hd)
            gu = packed(2 * F, d)
            pack_into(gu, f"{i}.w_gate", F, d, 1)
            pack_into(gu, f"{i}.w_up", F, d, 2)
            wd = packed(d, F)
            pack_into(wd, f"{i}.w_down", d, F)
            named.update({f"{i}.wqkv_tiles": qkv, f"{i}.wo_tiles": wo, f"{i}.wgu_tiles": gu,
                          f"{i}.wd_tiles": wd,
                          f"{i}.attn_norm": self._tensor(weights, f"{i}.attn_norm", (d,), torch.float32),
                          f"{i}.mlp_norm": self._tensor(weights, f"{i}.mlp_norm", (d,), torch.float32)})
        torch.cuda.synchronize(self._dev)
        return named

    def _gen_or_new(self):
        torch = _torch()
        if self._gen is None:
            self._gen = torch.Generator(device=self._dev)
            self._gen.manual_seed(self._seed)
        return self._gen
