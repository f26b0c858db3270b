"""CPU model oracles (TEST INFRASTRUCTURE ONLY).

* ``TinyTransformerOracle`` restates ``TinyTransformer`` (``models.py:189-271``)
  in float64, with weights drawn from ``default_rng(seed)`` in the reference's
  order (``models.py:219-242``) so that the oracle, the reference and the B200
  model share identical weights.
* ``LlamaOracle`` is the Llama-2-shaped decoder (RMSNorm, rotate-half RoPE,
  SwiGLU, GQA) that BASELINE configs 2-5 name.  The reference has no such
  model; this restatement follows the reference model *contract*
  (``models.py:33-93``: one distribution per query, conditioned on the query's
  chain; absolute position = len(prefix) + rel_pos, ``SPEC.md:179``).  With
  ``emulate_bf16=True`` it rounds to bf16 exactly where the device path stores
  bf16 (GEMM inputs, Q/K/V, attention output, SwiGLU output).

Both expose ``argmax_rows(prefix, rows)`` / ``logits_rows(prefix, rows)`` on
the flat ``Rows`` geometry of ``oracle.lookahead_oracle``.
"""

from __future__ import annotations

import numpy as np


def _chain_tokens(prefix, rows, i):
    return [int(t) for t in prefix] + [rows.ids[c] for c in rows.chains[i]] + [rows.ids[i]]


# ------------------------------------------------------ tiny transformer
class TinyTransformerOracle:
    def __init__(self, seed: int, vocab_size: int, d_model: int = 16, n_layers: int = 2,
                 n_heads: int = 2):
        self.vocab_size = vocab_size
        self.d = d_model
        self.L = n_layers
        self.H = n_heads
        self.dh = d_model // n_heads
        ff = 4 * d_model
        rng = np.random.default_rng(seed)
        s = 1.0 / np.sqrt(d_model)
        self.embedding = rng.normal(0.0, s, size=(vocab_size, d_model))
        self.layers = []
        for _ in range(n_layers):
            lw = {}
            for name in ("wq", "wk", "wv", "wo"):
                lw[name] = rng.normal(0.0, s, size=(d_model, d_model))
            lw["ln1_g"], lw["ln1_b"] = np.ones(d_model), np.zeros(d_model)
            lw["w1"] = rng.normal(0.0, s, size=(d_model, ff))
            lw["b1"] = np.zeros(ff)
            lw["w2"] = rng.normal(0.0, 1.0 / np.sqrt(ff), size=(ff, d_model))
            lw["b2"] = np.zeros(d_model)
            lw["ln2_g"], lw["ln2_b"] = np.ones(d_model), np.zeros(d_model)
            self.layers.append(lw)
        self.lnf_g, self.lnf_b = np.ones(d_model), np.zeros(d_model)
        self.unembed = rng.normal(0.0, s, size=(d_model, vocab_size))

    @staticmethod
    def _ln(x, g, b):                                   # models.py:183-186
        mu = x.mean(axis=-1, keepdims=True)
        var = x.var(axis=-1, keepdims=True)
        return (x - mu) / np.sqrt(var + 1e-8) * g + b

    def _pos(self, T):                                  # models.py:174-180
        pos = np.arange(T, dtype=np.float64)
        inv = np.power(10000.0, -np.arange(0, self.d, 2, dtype=np.float64) / self.d)
        ang = pos[:, None] * inv[None, :]
        enc = np.zeros((T, self.d))
        enc[:, 0::2] = np.sin(ang)
        enc[:, 1::2] = np.cos(ang[:, : self.d // 2])
        return enc

    def logits_seq(self, seq) -> np.ndarray:            # models.py:244-268
        tok = np.asarray(seq, dtype=np.int64)
        T = tok.shape[0]
        x = self.embedding[tok] + self._pos(T)
        mask = np.triu(np.full((T, T), -np.inf), k=1)
        for lw in self.layers:
            h = self._ln(x, lw["ln1_g"], lw["ln1_b"])
            q = (h @ lw["wq"]).reshape(T, self.H, self.dh).transpose(1, 0, 2)
            k = (h @ lw["wk"]).reshape(T, self.H, self.dh).transpose(1, 0, 2)
            v = (h @ lw["wv"]).reshape(T, self.H, self.dh).transpose(1, 0, 2)
            sc = q @ k.transpose(0, 2, 1) / np.sqrt(self.dh) + mask
            sc -= sc.max(axis=-1, keepdims=True)
            w = np.exp(sc)
            w /= w.sum(axis=-1, keepdims=True)
            x = x + (w @ v).transpose(1, 0, 2).reshape(T, self.d) @ lw["wo"]
            h = self._ln(x, lw["ln2_g"], lw["ln2_b"])
            inner = h @ lw["w1"] + lw["b1"]
            x = x + (inner * (inner > 0)) @ lw["w2"] + lw["b2"]
        return self._ln(x[-1], self.lnf_g, self.lnf_b) @ self.unembed

    def probs_seq(self, seq) -> np.ndarray:             # models.py:269-271
        lg = self.logits_seq(seq)
        lg = lg - lg.max()
        p = np.exp(lg)
        return p / p.sum()

    def logits_rows(self, prefix, rows) -> list[np.ndarray]:
        return [self.logits_seq(_chain_tokens(prefix, rows, i)) for i in range(len(rows))]

    def argmax_rows(self, prefix, rows) -> list[int]:
        # greedy_token is argmax of the probabilities (sampling.py:17-19)
        return [int(np.argmax(self.probs_seq(_chain_tokens(prefix, rows, i))))
                for i in range(len(rows))]

    def flat_weights_f32(self) -> dict:
        """Weights in the device layout (row-major, out-features x in-features)."""
        w = {"embed": self.embedding.astype(np.float32),
             "lnf_g": self.lnf_g.astype(np.float32), "lnf_b": self.lnf_b.astype(np.float32),
             "unembed_t": np.ascontiguousarray(self.unembed.T).astype(np.float32)}
        for i, lw in enumerate(self.layers):
            for n in ("wq", "wk", "wv", "wo", "w1", "w2"):
                w[f"{i}.{n}_t"] = np.ascontiguousarray(lw[n].T).astype(np.float32)
            for n in ("b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b"):
                w[f"{i}.{n}"] = lw[n].astype(np.float32)
        return w


# ------------------------------------------------------------ llama
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


class LlamaOracle:
    """fp32 Llama restatement; weights are a dict of float32 arrays in
    (out_features, in_features) layout, already bf16-representable."""

    def __init__(self, cfg: dict, weights: dict, emulate_bf16: bool = True):
        self.cfg = cfg
        self.w = weights
        self.vocab_size = cfg["vocab"]
        self.emul = emulate_bf16
        hd = cfg["head_dim"]
        self.inv_freq = (1.0 / (cfg["rope_theta"] ** (np.arange(0, hd, 2, dtype=np.float64) / hd)))

    def _r(self, x):
        return bf16_round(x) if self.emul else x.astype(np.float32)

    def _rms(self, x, g):
        ms = (x.astype(np.float64) ** 2).mean(axis=-1, keepdims=True)
        return (x / np.sqrt(ms + self.cfg["eps"]).astype(np.float32)) * g

    def _norm_in(self, x, g):
        """(GEMM input, row scale) of a normalised projection.  The device
        applies RMSNorm deferred (la_mega.cuh): the projection consumes
        bf16(x * g) and its fp32 accumulator is scaled by the row's
        rsqrt(mean(x^2) + eps) -- mathematically rms(x) * g @ W^T."""
        if not self.emul:
            return self._rms(x, g), np.float32(1.0)
        ms = (x.astype(np.float64) ** 2).mean(axis=-1, keepdims=True)
        rstd = (1.0 / np.sqrt(ms + self.cfg["eps"])).astype(np.float32)
        return bf16_round(x * g), rstd

    def _rope(self, x, pos):
        # x: (T, heads, hd); rotate-half convention
        hd = x.shape[-1]
        ang = np.asarray(pos, dtype=np.float64)[:, None] * self.inv_freq[None, :]
        c = np.cos(ang).astype(np.float32)[:, None, :]
        s = np.sin(ang).astype(np.float32)[:, None, :]
        x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)

    def _layer_kv(self, i, x, pos):
        c = self.cfg
        w = self.w
        T = x.shape[0]
        h, rs = self._norm_in(x, w[f"{i}.attn_norm"])
        # the device applies RoPE to the fp32 accumulator and stores bf16 once
        q = ((h @ w[f"{i}.wq"].T) * rs).reshape(T, c["heads"], c["head_dim"])
        k = ((h @ w[f"{i}.wk"].T) * rs).reshape(T, c["kv_heads"], c["head_dim"])
        v = self._r((h @ w[f"{i}.wv"].T) * rs).reshape(T, c["kv_heads"], c["head_dim"])
        q = self._r(self._rope(q, pos))
        k = self._r(self._rope(k, pos))
        return q, k, v

    def _attend(self, q, K, V, T0):
        """q: (T, H, hd) at positions T0..T0+T-1; K/V: (T0+T, KVH, hd), causal."""
        c = self.cfg
        T = q.shape[0]
        grp = c["heads"] // c["kv_heads"]
        Kx = np.repeat(K, grp, axis=1)
        Vx = np.repeat(V, grp, axis=1)
        sc = np.einsum("thd,shd->hts", q, Kx) / np.sqrt(c["head_dim"])
        S = Kx.shape[0]
        mask = np.arange(S)[None, :] > (T0 + np.arange(T))[:, None]
        sc = np.where(mask[None], -np.inf, sc)
        sc = sc - sc.max(axis=-1, keepdims=True)
        p = np.exp(sc)
        p /= p.sum(axis=-1, keepdims=True)
        return np.einsum("hts,shd->thd", p, Vx).reshape(T, -1).astype(np.float32)

    def _block(self, i, x, pos, K_prev, V_prev):
        w = self.w
        q, k, v = self._layer_kv(i, x, pos)
        K = k if K_prev is None else np.concatenate([K_prev, k], axis=0)
        V = v if V_prev is None else np.concatenate([V_prev, v], axis=0)
        T0 = K.shape[0] - x.shape[0]
        o = self._r(self._attend(q, K, V, T0))
        x = x + o @ w[f"{i}.wo"].T
        h, rs = self._norm_in(x, w[f"{i}.mlp_norm"])
        g = (h @ w[f"{i}.w_gate"].T) * rs
        u = (h @ w[f"{i}.w_up"].T) * rs
        a = self._r(g / (1.0 + np.exp(-g)) * u)
        x = x + a @ w[f"{i}.w_down"].T
        return x, K, V

    def run(self, tokens, start_pos=0, cache=None):
        """Causal forward of ``tokens`` on top of ``cache`` (list of (K, V))."""
        w = self.w
        x = w["embed"][np.asarray(tokens, dtype=np.int64)].astype(np.float32)
        pos = np.arange(start_pos, start_pos + len(tokens))
        new_cache = []
        for i in range(self.cfg["layers"]):
            Kp, Vp = (None, None) if cache is None else cache[i]
            x, K, V = self._block(i, x, pos, Kp, Vp)
            new_cache.append((K, V))
        return x, new_cache

    def final_logits(self, x_rows):
        w = self.w
        h, rs = self._norm_in(x_rows, w["final_norm"])
        return ((h @ w["lm_head"].T) * rs).astype(np.float32)

    def logits_rows(self, prefix, rows) -> list[np.ndarray]:
        prefix = [int(t) for t in prefix]
        cache = None
        if prefix:
            _, cache = self.run(prefix, 0)
        outs = []
        for i in range(len(rows)):
            chain = [rows.ids[c] for c in rows.chains[i]] + [rows.ids[i]]
            x, _ = self.run(chain, len(prefix), cache)
            outs.append(self.final_logits(x[-1:])[0])
        return outs

    def argmax_rows(self, prefix, rows) -> list[int]:
        return [int(np.argmax(l)) for l in self.logits_rows(prefix, rows)]


def llama_random_weights(cfg: dict, seed: int = 0, std: float | None = 0.02) -> dict:
    """bf16-representable float32 weights for tiny oracle checks.
    std=None draws each matrix with std 1/sqrt(in_features)."""
    rng = np.random.default_rng(seed)
    d, hd = cfg["dim"], cfg["head_dim"]
    H, KVH, F, V = cfg["heads"], cfg["kv_heads"], cfg["ffn"], cfg["vocab"]

    def mat(o, i, s=None):
        if s is None:
            s = std if std is not None else 1.0 / np.sqrt(i)
        return bf16_round(rng.normal(0.0, s, size=(o, i)).astype(np.float32))

    w = {"embed": mat(V, d, 1.0), "lm_head": mat(V, d),
         "final_norm": bf16_round(1.0 + 0.1 * rng.normal(size=d).astype(np.float32))}
    for i in range(cfg["layers"]):
        w[f"{i}.wq"] = mat(H * hd, d)
        w[f"{i}.wk"] = mat(KVH * hd, d)
        w[f"{i}.wv"] = mat(KVH * hd, d)
        w[f"{i}.wo"] = mat(d, H * hd)
        w[f"{i}.w_gate"] = mat(F, d)
        w[f"{i}.w_up"] = mat(F, d)
        w[f"{i}.w_down"] = mat(d, F)
        w[f"{i}.attn_norm"] = bf16_round(1.0 + 0.1 * rng.normal(size=d).astype(np.float32))
        w[f"{i}.mlp_norm"] = bf16_round(1.0 + 0.1 * rng.normal(size=d).astype(np.float32))
    return w
