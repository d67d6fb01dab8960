"""fp64 reference decoder used by the PIC oracle.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2410_15332_b200``) and never imports it.

The paper's layer sketch (§4.2 "The LegoLink Algorithm") is
``Q = E W_Q, K = E W_K, V = E W_V; A = softmax(Q K_exp^T · MASK); O = A V_exp W_O``.
It omits scale, norms, residuals, MLP and GQA; the models it evaluates are
Llama-family ("Mistral 7B, Llama 3.1 8B, Yi Coder 9B"), so the
standard pre-norm Llama decoder is the reading (readings R3/R4):

  x = rms(h) ⊙ g1;  q,k,v = x W_q^T, x W_k^T, x W_v^T;  q,k ← RoPE(·, pos)
  a = softmax(q k^T / √D + M) v     (M_ij = 0 if key j ≤ pos_i else −∞, GQA map)
  h += a W_o^T;  x = rms(h) ⊙ g2;  h += (silu(x W_g^T) ⊙ x W_u^T) W_d^T
  logits = (rms(h_last) ⊙ g_f) W_lm^T

Everything here is float64 NumPy; weights are the bf16-exact values from
``seedgen`` upcast to float64.
"""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np

import seedgen as sg


class Weights:
    """Lazily generated fp64 weights of a ``seedgen.ModelConfig``.

    Per-layer matrices are generated on first use and cached (``cache_layers``
    bounds the cache so full-width 7B/8B layers can be streamed)."""

    def __init__(self, cfg: sg.ModelConfig, cache_layers: int = 1 << 30):
        self.cfg = cfg
        self.cache_layers = cache_layers
        self._layers: Dict[int, Dict[str, np.ndarray]] = {}
        self._embed: Optional[np.ndarray] = None
        self._lm: Optional[np.ndarray] = None
        self._gf: Optional[np.ndarray] = None

    def layer(self, l: int) -> Dict[str, np.ndarray]:
        if l in self._layers:
            return self._layers[l]
        c = self.cfg
        s, d, D, F = c.seed, c.d_model, c.head_dim, c.ffn_dim
        T = lambda w: sg.layer_tag(l, w)
        W = {
            "q": sg.matrix(s, T(sg.TAG_Q), c.n_heads * D, d),
            "k": sg.matrix(s, T(sg.TAG_K), c.n_kv_heads * D, d),
            "v": sg.matrix(s, T(sg.TAG_V), c.n_kv_heads * D, d),
            "o": sg.matrix(s, T(sg.TAG_O), d, c.n_heads * D),
            "gate": sg.matrix(s, T(sg.TAG_GATE), F, d),
            "up": sg.matrix(s, T(sg.TAG_UP), F, d),
            "down": sg.matrix(s, T(sg.TAG_DOWN), d, F),
            "g1": sg.gains(s, T(sg.TAG_G1), d),
            "g2": sg.gains(s, T(sg.TAG_G2), d),
        }
        W = {k: v.astype(np.float64) for k, v in W.items()}
        if len(self._layers) >= self.cache_layers:
            self._layers.pop(next(iter(self._layers)))
        self._layers[l] = W
        return W

    @property
    def embed(self) -> np.ndarray:
        if self._embed is None:
            c = self.cfg
            self._embed = sg.matrix(c.seed, sg.TAG_EMBED, c.vocab, c.d_model, fan_in=0).astype(np.float64)
        return self._embed

    def embed_rows(self, tok: np.ndarray) -> np.ndarray:
        """Rows E[tok] without materialising E (large vocabularies)."""
        if self._embed is not None:
            return self._embed[tok]
        c = self.cfg
        out = np.empty((len(tok), c.d_model))
        for i, t in enumerate(np.asarray(tok)):
            out[i] = sg.matrix(c.seed, sg.TAG_EMBED, c.vocab, c.d_model, fan_in=0, row0=int(t), nrows=1)[0]
        return out

    @property
    def lm_head(self) -> np.ndarray:
        if self._lm is None:
            c = self.cfg
            self._lm = sg.matrix(c.seed, sg.TAG_LM, c.vocab, c.d_model).astype(np.float64)
        return self._lm

    @property
    def g_final(self) -> np.ndarray:
        if self._gf is None:
            c = self.cfg
            self._gf = sg.gains(c.seed, sg.TAG_GF, c.d_model).astype(np.float64)
        return self._gf


# ----------------------------------------------------------------------------
# primitives
# ----------------------------------------------------------------------------
def rms_norm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    """rms(x) ⊙ g with rms(x) = x / sqrt(mean(x²) + ε)  (Llama RMSNorm, reading R4)."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def rope_angles(pos: np.ndarray, head_dim: int, theta: float) -> np.ndarray:
    """angle[i, j] = pos_i · θ^(−2j/D), j < D/2, in fp64 (reading R2: NeoX pairs (j, j+D/2))."""
    j = np.arange(head_dim // 2, dtype=np.float64)
    inv_freq = theta ** (-2.0 * j / head_dim)
    return np.asarray(pos, dtype=np.float64)[:, None] * inv_freq[None, :]


def rotate(x: np.ndarray, ang: np.ndarray) -> np.ndarray:
    """Rotate pairs (x_j, x_{j+D/2}) of x[n, H, D] by ang[n, D/2] (same angle for every head)."""
    h = x.shape[-1] // 2
    c = np.cos(ang)[:, None, :]
    s = np.sin(ang)[:, None, :]
    x1, x2 = x[..., :h], x[..., h:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """RoPE(x, p) = R(p)·x for x[n, H, D] at positions pos[n]."""
    return rotate(x, rope_angles(pos, x.shape[-1], theta))


def causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, q_pos: np.ndarray) -> np.ndarray:
    """Eq. (1) with MASK as additive −∞ (reading R5) and 1/√D scale.

    q[n_q, H_q, D] at positions q_pos; k, v[n_k, H_kv, D] at positions 0..n_k−1.
    Query i sees key j iff j ≤ q_pos[i] ("attend to only tokens before them").
    GQA head map g(h) = ⌊h·H_kv/H_q⌋.  Returns a[n_q, H_q, D]."""
    n_q, H_q, D = q.shape
    n_k, H_kv, _ = k.shape
    out = np.empty_like(q)
    keypos = np.arange(n_k)
    mask = keypos[None, :] > np.asarray(q_pos)[:, None]          # [n_q, n_k]
    for h in range(H_q):
        g = h * H_kv // H_q
        s = q[:, h, :] @ k[:, g, :].T / np.sqrt(D)
        s = np.where(mask, -np.inf, s)
        s = s - s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=1, keepdims=True)
        out[:, h, :] = p @ v[:, g, :]
    return out


def attention_matrix_dense(q: np.ndarray, k: np.ndarray) -> np.ndarray:
    """Explicit softmax matrix for one head (pin C1): q[n, D], k[n, D], causal over indices."""
    n, D = q.shape
    s = q @ k.T / np.sqrt(D)
    a = np.zeros((n, n))
    for i in range(n):
        row = s[i, : i + 1]
        e = np.exp(row - row.max())
        a[i, : i + 1] = e / e.sum()
    return a


def qkv(W: Dict[str, np.ndarray], cfg: sg.ModelConfig, h: np.ndarray, pos: np.ndarray):
    """Step 2 of PAPER.md:213 (Q = E W_Q, K = E W_K, V = E W_V) on the pre-norm input,
    then RoPE at the rows' absolute positions.  Returns q[n,H_q,D], k, v[n,H_kv,D]."""
    n = h.shape[0]
    x = rms_norm(h, W["g1"], cfg.rms_eps)
    q = (x @ W["q"].T).reshape(n, cfg.n_heads, cfg.head_dim)
    k = (x @ W["k"].T).reshape(n, cfg.n_kv_heads, cfg.head_dim)
    v = (x @ W["v"].T).reshape(n, cfg.n_kv_heads, cfg.head_dim)
    return rope(q, pos, cfg.rope_theta), rope(k, pos, cfg.rope_theta), v


def layer_rows(W: Dict[str, np.ndarray], cfg: sg.ModelConfig, h: np.ndarray, pos: np.ndarray,
               sel: np.ndarray, K_l: np.ndarray, V_l: np.ndarray) -> np.ndarray:
    """One decoder layer for the selected rows.

    h[k', d] are the residual rows of linked indices ``sel`` (positions ``pos``).
    K_l, V_l[N, H_kv, D] are this layer's expanded K_exp / V_exp; the recomputed rows'
    K/V are written into them at ``sel`` BEFORE attention (step 3: "expand the K and V
    matrices by incorporating the cached KV vectors of the N − k' unselected tokens at
    correct positions"), so selected rows also see each other.  Returns the new h."""
    n = h.shape[0]
    q, k, v = qkv(W, cfg, h, pos)
    K_l[sel] = k
    V_l[sel] = v
    a = causal_attention(q, K_l, V_l, pos)
    h = h + a.reshape(n, -1) @ W["o"].T
    x = rms_norm(h, W["g2"], cfg.rms_eps)
    return h + (silu(x @ W["gate"].T) * (x @ W["up"].T)) @ W["down"].T


def logits_of(Wt: Weights, h_last: np.ndarray) -> np.ndarray:
    """logits = (rms(h_last) ⊙ g_f) W_lm^T  (first output token)."""
    x = rms_norm(h_last, Wt.g_final, Wt.cfg.rms_eps)
    return x @ Wt.lm_head.T


def full_prefill(Wt: Weights, tok: np.ndarray):
    """Ordinary causal prefill of a whole prompt at positions 0..N−1 (the definition FR,
    saturated LegoLink and the compile step reduce to).  Returns (logits, K[L], V[L], h_final)."""
    cfg = Wt.cfg
    N = len(tok)
    pos = np.arange(N)
    sel = np.arange(N)
    h = Wt.embed_rows(tok)
    K = np.zeros((cfg.n_layers, N, cfg.n_kv_heads, cfg.head_dim))
    V = np.zeros_like(K)
    for l in range(cfg.n_layers):
        h = layer_rows(Wt.layer(l), cfg, h, pos, sel, K[l], V[l])
    return logits_of(Wt, h[-1]), K, V, h
