"""PIC compile / plan / link oracle (fp64, step by step).  TEST INFRASTRUCTURE ONLY.

Follows the paper in its own order:
  * compile (§2.2 "each chunk is encoded with position IDs starting from
    zero, and the LLM performs only the prefill stage");
  * link ("retrieves and concatenates cached KV vectors and recomputes a
    subset"), with the four algorithms of Fig. 3:
      Naive      PAPER.md:166 "reuses cached KV vectors directly ... without any recomputation"
      FR         PAPER.md:166 "recomputes all KV vectors in the link step"
      CacheBlend PAPER.md:169-170 (steps 1-4) with the layer reading of PAPER.md:376
      LegoLink   PAPER.md:211 "recomputes each chunk's first k tokens (except the first
                 chunk)", PAPER.md:213-217 (E, Q/K/V, K_exp/V_exp, Eq. (1), O)
  * the block allocator / slot map model used to pin the engine's paged layout
    (block size 16, "16 is the block size of vLLM").

Readings of silent or ambiguous passages are listed in DESIGN.md §3 (R1..R20) and
cited inline as [Rn].
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

import seedgen as sg
from . import model as M

BLOCK = 16  # tokens per KV block


# ----------------------------------------------------------------------------
# KV store: compiled chunks (the "KVCache" of PAPER.md:185)
# ----------------------------------------------------------------------------
@dataclass
class Chunk:
    cid: int
    tokens: np.ndarray
    K: np.ndarray          # [L, n, H_kv, D] post-RoPE keys at positions c0..c0+n-1
    V: np.ndarray
    c0: int = 0            # compile position of the chunk's first row (0; m for a LegoLink-0 compile)


class Store:
    """Explicit-ID cache store: ids are monotone from 1, never reused
    (S:167-170); ``expire`` is idempotent."""

    def __init__(self, weights: M.Weights):
        self.W = weights
        self.chunks: Dict[int, Chunk] = {}
        self.next_id = 1

    def compile(self, chunk_tokens: Sequence[np.ndarray],
                compiled_override: Optional[Sequence[Tuple[np.ndarray, np.ndarray]]] = None,
                dummy_prefix: int = 0) -> List[int]:
        """generate_context_cache(static_token_chunks[]) -> cache_ids.
        Each chunk alone, positions 0..n−1, prefill only (no decode).  ``compiled_override``
        supplies (K, V) computed elsewhere (the GPU) for full-depth large-shape tests.

        ``dummy_prefix`` = m > 0 is the LegoLink-0 compile ("prepends four dummy
        tokens (e.g., begin-of-sentence tokens) to each immutable chunk during compilation, then
        discards their corresponding KV vectors"): prefill BOS^m ‖ chunk at positions
        0..m+n−1 and keep rows m..m+n−1, whose keys are rotated at positions m.. (c0 = m) [R21]."""
        ids = []
        m = int(dummy_prefix)
        if m < 0:
            raise ValueError("negative dummy prefix")
        for i, t in enumerate(chunk_tokens):
            t = np.asarray(t, dtype=np.int32)
            if len(t) == 0:
                raise ValueError("empty chunk")
            if compiled_override is not None:
                K, V = compiled_override[i]
            elif m == 0:
                _, K, V, _ = M.full_prefill(self.W, t)
            else:
                full = np.concatenate([np.full(m, self.W.cfg.bos_id, np.int32), t])
                _, K, V, _ = M.full_prefill(self.W, full)
                K, V = K[:, m:], V[:, m:]
            cid = self.next_id
            self.next_id += 1
            self.chunks[cid] = Chunk(cid, t.copy(), K, V, c0=m)
            ids.append(cid)
        return ids

    def expire(self, cid: int) -> bool:
        return self.chunks.pop(cid, None) is not None


# ----------------------------------------------------------------------------
# assemble + plan (step a1)
# ----------------------------------------------------------------------------
@dataclass
class Plan:
    tokens: np.ndarray                 # int32[N]
    src: np.ndarray                    # int32[N, 2]: (cache id, row) or (-1, -1) for dynamic
    chunks: List[Tuple[int, int, int, int]]   # (cid, start s_c, len n_c, delta Δ_c = s_c − c0)
    sel: np.ndarray                    # sorted int32 linked indices recomputed (pre-CacheBlend set)
    dynamic: np.ndarray                # int32 linked indices of literal tokens
    alg: str
    param: int

    @property
    def N(self) -> int:
        return len(self.tokens)

    @property
    def positions(self) -> np.ndarray:
        return np.arange(self.N, dtype=np.int32)   # p_i = i  [R18]


def assemble(store: Store, segments: Sequence[Tuple[str, object]]):
    """Concatenate segments in the given order (PAPER.md:391 'arranged in any order').
    ``segments`` is a list of ("cached", cid) / ("tokens", int array)."""
    toks, src, chunks, dyn = [], [], [], []
    pos = 0
    if len(segments) == 0:
        raise ValueError("empty message list")
    for kind, val in segments:
        if kind == "cached":
            c = store.chunks.get(int(val))
            if c is None:
                raise KeyError(f"missing cache id {val}")
            n = len(c.tokens)
            toks.append(c.tokens)
            src.extend((c.cid, j) for j in range(n))
            chunks.append((c.cid, pos, n, pos - c.c0))
            pos += n
        elif kind == "tokens":
            t = np.asarray(val, dtype=np.int32)
            if len(t) == 0:
                raise ValueError("empty literal segment")
            toks.append(t)
            src.extend((-1, -1) for _ in range(len(t)))
            dyn.extend(range(pos, pos + len(t)))
            pos += len(t)
        else:
            raise ValueError(kind)
    return (np.concatenate(toks).astype(np.int32), np.asarray(src, dtype=np.int32).reshape(-1, 2),
            chunks, np.asarray(dyn, dtype=np.int32))


def plan(store: Store, segments, alg: str) -> Plan:
    """Selected set per algorithm, then ∪ {N−1} [R8]."""
    name, param = sg.parse_alg(alg)
    tok, src, chunks, dyn = assemble(store, segments)
    N = len(tok)
    sel = set(int(i) for i in dyn)                      # literal tokens are always computed
    if name == "fr":
        sel = set(range(N))
    elif name == "naive":
        pass                                            # PAPER.md:166 (≡ LegoLink k=0)
    elif name == "legolink0":
        # PAPER.md:286 "in the link step, LegoLink-0 skips recomputation entirely": Naive over
        # chunks compiled with a dummy prefix (Δ = s_c − m, negative for a chunk placed at 0) [R21]
        for cid, s, n, _ in chunks:
            if store.chunks[cid].c0 <= 0:
                raise ValueError(f"legolink0 needs chunks compiled with a dummy prefix (cache id {cid})")
    elif name == "legolink":
        k = param
        for cid, s, n, _ in chunks:
            if s == 0:                                  # "(except the first chunk)" [R6]
                continue
            sel.update(range(s, s + min(k, n)))         # first k tokens of each chunk [R7]
    elif name == "cacheblend":
        pass                                            # decided at the check layer (link)
    sel.add(N - 1)                                      # first-token logits row [R8]
    return Plan(tok, src, chunks, np.asarray(sorted(sel), dtype=np.int32), dyn, name, param)


def cacheblend_count(plan: Plan) -> int:
    """T = ⌈R·N_cached/100⌉ cached tokens (PAPER.md:170 '15% of tokens') [R11], integer math."""
    n_cached = plan.N - len(plan.dynamic)
    return (plan.param * n_cached + 99) // 100


def cacheblend_select(plan: Plan, dev: np.ndarray) -> np.ndarray:
    """Top-T cached indices by deviation (ties → lower index [R13]), excluding the forced
    last row [R8/R11], ∪ dynamic ∪ {N−1}; sorted."""
    N = plan.N
    is_dyn = np.zeros(N, bool)
    is_dyn[plan.dynamic] = True
    cand = [i for i in range(N) if not is_dyn[i] and i != N - 1]
    T = min(cacheblend_count(plan), len(cand))
    cand.sort(key=lambda i: (-dev[i], i))
    keep = set(cand[:T]) | set(int(i) for i in plan.dynamic) | {N - 1}
    return np.asarray(sorted(keep), dtype=np.int32)


# ----------------------------------------------------------------------------
# link (KVLink, PAPER.md:185 and §4.2)
# ----------------------------------------------------------------------------
@dataclass
class LinkResult:
    logits: np.ndarray
    first_token: int
    K: np.ndarray                      # [L, N, H_kv, D] linked K (K_exp per layer)
    V: np.ndarray
    sel_per_layer: List[np.ndarray]
    hidden: List[np.ndarray]           # residual of the selected rows after each layer
    plan: Plan
    dev: Optional[np.ndarray] = None   # CacheBlend deviations (check layer)


def rebase(K: np.ndarray, delta: int, head_dim: int, theta: float) -> np.ndarray:
    """R(Δ)·K for post-RoPE keys K[n, H, D]: rotation of each pair by Δ·θ_j [R1].
    RoPE(k, p+Δ) = R(Δ)·RoPE(k, p) (pin C7)."""
    ang = M.rope_angles(np.full(K.shape[0], delta), head_dim, theta)
    return M.rotate(K, ang)


def link(store: Store, segments, alg: str, rebase_keys: bool = True, check_layer: int = 1,
         sel_override: Optional[np.ndarray] = None, layers: Optional[int] = None) -> LinkResult:
    """link(message_list, algorithm, k) -> linked KV + first-token logits (BASELINE north_star).

    ``layers`` truncates the depth (tests); ``sel_override`` replaces CacheBlend's selection
    (SURVEY §8(c).8 protocol (ii))."""
    W = store.W
    cfg = W.cfg
    L = cfg.n_layers if layers is None else layers
    pl = plan(store, segments, alg)
    N = pl.N
    pos_all = pl.positions

    # step 3 of §4.2: K_exp / V_exp initialised from cached chunks at correct positions
    K = np.zeros((L, N, cfg.n_kv_heads, cfg.head_dim))
    V = np.zeros_like(K)
    for cid, s, n, delta in pl.chunks:
        c = store.chunks[cid]
        for l in range(L):
            Kc = c.K[l]
            K[l, s:s + n] = rebase(Kc, delta, cfg.head_dim, cfg.rope_theta) if rebase_keys else Kc
            V[l, s:s + n] = c.V[l]

    sels, hidden = [], []
    dev = None
    if pl.alg == "cacheblend":
        # PAPER.md:170 step 2: recompute all KV vectors of the first layer(s)
        sel = np.arange(N, dtype=np.int32)
        h = W.embed_rows(pl.tokens)
        for l in range(L):
            if l == check_layer:
                # step 3: compare new vs old KV of the check layer [R9, R10]
                _, k_new, v_new = M.qkv(W.layer(l), cfg, h, pos_all)
                dev = (((k_new - K[l]) ** 2).sum(axis=(1, 2)) + ((v_new - V[l]) ** 2).sum(axis=(1, 2)))
                sel = (np.asarray(sorted(sel_override), dtype=np.int32) if sel_override is not None
                       else cacheblend_select(pl, dev))
                h = h[sel]                                # step 4: only these from now on [R12, R14]
            h = M.layer_rows(W.layer(l), cfg, h, pos_all[sel], sel, K[l], V[l])
            sels.append(sel)
            hidden.append(h.copy())
    else:
        sel = pl.sel
        h = W.embed_rows(pl.tokens[sel])                  # step 1: E (k', d)
        for l in range(L):
            h = M.layer_rows(W.layer(l), cfg, h, pos_all[sel], sel, K[l], V[l])
            sels.append(sel)
            hidden.append(h.copy())

    assert sel[-1] == N - 1
    logits = M.logits_of(W, h[-1])
    tok1 = int(np.argmax(logits))                         # ties → lowest id [R20]
    return LinkResult(logits, tok1, K, V, sels, hidden, pl, dev)


# ----------------------------------------------------------------------------
# paged layout model (D3/D5): deterministic lowest-free-id-first allocator
# ----------------------------------------------------------------------------
class BlockAllocator:
    """Model of the engine's block allocator: one block id spans all layers' K and V;
    allocation takes the lowest free ids in increasing order; frees return ids.  Blocks are
    reference counted (a chunk-store block linked by reference is also held by the linked
    cache, see share_blocks): release returns an id to the free set at its last reference."""

    def __init__(self, num_blocks: int):
        self.free = set(range(num_blocks))
        self.refs: Dict[int, int] = {}

    def retain(self, b: int) -> None:
        self.refs[int(b)] += 1

    def peek(self, n: int) -> List[int]:
        return sorted(self.free)[:n]

    def alloc(self, n: int) -> List[int]:
        if n > len(self.free):
            raise MemoryError("pool full")
        ids = sorted(self.free)[:n]
        self.free.difference_update(ids)
        for i in ids:
            self.refs[i] = 1
        return ids

    def release(self, ids: Sequence[int]) -> None:
        for i in ids:
            i = int(i)
            self.refs[i] = self.refs.get(i, 1) - 1
            if self.refs[i] == 0:
                self.free.add(i)


def share_blocks(pl: Plan, chunk_blocks: Dict[int, Sequence[int]], rebase: bool = True):
    """Shared-block link layout: linked block b (rows 16b..16b+15)
    is the chunk-store block of chunk c holding rows 16b − s_c .. 16b − s_c + 15 — linked by
    reference instead of copied — iff s_c is a multiple of 16 and all 16 rows are unselected rows
    of c; its keys then still carry Δ_c (0 without re-base) to apply when they are read.
    CacheBlend shares nothing (its layer 0 rewrites every row).  Returns (shared, delta) per linked
    block: store block id or -1, and Δ (0 for fresh blocks)."""
    nb = n_blocks(pl.N)
    shared, delta = [-1] * nb, [0] * nb
    if pl.alg == "cacheblend":
        return shared, delta
    sel = set(int(i) for i in pl.sel)
    for cid, s0, n, dl in pl.chunks:
        if s0 % BLOCK:
            continue
        for j in range(0, n - BLOCK + 1, BLOCK):
            if any(s0 + j + r in sel for r in range(BLOCK)):
                continue
            shared[(s0 + j) // BLOCK] = int(chunk_blocks[cid][j // BLOCK])
            delta[(s0 + j) // BLOCK] = int(dl) if rebase else 0
    return shared, delta


def n_blocks(n_tokens: int) -> int:
    return (n_tokens + BLOCK - 1) // BLOCK


def slot_map(block_table: Sequence[int], rows: Sequence[int]) -> np.ndarray:
    """slot[i] = blk[i // 16]·16 + i % 16 (D5)."""
    bt = np.asarray(block_table, dtype=np.int64)
    r = np.asarray(rows, dtype=np.int64)
    return (bt[r // BLOCK] * BLOCK + r % BLOCK).astype(np.int32)


# ----------------------------------------------------------------------------
# decode over the linked cache
# ----------------------------------------------------------------------------
def decode(W: M.Weights, K: np.ndarray, V: np.ndarray, token: int):
    """One decode step (PAPER.md:141 "proceeds to the decode stage", :185): the new token at position
    N = len(K[0]) attends to keys 0..N — the linked cache plus its own K/V, which are appended
    (PAPER.md:217 causal mask).  K, V: [L, N, H_kv, D].  Returns (logits, K', V') with N + 1 rows."""
    cfg = W.cfg
    L, N = K.shape[0], K.shape[1]
    pad = np.zeros((L, 1) + K.shape[2:])
    K2 = np.concatenate([K, pad], axis=1)
    V2 = np.concatenate([V, pad], axis=1)
    h = W.embed_rows(np.asarray([token], dtype=np.int32))
    row = np.asarray([N])
    for l in range(L):
        h = M.layer_rows(W.layer(l), cfg, h, row, row, K2[l], V2[l])
    return M.logits_of(W, h[-1]), K2, V2
