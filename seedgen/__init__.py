"""Seeded synthetic-input generators shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no attention, RoPE, norms,
projections, selection rules).  It only defines *inputs*: model shapes,
random-init weights and token workloads, all drawn from the counter-based
generator fixed in SURVEY.md §8(c).6.  The CUDA path implements the same
generator independently in ``csrc/kernels/pointwise.cu`` (gen_matrix / gen_gateup kernels; it never imports
this module); the parity tests check the two bit-exactly.

Generator:
  sm64(x):  x += 0x9E3779B97F4A7C15; z = (x ^ x>>30) * 0xBF58476D1CE4E5B9;
            z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31   (mod 2^64)
  U(seed, tag, i) = sm64(sm64(seed ^ tag*0xD1B54A32D192ED03) + i)
  f = (U >> 40) * 2^-23 - 1            in [-1, 1), exact in fp32
  matrix weight  w = bf16_rne(f) * 2^e,  e = round(log2(sqrt(3 / fan_in)))
  embedding      e = 0
  norm gains     1 + ((U >> 61) - 4) / 32          (exact in bf16)
  tokens         chunk c offset j>=1: (U(wseed, 0xC0000000 + c, j) >> 33) % V,
                 offset 0 = BOS; query q: tag 0xD0000000 + q.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Tuple

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
TAGMUL = 0xD1B54A32D192ED03

# weight tags: layer*16 + offset
TAG_Q, TAG_K, TAG_V, TAG_O, TAG_GATE, TAG_UP, TAG_DOWN, TAG_G1, TAG_G2 = range(9)
TAG_EMBED = 0xE0000001
TAG_LM = 0xE0000002
TAG_GF = 0xE0000003
TAG_CHUNK = 0xC0000000
TAG_QUERY = 0xD0000000


def layer_tag(layer: int, which: int) -> int:
    return layer * 16 + which


# ----------------------------------------------------------------------------
# counter-based generator
# ----------------------------------------------------------------------------
def sm64_int(x: int) -> int:
    x = (x + GOLDEN) & M64
    z = ((x ^ (x >> 30)) * MIX1) & M64
    z = ((z ^ (z >> 27)) * MIX2) & M64
    return z ^ (z >> 31)


def _sm64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(GOLDEN)
        z = (x ^ (x >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, tag: int) -> int:
    return sm64_int((seed ^ ((tag * TAGMUL) & M64)) & M64)


def U(seed: int, tag: int, idx: np.ndarray) -> np.ndarray:
    """U(seed, tag, i) for an array of counters i (uint64)."""
    key = np.uint64(stream_key(seed, tag))
    with np.errstate(over="ignore"):
        return _sm64_np(key + np.asarray(idx, dtype=np.uint64))


def uniform_pm1(u: np.ndarray) -> np.ndarray:
    """f = (U>>40)*2^-23 - 1 as float32 (exact)."""
    return ((u >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23)) - np.float32(1.0)


def bf16_rne(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bfloat16 (ties to even); returned as float32."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (b >> np.uint32(16)) & np.uint32(1)
    with np.errstate(over="ignore"):
        r = (b + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def weight_exponent(fan_in: int) -> int:
    return int(round(math.log2(math.sqrt(3.0 / fan_in))))


def matrix(seed: int, tag: int, rows: int, cols: int, fan_in: Optional[int] = None,
           row0: int = 0, nrows: Optional[int] = None) -> np.ndarray:
    """Logical [rows][cols] weight (row-major counter i = r*cols + c), float32, bf16-exact.

    ``row0``/``nrows`` select a row slice without generating the rest (TP shards and
    sampled checks use this).  ``fan_in`` defaults to ``cols``; ``fan_in=0`` means
    exponent 0 (embedding)."""
    if nrows is None:
        nrows = rows - row0
    fi = cols if fan_in is None else fan_in
    e = 0 if fi == 0 else weight_exponent(fi)
    out = np.empty(nrows * cols, dtype=np.float32)
    scale = np.float32(2.0 ** e)

    def fill(a: int, b: int) -> None:
        idx = np.arange(row0 * cols + a, row0 * cols + b, dtype=np.uint64)
        out[a:b] = bf16_rne(uniform_pm1(U(seed, tag, idx))) * scale

    _parallel_ranges(nrows * cols, fill)
    return out.reshape(nrows, cols)


_POOL = None


def _parallel_ranges(n: int, fn, grain: int = 1 << 22) -> None:
    """fn(a, b) over [0, n) in slices on a thread pool (NumPy ufuncs release the GIL); element i
    depends only on its counter, so the result is independent of the split."""
    global _POOL
    if n <= grain:
        fn(0, n)
        return
    import concurrent.futures as cf
    import os
    if _POOL is None:
        try:
            nt = len(os.sched_getaffinity(0))
        except AttributeError:
            nt = os.cpu_count() or 1
        _POOL = cf.ThreadPoolExecutor(max_workers=max(1, nt))
    list(_POOL.map(lambda a: fn(a, min(n, a + grain)), range(0, n, grain)))


def gains(seed: int, tag: int, n: int) -> np.ndarray:
    u = U(seed, tag, np.arange(n, dtype=np.uint64))
    return (1.0 + ((u >> np.uint64(61)).astype(np.float32) - 4.0) / 32.0).astype(np.float32)


def tokens(seed: int, tag: int, n: int, vocab: int, bos: Optional[int]) -> np.ndarray:
    u = U(seed, tag, np.arange(n, dtype=np.uint64))
    t = ((u >> np.uint64(33)) % np.uint64(vocab)).astype(np.int32)
    if bos is not None and n > 0:
        t[0] = bos
    return t


# ----------------------------------------------------------------------------
# model shapes
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class ModelConfig:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    rope_theta: float
    max_pos: int
    seed: int
    rms_eps: float = 1e-5
    bos_id: int = 1
    dtype: int = 0      # engine numeric mode under test: 0 bf16 product, 1 fp32 debug build (not model data)

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def params_per_layer(self) -> int:
        d, D = self.d_model, self.head_dim
        return d * self.qkv_dim + self.n_heads * D * d + 3 * d * self.ffn_dim


TINY = ModelConfig("tiny", 2, 64, 4, 4, 16, 128, 256, 1e4, 4096, 0x5EED0001)
TINY_GQA = replace(TINY, name="tiny-gqa", n_kv_heads=2, seed=0x5EED0011)
TINY_D128 = ModelConfig("tiny-d128", 2, 256, 2, 1, 128, 512, 512, 1e4, 4096, 0x5EED0021)
TINY_TP = ModelConfig("tiny-tp", 2, 256, 4, 2, 128, 512, 512, 1e4, 4096, 0x5EED0031)   # shardable over 2 ranks
TINY_TP8 = ModelConfig("tiny-tp8", 2, 1024, 16, 8, 128, 1024, 1024, 1e4, 4096, 0x5EED0041)  # 8 kv-heads: TP 2/4/8
MISTRAL7B = ModelConfig("mistral7b", 32, 4096, 32, 8, 128, 14336, 32000, 1e6, 32768, 0x5EED0002)
LLAMA31_8B = ModelConfig("llama31_8b", 32, 4096, 32, 8, 128, 14336, 128256, 5e5, 32768, 0x5EED0003)
LLAMA3_70B = ModelConfig("llama3_70b", 80, 8192, 64, 8, 128, 28672, 128256, 5e5, 65536, 0x5EED0005)

MODELS = {m.name: m for m in (TINY, TINY_GQA, TINY_D128, TINY_TP, TINY_TP8, MISTRAL7B, LLAMA31_8B, LLAMA3_70B)}


def truncated(cfg: ModelConfig, n_layers: int) -> ModelConfig:
    """Same weights (same seed/tags) for the first ``n_layers`` layers."""
    return replace(cfg, n_layers=n_layers, name=f"{cfg.name}-L{n_layers}")


# ----------------------------------------------------------------------------
# workloads
# ----------------------------------------------------------------------------
@dataclass
class Segment:
    """One message-list entry: a cached chunk (by chunk index in ``Workload.chunks``)
    or literal dynamic tokens."""
    chunk: Optional[int] = None
    tokens: Optional[np.ndarray] = None

    @property
    def cached(self) -> bool:
        return self.chunk is not None


@dataclass
class Workload:
    name: str
    model: ModelConfig
    chunks: List[np.ndarray]                 # static token chunks (compile inputs)
    requests: List[List[Segment]]            # message lists, chunk refs index ``chunks``
    alg: str                                 # SPEC grammar: naive | fr | legolink:K | cacheblend:R
    note: str = ""


def workload_seed(cfg_no: int) -> int:
    return 0xC0FFEE00 + cfg_no


def make_chunks(wseed: int, n_chunks: int, chunk_len: int, vocab: int, bos: int) -> List[np.ndarray]:
    return [tokens(wseed, TAG_CHUNK + c, chunk_len, vocab, bos) for c in range(n_chunks)]


def make_query(wseed: int, q: int, n: int, vocab: int) -> np.ndarray:
    return tokens(wseed, TAG_QUERY + q, n, vocab, None)


def rag_workload(name: str, model: ModelConfig, cfg_no: int, n_chunks: int, chunk_len: int,
                 query_len: int, alg: str) -> Workload:
    ws = workload_seed(cfg_no)
    chunks = make_chunks(ws, n_chunks, chunk_len, model.vocab, model.bos_id)
    segs = [Segment(chunk=c) for c in range(n_chunks)]
    if query_len:
        segs.append(Segment(tokens=make_query(ws, 0, query_len, model.vocab)))
    return Workload(name, model, chunks, [segs], alg)


def cfg1(alg: str = "legolink:4", model: ModelConfig = TINY) -> Workload:
    return rag_workload("cfg1", model, 1, 3, 32, 16, alg)


def cfg2(alg: str = "legolink:16", n_layers: Optional[int] = None) -> Workload:
    m = MISTRAL7B if n_layers is None else truncated(MISTRAL7B, n_layers)
    return rag_workload("cfg2", m, 2, 5, 512, 64, alg)


def cfg3(alg: str = "legolink:32", n_layers: Optional[int] = None) -> Workload:
    m = LLAMA31_8B if n_layers is None else truncated(LLAMA31_8B, n_layers)
    return rag_workload("cfg3", m, 3, 20, 256, 0, alg)


def cfg4(n_requests: int = 256, corpus: int = 256, per_req: int = 10, chunk_len: int = 512,
         query_len: int = 64, alg: str = "legolink:16", n_layers: Optional[int] = None) -> Workload:
    """256 independent RAG requests; each draws ``per_req`` distinct chunks from a
    seeded corpus in seeded order, then a 64-token query."""
    m = LLAMA31_8B if n_layers is None else truncated(LLAMA31_8B, n_layers)
    ws = workload_seed(4)
    chunks = make_chunks(ws, corpus, chunk_len, m.vocab, m.bos_id)
    reqs = []
    for r in range(n_requests):
        # seeded partial Fisher-Yates driven by the counter generator
        u = U(ws, 0xA0000000 + r, np.arange(per_req, dtype=np.uint64))
        pool = list(range(corpus))
        pick = []
        for j in range(per_req):
            k = j + int(u[j] % np.uint64(corpus - j))
            pool[j], pool[k] = pool[k], pool[j]
            pick.append(pool[j])
        segs = [Segment(chunk=c) for c in pick]
        segs.append(Segment(tokens=make_query(ws, r, query_len, m.vocab)))
        reqs.append(segs)
    return Workload("cfg4", m, chunks, reqs, alg)


def cfg5(alg: str = "legolink:16", n_layers: Optional[int] = None) -> Workload:
    m = LLAMA3_70B if n_layers is None else truncated(LLAMA3_70B, n_layers)
    return rag_workload("cfg5", m, 5, 64, 512, 64, alg)


LLAMA31_8B_LONG = replace(LLAMA31_8B, name="llama31_8b_64k", max_pos=65536)   # long-context sweep (f3)


def long_context(n_chunks: int, alg: str = "legolink:16", n_layers: Optional[int] = None) -> Workload:
    """SURVEY §8(f) f3 / PAPER.md:307-316 (Fig. 8): n_chunks x 512-token chunks + a 64-token query,
    Llama-3.1-8B shape with a 64K position table."""
    m = LLAMA31_8B_LONG if n_layers is None else truncated(LLAMA31_8B_LONG, n_layers)
    return rag_workload(f"long{n_chunks}", m, 6, n_chunks, 512, 64, alg)


def permuted_requests(w: Workload, n_perm: int, seed: int = 0xBADC0DE) -> List[List[Segment]]:
    """Seeded permutations / interleavings of request 0's segments (cfg1 planner tests):
    includes dynamic-first orders, split queries and repeated cache ids."""
    base = w.requests[0]
    out = []
    for p in range(n_perm):
        u = U(seed, p, np.arange(16, dtype=np.uint64))
        segs = list(base)
        # shuffle
        for j in range(len(segs) - 1, 0, -1):
            k = int(u[j] % np.uint64(j + 1))
            segs[j], segs[k] = segs[k], segs[j]
        # split a literal segment in two around a chunk, repeat a chunk id sometimes
        lit = [i for i, s in enumerate(segs) if not s.cached]
        if lit and p % 3 == 1:
            i = lit[0]
            t = segs[i].tokens
            h = max(1, len(t) // 2)
            segs = segs[:i] + [Segment(tokens=t[:h])] + segs[i + 1:] + [Segment(tokens=t[h:])]
        if p % 4 == 2:
            ch = [s for s in segs if s.cached]
            if ch:
                segs.insert(int(u[15] % np.uint64(len(segs) + 1)), Segment(chunk=ch[0].chunk))
        out.append(segs)
    return out


def parse_alg(alg: str) -> Tuple[str, int]:
    """SPEC grammar: naive | fr | legolink:K | cacheblend:R | legolink0  ->  (name, param)."""
    if alg == "naive":
        return "naive", 0
    if alg == "legolink0":
        return "legolink0", 0
    if alg == "fr":
        return "fr", 0
    if alg.startswith("legolink:"):
        return "legolink", int(alg.split(":")[1])
    if alg.startswith("cacheblend:"):
        return "cacheblend", int(alg.split(":")[1])
    raise ValueError(f"unknown algorithm {alg!r}")
