"""f1 decode attention kernel (attention_decode.cu: split-KV, the K tile transposed onto the MMA rows).

Decode steps after a link over 128-token chunks (contexts of 5-8 K tiles, so the split-KV schedule cuts
every sequence into several pieces merged by attn_combine), for every GQA group size the kernel is built
for (G = 2, 4, 8), held to
  * the fp64 oracle's decode ("proceeds to the decode stage"; P.decode) at 2e-2;
  * the prefill kernel's decode path (PIC_NO_ATTN_DECODE=1, the one-lane kernel) at 2e-2, and not
    bit-identical to it — which shows the two runs took different kernels;
  * batched = single bit-exactly when the split schedule is the same (same batch composition)."""
import os
from dataclasses import replace

import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
STEPS = 6

MODELS = [
    sg.TINY_D128,                                                   # G = 2, one kv-head
    replace(sg.TINY_TP8, name="tiny-tp8-g4", n_kv_heads=4),         # G = 4 (Llama-3.1-8B / Mistral-7B)
    replace(sg.TINY_TP8, name="tiny-tp8-g8", n_kv_heads=2),         # G = 8 (Llama-3-70B)
]


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", params=MODELS, ids=lambda c: c.name)
def env(request):
    cfg = request.param
    ws = sg.workload_seed(0x52)
    chunks = sg.make_chunks(ws, 6, 128, cfg.vocab, cfg.bos_id) + sg.make_chunks(ws + 1, 1, 200, cfg.vocab, cfg.bos_id)
    eng = B.Engine(cfg, num_blocks=2048, max_rows=2048, max_tokens=2048, max_requests=4, device=0)
    ids = eng.generate_context_cache(chunks)
    Wt = M.Weights(cfg)
    store = P.Store(Wt)
    oids = store.compile(chunks)
    yield cfg, eng, ids, oids, Wt, store
    eng.close()


ORDERS = [[0, 1, 2, 3, 4], [6, 5, 0, 3, 2, 1]]


def test_decode_kernel_matches_oracle_and_prefill_kernel(env):
    cfg, eng, ids, oids, Wt, store = env
    q = sg.make_query(sg.workload_seed(0x52), 0, 24, cfg.vocab)
    toks = [int(t) for t in sg.tokens(0xDEC0DE, 9, STEPS, cfg.vocab, None)]
    for order in ORDERS:
        segs = [("cached", ids[c]) for c in order] + [("tokens", q)]
        outs = [eng.link(segs, "legolink:16", keep_linked=True) for _ in range(2)]
        ref = P.link(store, [("cached", oids[c]) for c in order] + [("tokens", q)], "legolink:16")
        K, V = ref.K, ref.V
        try:
            for i, t in enumerate(toks):
                d_new = eng.decode([outs[0].linked], [t], use_graph=False)
                assert B.last_attention_kernel() == 5                      # the split-KV decode kernel
                os.environ["PIC_NO_ATTN_DECODE"] = "1"
                try:
                    d_old = eng.decode([outs[1].linked], [t], use_graph=False)
                    assert B.last_attention_kernel() in (1, 2)             # a prefill kernel
                finally:
                    os.environ.pop("PIC_NO_ATTN_DECODE", None)
                lg, K, V = P.decode(Wt, K, V, t)
                assert rel(d_new.logits[0], lg) < 2e-2, (order, i)
                assert rel(d_new.logits[0], d_old.logits[0]) < 2e-2, (order, i)
                assert not np.array_equal(d_new.logits[0], d_old.logits[0])
                assert d_new.next_token[0] == int(np.argmax(d_new.logits[0]))
        finally:
            for o in outs:
                eng.release(o.linked)


def test_decode_kernel_batched_equals_single(env):
    cfg, eng, ids, oids, Wt, store = env
    q = sg.make_query(sg.workload_seed(0x52), 1, 17, cfg.vocab)
    reqs = [[("cached", ids[c]) for c in o] + [("tokens", q)] for o in ORDERS]
    a = [eng.link(r, "legolink:16", keep_linked=True) for r in reqs]
    b = [eng.link(r, "legolink:16", keep_linked=True) for r in reqs]
    c = [eng.link(r, "legolink:16", keep_linked=True) for r in reqs]
    try:
        ta = [x.first_token for x in a]
        for step in range(STEPS):
            batch = eng.decode([x.linked for x in a], ta)
            batch2 = eng.decode([x.linked for x in b], ta)      # same composition, same split schedule
            for j in range(len(a)):
                assert np.array_equal(batch.logits[j], batch2.logits[j]), (step, j)
            for j, (x, t) in enumerate(zip(c, ta)):
                single = eng.decode([x.linked], [t])
                assert rel(single.logits[0], batch.logits[j]) < 1e-2, (step, j)
            ta = [int(t) for t in batch.next_token]
    finally:
        for x in a + b + c:
            eng.release(x.linked)


@pytest.mark.parametrize("kv_share", [0, 3], ids=["copy", "chunk-frame"])
def test_decode_kernel_unsplit_large_batch(kv_share):
    """>= 148 (sequence, kv-head) items: the decode kernel runs them unsplit (no combine; the bench's batch-32
    decode takes this path).  20 sequences x 8 kv-heads of TINY_TP8 against the oracle's decode, and against
    the split schedule (PIC_DEC_SPLIT=1) within bf16 rounding.  kv_share 3 is the bench's own case: the
    batch decodes chunk-frame links directly, each sequence with its own per-frame Δ (reading R24)."""
    cfg = sg.TINY_TP8
    ws = sg.workload_seed(0x55)
    chunks = sg.make_chunks(ws, 6, 128, cfg.vocab, cfg.bos_id)
    eng = B.Engine(cfg, num_blocks=4096, max_rows=4096, max_tokens=1024, max_requests=20, device=0)
    try:
        ids = eng.generate_context_cache(chunks)
        Wt = M.Weights(cfg)
        store = P.Store(Wt)
        oids = store.compile(chunks)
        orders = [[(i + j) % 6 for j in range(3 + i % 3)] for i in range(20)]
        qs = [sg.make_query(ws, i, 8 + i, cfg.vocab) for i in range(20)]
        reqs = [[("cached", ids[c]) for c in o] + [("tokens", q)] for o, q in zip(orders, qs)]
        hs = [o.linked for o in eng.link_batch(reqs, "legolink:16", keep_linked=True, kv_share=kv_share)]
        hs2 = [o.linked for o in eng.link_batch(reqs, "legolink:16", keep_linked=True, kv_share=kv_share)]
        if kv_share == 3:
            assert any((eng.linked_sharing(h)[1] != 0).any() for h in hs)    # frames pending on the keys
        refs = [P.link(store, [("cached", oids[c]) for c in o] + [("tokens", q)], "legolink:16")
                for o, q in zip(orders, qs)]
        KV = [(r.K, r.V) for r in refs]
        for t in (3, 11):
            d = eng.decode(hs, [t] * 20, use_graph=False)
            assert B.last_attention_kernel() == 5
            os.environ["PIC_DEC_SPLIT"] = "1"
            try:
                d2 = eng.decode(hs2, [t] * 20, use_graph=False)
            finally:
                os.environ.pop("PIC_DEC_SPLIT", None)
            for b in range(20):
                lg, K, V = P.decode(Wt, KV[b][0], KV[b][1], t)
                KV[b] = (K, V)
                assert rel(d.logits[b], lg) < 2e-2, (t, b)
                assert rel(d.logits[b], d2.logits[b]) < 1e-2, (t, b)
        for h in hs + hs2:
            eng.release(h)
    finally:
        eng.close()


def test_decode_kernel_over_chunk_frame_links(env):
    """Decode over kv_share 3 links without materializing them: the cached keys still sit in their chunks'
    compile frames and the decode kernel rotates the query by −Δ per 128-key frame (the Q-side re-base,
    reading R24).  Against the oracle's decode and against decode after materialize (re-based copies)."""
    cfg, eng, ids, oids, Wt, store = env
    q = sg.make_query(sg.workload_seed(0x52), 2, 24, cfg.vocab)
    toks = [int(t) for t in sg.tokens(0xDEC0DE, 11, STEPS, cfg.vocab, None)]
    order = [0, 1, 2, 3, 4]
    segs = [("cached", ids[c]) for c in order] + [("tokens", q)]
    ha = eng.link(segs, "legolink:16", keep_linked=True, kv_share=3).linked
    hb = eng.link(segs, "legolink:16", keep_linked=True, kv_share=3).linked
    try:
        assert (eng.linked_sharing(ha)[1] != 0).any()           # frames still pending on the keys
        eng.materialize(hb)
        ref = P.link(store, [("cached", oids[c]) for c in order] + [("tokens", q)], "legolink:16")
        K, V = ref.K, ref.V
        for t in toks:
            da = eng.decode([ha], [t], use_graph=False)
            assert B.last_attention_kernel() == 5                      # the decode kernel, frames and all
            db = eng.decode([hb], [t], use_graph=False)
            lg, K, V = P.decode(Wt, K, V, t)
            assert rel(da.logits[0], lg) < 2e-2
            assert rel(da.logits[0], db.logits[0]) < 2e-2
    finally:
        eng.release(ha)
        eng.release(hb)


def test_decode_over_unaligned_chunk_frames(env):
    """Chunk-frame links whose chunks do not start on a 128-key tile (the 200-token chunk 6 first): the
    blocks of a tile may then carry different Δ, which the decode kernel's one-rotation-per-tile schedule
    cannot take, so the engine falls back to a prefill kernel with per-block rotation (or the decode kernel
    where every tile is uniform).  Whichever kernel runs, the decode must equal the oracle's."""
    cfg, eng, ids, oids, Wt, store = env
    q = sg.make_query(sg.workload_seed(0x52), 3, 9, cfg.vocab)
    toks = [int(t) for t in sg.tokens(0xDEC0DE, 13, 4, cfg.vocab, None)]
    for order in ([6, 0, 1, 2], [0, 6, 3]):
        segs = [("cached", ids[c]) for c in order] + [("tokens", q)]
        h = eng.link(segs, "legolink:16", keep_linked=True, kv_share=3).linked
        ref = P.link(store, [("cached", oids[c]) for c in order] + [("tokens", q)], "legolink:16")
        K, V = ref.K, ref.V
        try:
            for t in toks:
                d = eng.decode([h], [t], use_graph=False)
                assert B.last_attention_kernel() in (1, 2, 5)
                lg, K, V = P.decode(Wt, K, V, t)
                assert rel(d.logits[0], lg) < 2e-2, (order, t)
        finally:
            eng.release(h)
