"""Chunk-frame link (kv_share 3) on the Q-side re-base kernel (QROT) at small sizes.

kv_share 3 leaves every block of an aligned cached chunk in the chunk's compile frame; when every
128-key K tile carries one frame Δ the one-lane attention kernel re-bases the QUERIES instead of the
keys: q·R(Δ)k = (R(−Δ)q)·k (PAPER.md:213 step 3, "incorporating the cached KV vectors … at correct
positions"; the RoPE identity of §3, reading R1), R(−Δ)·q built once per frame by the rotation warps.
These tests use 128-token chunks (D = 128) so the QROT kernel runs, at every GQA group size the
kernel is instantiated for (G = 2, 4, 8), and hold it to

  * the fp64 oracle (logits, every layer's linked K re-based on export) at the north star's 2e-2;
  * the copy path (kv_share 0) at 2e-2 (not bit-identical: the rotated operand is rounded once more);
  * the K-tile re-base of the same chunk-frame link (PIC_NO_QROT=1) — close, and NOT bit-identical,
    which proves the two runs took different kernels.
"""
import os
from dataclasses import replace

import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu

MODELS = [
    sg.TINY_D128,                                                            # Hq 2, Hkv 1: G = 2
    replace(sg.TINY_TP8, name="tiny-tp8-g4", n_kv_heads=4),                  # G = 4 (Llama-3.1-8B's group)
    replace(sg.TINY_TP8, name="tiny-tp8-g8", n_kv_heads=2),                  # G = 8 (Llama-3-70B's group)
]


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", params=MODELS, ids=lambda c: c.name)
def env(request):
    cfg = request.param
    # 4 chunks x 128 tokens (+ one of 256) and a 40-token query: every K tile lies inside one chunk frame
    ws = sg.workload_seed(0x51)
    chunks = sg.make_chunks(ws, 4, 128, cfg.vocab, cfg.bos_id) + sg.make_chunks(ws + 1, 1, 256, cfg.vocab, cfg.bos_id)
    q = sg.make_query(ws, 0, 40, cfg.vocab)
    eng = B.Engine(cfg, num_blocks=1024, max_rows=1024, max_tokens=2048, max_requests=2, device=0)
    ids = eng.generate_context_cache(chunks)
    store = P.Store(M.Weights(cfg))
    oids = store.compile(chunks)
    yield cfg, eng, ids, oids, store, q
    eng.close()


ORDERS = [[0, 1, 2, 3, 4], [4, 2, 0, 3, 1], [3, 4, 1]]


@pytest.mark.parametrize("order", ORDERS, ids=lambda o: "-".join(map(str, o)))
@pytest.mark.parametrize("alg", ["naive", "legolink:16", "legolink:32"])
def test_qrot_link_matches_oracle_and_copy(env, alg, order):
    cfg, eng, ids, oids, store, q = env
    segs = [("cached", ids[c]) for c in order] + [("tokens", q)]
    ref = P.link(store, [("cached", oids[c]) for c in order] + [("tokens", q)], alg)
    outs, kinds = {}, {}
    try:
        for name, share, noq in (("copy", 0, False), ("qrot", 3, False), ("krot", 3, True)):
            if noq:
                os.environ["PIC_NO_QROT"] = "1"
            try:
                outs[name] = eng.link(segs, alg, keep_linked=True, kv_share=share, use_graph=False)
                kinds[name] = B.last_attention_kernel()
            finally:
                os.environ.pop("PIC_NO_QROT", None)
        qr, cp, kr = outs["qrot"], outs["copy"], outs["krot"]
        assert rel(qr.logits, ref.logits) < 2e-2
        assert rel(qr.logits, cp.logits) < 2e-2
        assert rel(qr.logits, kr.logits) < 2e-2
        assert qr.first_token == int(np.argmax(qr.logits))
        # Q-side and K-side re-base round different operands: equal results would mean one kernel ran twice
        assert not np.array_equal(qr.logits, kr.logits)
        assert kinds["qrot"] in (3, 4) and kinds["krot"] in (1, 2), kinds
        for l in range(cfg.n_layers):
            k, v = eng.linked_export(qr.linked, l)
            assert rel(B.bf16_bits_to_f32(k), ref.K[l]) < 2e-2, l
            assert rel(B.bf16_bits_to_f32(v), ref.V[l]) < 2e-2, l
    finally:
        for o in outs.values():
            eng.release(o.linked)


def test_qrot_batch_matches_oracle(env):
    """Two requests with different frame sequences in one link_batch (one QROT launch per layer over both
    sequences' q-tiles): each held to its own oracle link."""
    cfg, eng, ids, oids, store, q = env
    batch = eng.link_batch([[("cached", ids[c]) for c in o] + [("tokens", q)] for o in ORDERS[:2]], "legolink:16",
                           kv_share=3)
    for o, b in zip(ORDERS[:2], batch):
        ref = P.link(store, [("cached", oids[c]) for c in o] + [("tokens", q)], "legolink:16")
        assert rel(b.logits, ref.logits) < 2e-2


def _eager_links(eng, reqs, persistent):
    # small batches run the one-CTA kernel by default (fewer than 2 items per SM): force either kernel
    key = "PIC_ATTN_PERSIST" if persistent else "PIC_NO_ATTN_PERSIST"
    os.environ[key] = "1"
    try:
        out = eng.link_batch(reqs, "legolink:16", kv_share=3, use_graph=False, keep_linked=True)
        assert B.last_attention_kernel() == (4 if persistent else 3)  # persistent / one-CTA chunk-frame kernel
        return out
    finally:
        os.environ.pop(key, None)


def test_qrot_persistent_kernel_bit_identical(env):
    """attention_qp.cu (the persistent QROT kernel, the default for these links) against the one-CTA-per-item
    QROT kernel (PIC_NO_ATTN_PERSIST=1): same arithmetic, so logits and every layer's linked K/V are equal bit
    for bit, for a batch whose items cross CTA boundaries (eager launches: the env switch picks the kernel)."""
    cfg, eng, ids, oids, store, q = env
    reqs = [[("cached", ids[c]) for c in o] + [("tokens", q)] for o in ORDERS[:2]]
    a = _eager_links(eng, reqs, True)
    b = _eager_links(eng, reqs, False)
    try:
        for x, y in zip(a, b):
            assert np.array_equal(x.logits, y.logits)
            for l in range(cfg.n_layers):
                kx, vx = eng.linked_export(x.linked, l)
                ky, vy = eng.linked_export(y.linked, l)
                assert np.array_equal(kx, ky) and np.array_equal(vx, vy), l
    finally:
        for o in a + b:
            eng.release(o.linked)
