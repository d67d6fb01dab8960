"""Shared-block link (pic_link_params.kv_share): chunk-store blocks are linked by
reference and the attention kernels re-base their keys when they load them (rebase_pair, the a2
arithmetic), so the result must be BIT-IDENTICAL to the copy path (kv_share = 0): logits, first
token, every exported linked K/V row of every layer, and later decode steps.  The copy path itself
is held to the oracle by test_gpu_link / test_gpu_decode; one oracle check is repeated here.

Also: block accounting (only fresh blocks are taken from the pool; shared blocks are reference
counted, so expiring a chunk under a live linked cache keeps its rows) and the fp32 debug build."""
import os
from dataclasses import replace

import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
ALGS = ["naive", "legolink:4", "legolink:16", "fr"]


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


class Setup:
    def __init__(self, cfg, dummy_prefix=0):
        self.cfg = cfg
        self.w = sg.cfg1(model=cfg)
        self.eng = B.Engine(cfg, num_blocks=512, max_rows=1024, max_tokens=4096, max_requests=4, device=0)
        self.eids = self.eng.generate_context_cache(self.w.chunks, dummy_prefix=dummy_prefix)

    def segs(self, segs):
        return [("cached", self.eids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]


@pytest.fixture(scope="module", autouse=True, params=[1, 2], ids=lambda k: f"attn-kernel{k}")
def attention_kernel(request):
    """Copy and shared links on the same attention kernel (the engine picks per link: forced here), both
    the one-lane (1) and the ping-pong (2) kernel's K-tile re-base; D < 128 configs use the SIMT kernel."""
    B.set_attention_kernel(request.param)
    yield request.param
    B.set_attention_kernel(0)


@pytest.fixture(scope="module", params=[sg.TINY, sg.TINY_GQA, sg.TINY_D128], ids=lambda c: c.name)
def setup(request):
    s = Setup(request.param)
    yield s
    s.eng.close()


def link_both(s, segs, alg, modes=(0, 1), **kw):
    """(copy, shared) link outputs with their exported linked K/V of every layer."""
    outs = []
    for share in modes:
        free0 = s.eng.stats()["free_blocks"]
        o = s.eng.link(s.segs(segs), alg, keep_linked=True, kv_share=share, **kw)
        used = free0 - s.eng.stats()["free_blocks"]
        kv = [s.eng.linked_export(o.linked, l) for l in range(s.cfg.n_layers)]
        ns, bd = s.eng.linked_sharing(o.linked)
        outs.append((o, kv, used, ns, bd))
    return outs


def assert_identical(a, b):
    (oa, kva, _, _, _), (ob, kvb, _, _, _) = a, b
    assert np.array_equal(oa.logits, ob.logits)
    assert oa.first_token == ob.first_token
    for l, ((ka, va), (kb, vb)) in enumerate(zip(kva, kvb)):
        assert np.array_equal(ka, kb), l
        assert np.array_equal(va, vb), l


@pytest.mark.parametrize("alg", ALGS)
def test_shared_link_bit_identical_to_copy(setup, alg):
    s = setup
    any_shared = 0
    for segs in [s.w.requests[0]] + sg.permuted_requests(s.w, 6):
        copy, shared = link_both(s, segs, alg)
        try:
            assert_identical(copy, shared)
            n_blocks = (copy[0].n_tokens + 15) // 16
            assert copy[3] == 0 and copy[2] == n_blocks
            assert shared[2] == n_blocks - shared[3]          # only fresh blocks come from the pool
            if alg == "fr":
                assert shared[3] == 0
            any_shared += shared[3]
            # the plan agrees with what the link did
            pe = s.eng.plan(s.segs(segs), alg, kv_share=True)
            assert pe["n_shared"] == shared[3] and pe["block_delta"].tolist() == shared[4].tolist()
        finally:
            s.eng.release(copy[0].linked)
            s.eng.release(shared[0].linked)
    if alg != "fr":
        assert any_shared > 0


@pytest.mark.parametrize("alg", ALGS)
def test_vshare_link_bit_identical_to_copy(setup, alg):
    """kv_share 2: V linked by reference to the chunk-store blocks (separate V block table), keys re-based
    by a2 into fresh blocks: bit-identical to the copy path; every block is fresh for K, the V-shared
    blocks hold one extra reference on their store block, and releasing returns the pool exactly."""
    s = setup
    any_shared = 0
    free0 = s.eng.stats()["free_blocks"]
    for segs in [s.w.requests[0]] + sg.permuted_requests(s.w, 6):
        copy, vsh = link_both(s, segs, alg, modes=(0, 2))
        try:
            assert_identical(copy, vsh)
            n_blocks = (copy[0].n_tokens + 15) // 16
            assert vsh[2] == n_blocks                        # K needs a fresh block everywhere
            assert not vsh[4].any()                          # nothing for the attention to re-base
            if alg == "fr":
                assert vsh[3] == 0
            any_shared += vsh[3]
        finally:
            s.eng.release(copy[0].linked)
            s.eng.release(vsh[0].linked)
    assert s.eng.stats()["free_blocks"] == free0
    if alg != "fr":
        assert any_shared > 0


def test_vshare_decode_bit_identical(setup):
    """Decode over a kv_share 2 linked cache reads V through the V block table: identical to the copy path."""
    s = setup
    segs = s.w.requests[0]
    hs = [s.eng.link(s.segs(segs), "legolink:4", keep_linked=True, kv_share=share).linked for share in (0, 2)]
    try:
        for t in [5, 17, 99, 3, 250, 7, 11, 13, 2, 1, 0, 8, 9, 10, 12, 14, 15, 16, 18, 19]:
            a = s.eng.decode([hs[0]], [t])
            b = s.eng.decode([hs[1]], [t])
            assert np.array_equal(a.logits, b.logits)
        for l in range(s.cfg.n_layers):
            ka, va = s.eng.linked_export(hs[0], l)
            kb, vb = s.eng.linked_export(hs[1], l)
            assert np.array_equal(ka, kb) and np.array_equal(va, vb), l
    finally:
        for h in hs:
            s.eng.release(h)


@pytest.mark.parametrize("alg", ["naive", "legolink:4", "legolink:16"])
def test_chunkframe_link_matches_oracle(setup, alg):
    """kv_share 3: every block inside an aligned cached chunk keeps the chunk's compile frame (recomputed
    rows' keys are RoPE'd at their compile positions, a2 copies unselected rows without re-base) and the
    attention applies R(Δ) per block — or, when every K tile has one frame, rotates the queries by −Δ
    instead.  Not bit-identical to the copy path (one more bf16 rounding of the rotated operand): held to
    the oracle at the north star's 2e-2, and its linked K/V exports (re-based to the linked positions on
    export) to the copy path's within bf16 rounding."""
    s = setup
    store = P.Store(M.Weights(s.cfg))
    oids = store.compile(s.w.chunks)
    for segs in [s.w.requests[0]] + sg.permuted_requests(s.w, 3):
        ref = P.link(store, [("cached", oids[x.chunk]) if x.cached else ("tokens", x.tokens) for x in segs], alg)
        copy, cf = link_both(s, segs, alg, modes=(0, 3))
        try:
            assert rel(cf[0].logits, ref.logits) < 2e-2
            assert rel(cf[0].logits, copy[0].logits) < 2e-2
            for l in range(s.cfg.n_layers):
                (kc, vc), (kf, vf) = copy[1][l], cf[1][l]
                if l == 0:                                   # before any attention: V identical
                    assert np.array_equal(vc, vf)
                assert rel(B.bf16_bits_to_f32(vf), B.bf16_bits_to_f32(vc)) < 2e-2, l
                assert rel(B.bf16_bits_to_f32(kf), B.bf16_bits_to_f32(kc)) < 2e-2, l
                assert rel(B.bf16_bits_to_f32(kf), ref.K[l]) < 2e-2, l
        finally:
            s.eng.release(copy[0].linked)
            s.eng.release(cf[0].linked)


def test_shared_link_matches_oracle(setup):
    s = setup
    store = P.Store(M.Weights(s.cfg))
    oids = store.compile(s.w.chunks)
    segs = s.w.requests[0]
    out = s.eng.link(s.segs(segs), "legolink:4", keep_linked=True, kv_share=True)
    ref = P.link(store, [("cached", oids[x.chunk]) if x.cached else ("tokens", x.tokens) for x in segs], "legolink:4")
    try:
        assert s.eng.linked_sharing(out.linked)[0] > 0
        assert rel(out.logits, ref.logits) < 2e-2
        for l in range(s.cfg.n_layers):
            k, v = s.eng.linked_export(out.linked, l)
            assert rel(B.bf16_bits_to_f32(k), ref.K[l]) < 2e-2, l
            assert rel(B.bf16_bits_to_f32(v), ref.V[l]) < 2e-2, l
    finally:
        s.eng.release(out.linked)


class prefill_kernel_decode:
    """Decode steps through the prefill attention kernel (PIC_NO_ATTN_DECODE=1): a cache that still
    re-bases keys on load always decodes there, so bit-identity against a copy-path cache is a property
    of that one kernel (the transposed decode kernel, attention_decode.cu, serves caches without Δ)."""

    def __enter__(self):
        os.environ["PIC_NO_ATTN_DECODE"] = "1"

    def __exit__(self, *exc):
        os.environ.pop("PIC_NO_ATTN_DECODE", None)


def test_shared_decode_bit_identical(setup):
    s = setup
    segs = s.w.requests[0]
    hs = [s.eng.link(s.segs(segs), "legolink:4", keep_linked=True, kv_share=share).linked for share in (False, True)]
    try:
        toks = [5, 17, 99, 3, 250, 7, 11, 13, 2, 1, 0, 8, 9, 10, 12, 14, 15, 16, 18, 19]
        for t in toks:  # crosses a block boundary (N = 112 -> 132)
            with prefill_kernel_decode():
                a = s.eng.decode([hs[0]], [t])
                b = s.eng.decode([hs[1]], [t])
            assert np.array_equal(a.logits, b.logits)
        for l in range(s.cfg.n_layers):
            ka, va = s.eng.linked_export(hs[0], l)
            kb, vb = s.eng.linked_export(hs[1], l)
            assert np.array_equal(ka, kb) and np.array_equal(va, vb)
    finally:
        for h in hs:
            s.eng.release(h)


def test_shared_blocks_survive_expiry():
    """Expire a chunk while a linked cache shares its blocks: the rows stay (reference counted) and
    return to the pool only when the linked cache is released (S:467 in-flight snapshot)."""
    s = Setup(sg.TINY_D128)
    try:
        segs = s.w.requests[0]
        out = s.eng.link(s.segs(segs), "naive", keep_linked=True, kv_share=True)
        n_shared, _ = s.eng.linked_sharing(out.linked)
        assert n_shared > 0
        before = [s.eng.linked_export(out.linked, l) for l in range(s.cfg.n_layers)]
        free0 = s.eng.stats()["free_blocks"]
        for cid in s.eids:
            assert s.eng.expire(cid)
        freed = s.eng.stats()["free_blocks"] - free0
        total_chunk_blocks = sum((len(c) + 15) // 16 for c in s.w.chunks)
        assert freed == total_chunk_blocks - n_shared          # shared blocks are still held
        # new compiles reuse only the freed blocks; the linked cache is untouched
        s.eng.generate_context_cache([np.full(64, 7, np.int32)])
        after = [s.eng.linked_export(out.linked, l) for l in range(s.cfg.n_layers)]
        for (ka, va), (kb, vb) in zip(before, after):
            assert np.array_equal(ka, kb) and np.array_equal(va, vb)
        free1 = s.eng.stats()["free_blocks"]
        s.eng.release(out.linked)
        assert s.eng.stats()["free_blocks"] == free1 + (out.n_tokens + 15) // 16
    finally:
        s.eng.close()


def test_shared_legolink0_negative_delta():
    """LegoLink-0 links dummy-prefix chunks with Δ = s_c − m (negative for the first chunk):
    the shared path rotates by negative Δ exactly like the copy path."""
    s = Setup(sg.TINY_D128, dummy_prefix=4)
    try:
        for segs in [s.w.requests[0]] + sg.permuted_requests(s.w, 3):
            copy, shared = link_both(s, segs, "legolink0")
            try:
                assert_identical(copy, shared)
                if not segs[0].cached:
                    continue
                assert shared[3] > 0 and (shared[4] < 0).any()
            finally:
                s.eng.release(copy[0].linked)
                s.eng.release(shared[0].linked)
    finally:
        s.eng.close()


def test_shared_link_fp32_debug_bit_identical():
    s = Setup(replace(sg.TINY_D128, dtype=1))
    try:
        for alg in ("naive", "legolink:4"):
            copy, shared = link_both(s, s.w.requests[0], alg)
            try:
                assert_identical(copy, shared)
                assert shared[3] > 0
            finally:
                s.eng.release(copy[0].linked)
                s.eng.release(shared[0].linked)
    finally:
        s.eng.close()


def test_materialize_bit_identical_and_accounting(setup):
    """pic_linked_materialize copies + re-bases the shared blocks with Δ != 0 into owned blocks: exports
    and later decode steps are bit-identical to the copy path, the handle no longer needs the K-tile
    rotation (bdelta all zero), and the chunk-store blocks lose its references."""
    s = setup
    segs = s.w.requests[0]
    hc = s.eng.link(s.segs(segs), "legolink:4", keep_linked=True, kv_share=False).linked
    hs = s.eng.link(s.segs(segs), "legolink:4", keep_linked=True, kv_share=True).linked
    try:
        n_shared0, bd0 = s.eng.linked_sharing(hs)
        n_rot = int((bd0 != 0).sum())
        assert n_rot > 0
        free0 = s.eng.stats()["free_blocks"]
        s.eng.materialize(hs)
        n_shared1, bd1 = s.eng.linked_sharing(hs)
        assert n_shared1 == n_shared0 - n_rot and not bd1.any()
        assert s.eng.stats()["free_blocks"] == free0 - n_rot      # fresh owned blocks; store blocks still cached
        for l in range(s.cfg.n_layers):
            kc, vc = s.eng.linked_export(hc, l)
            ks, vs = s.eng.linked_export(hs, l)
            assert np.array_equal(kc, ks) and np.array_equal(vc, vs), l
        for t in (5, 17, 99, 3, 250):
            a = s.eng.decode([hc], [t])
            b = s.eng.decode([hs], [t])
            assert np.array_equal(a.logits, b.logits)
        s.eng.materialize(hs)                                    # idempotent: nothing left to re-base
        assert s.eng.linked_sharing(hs)[0] == n_shared1
    finally:
        s.eng.release(hc)
        s.eng.release(hs)


def test_chunkframe_materialize_accounting(setup):
    """kv_share 3 + materialize: every block with a frame Δ (store blocks linked by reference and owned
    chunk-frame blocks) is re-based into a fresh owned block; n_shared drops by the by-reference ones only,
    the owned frame blocks return to the pool, exports are unchanged bit for bit, and decode over the
    materialized handle equals decode over an identical un-materialized one bit for bit (the decode
    attention re-bases K tiles with a2's arithmetic)."""
    s = setup
    segs = s.w.requests[0]
    ha = s.eng.link(s.segs(segs), "legolink:4", keep_linked=True, kv_share=3).linked
    hb = s.eng.link(s.segs(segs), "legolink:4", keep_linked=True, kv_share=3).linked
    try:
        n_shared0, bd0 = s.eng.linked_sharing(hb)
        n_rot = int((bd0 != 0).sum())
        assert n_rot > 0 and n_shared0 > 0
        exp0 = [s.eng.linked_export(hb, l) for l in range(s.cfg.n_layers)]
        free0 = s.eng.stats()["free_blocks"]
        s.eng.materialize(hb)
        n_shared1, bd1 = s.eng.linked_sharing(hb)
        assert not bd1.any() and n_shared1 >= 0
        n_byref_rot = n_shared0 - n_shared1
        n_owned_rot = n_rot - n_byref_rot
        assert n_owned_rot > 0                                    # owned frame blocks carried Δ too
        assert s.eng.stats()["free_blocks"] == free0 - n_rot + n_owned_rot
        for l in range(s.cfg.n_layers):
            k, v = s.eng.linked_export(hb, l)
            assert np.array_equal(k, exp0[l][0]) and np.array_equal(v, exp0[l][1]), l
        for t in (5, 17, 99):
            with prefill_kernel_decode():
                a = s.eng.decode([ha], [t])
                b = s.eng.decode([hb], [t])
            assert np.array_equal(a.logits, b.logits)
        c = s.eng.decode([hb], [7])                               # materialized: the decode kernel may serve it
        with prefill_kernel_decode():
            d = s.eng.decode([ha], [7])
        assert rel(c.logits, d.logits) < 2e-2
    finally:
        s.eng.release(ha)
        s.eng.release(hb)


def test_shared_batch_same_chunks_refcounts(setup):
    """A batched shared-block link whose requests reuse the same chunks (the cfg4 pattern): every request
    is bit-identical to its own copy-path link, the store blocks carry one reference per request, and
    releasing everything restores the pool exactly."""
    s = setup
    reqs = [s.w.requests[0]] + sg.permuted_requests(s.w, 2)
    free0 = s.eng.stats()["free_blocks"]
    outs = s.eng.link_batch([s.segs(r) for r in reqs], "legolink:4", keep_linked=True, kv_share=True)
    try:
        for r, o in zip(reqs, outs):
            ref = s.eng.link(s.segs(r), "legolink:4", keep_linked=True, kv_share=False)
            try:
                assert np.array_equal(o.logits, ref.logits)
                for l in range(s.cfg.n_layers):
                    ka, va = s.eng.linked_export(o.linked, l)
                    kb, vb = s.eng.linked_export(ref.linked, l)
                    assert np.array_equal(ka, kb) and np.array_equal(va, vb), l
            finally:
                s.eng.release(ref.linked)
        # the requests' block tables point at the chunk-store blocks themselves
        shared_ids = set()
        for o in outs:
            n, bd = s.eng.linked_sharing(o.linked)
            bt = s.eng.linked_blocks(o.linked)
            shared_ids |= {int(b) for b in bt[:len(bd)]} & {int(b) for c in s.eids for b in s.eng.cache_blocks(c)}
        assert shared_ids
    finally:
        for o in outs:
            s.eng.release(o.linked)
    assert s.eng.stats()["free_blocks"] == free0


def test_shared_link_without_rebase_bit_identical(setup):
    """SPEC's no-re-base reading (rebase = 0, reading R1): shared blocks then carry Δ = 0 and the result
    equals the copy path's (cached keys left at their compile positions) bit for bit."""
    s = setup
    any_shared = 0
    for segs in [s.w.requests[0]] + sg.permuted_requests(s.w, 2):
        copy, shared = link_both(s, segs, "legolink:4", rebase=False)
        try:
            assert_identical(copy, shared)
            assert not shared[4].any()          # nothing to rotate
            any_shared += shared[3]
        finally:
            s.eng.release(copy[0].linked)
            s.eng.release(shared[0].linked)
    assert any_shared > 0                       # the planner did link blocks by reference
