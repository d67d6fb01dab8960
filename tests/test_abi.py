"""C-ABI library: loads on a CPU-only host, exports every symbol include/*.h declares, and its
host-only planner / allocator / store bookkeeping agrees bit-exactly with the oracle's model."""
import os
import re

import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("pic.h", "pic_test.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names.update(re.findall(r"\b(pic_[a-z_0-9]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    L = B.lib()
    decl = declared_symbols()
    assert len(decl) >= 19
    for n in decl:
        assert hasattr(L, n), n
    assert set(B.EXPORTS) == decl


def test_status_strings():
    L = B.lib()
    assert L.pic_status_string(0) == b"PIC_OK"
    assert L.pic_status_string(5) == b"PIC_E_MISSING_CACHE"


def test_arena_bytes_and_config_errors():
    import ctypes as C
    L = B.lib()
    cfg = B.config_struct(sg.TINY)
    lim = B.LimitsC(64, 256, 512, 2)
    n = C.c_size_t()
    assert L.pic_arena_bytes(C.byref(cfg), C.byref(lim), C.byref(n)) == 0 and n.value > 0
    bad = B.config_struct(sg.TINY)
    bad.n_kv_heads = 3
    assert L.pic_arena_bytes(C.byref(bad), C.byref(lim), C.byref(n)) == 2        # PIC_E_CONFIG
    bad = B.config_struct(sg.TINY)
    bad.head_dim = 24
    assert L.pic_arena_bytes(C.byref(bad), C.byref(lim), C.byref(n)) == 2


def host_engine(cfg=sg.TINY, blocks=256, max_tokens=1024):
    return B.Engine(cfg, num_blocks=blocks, max_rows=512, max_tokens=max_tokens, max_requests=4, device=None)


def oracle_store(cfg, chunks):
    st = P.Store(M.Weights(cfg))
    ids = st.compile(chunks, compiled_override=[(None, None)] * len(chunks))
    return st, ids


def to_engine_segs(segs, ids):
    return [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]


def test_planner_bit_exact_vs_oracle_cfg1_and_permutations():
    w = sg.cfg1()
    eng = host_engine()
    eids = eng.generate_context_cache(w.chunks)
    st, oids = oracle_store(sg.TINY, w.chunks)
    assert eids == oids == [1, 2, 3]                      # ids monotone from 1
    alloc = P.BlockAllocator(256)
    chunk_blocks = [alloc.alloc(P.n_blocks(len(c))) for c in w.chunks]
    for i, cid in enumerate(eids):
        assert eng.cache_blocks(cid).tolist() == chunk_blocks[i]
    reqs = [w.requests[0]] + sg.permuted_requests(w, 100)
    for segs in reqs:
        for alg in ("naive", "fr", "legolink:4", "legolink:0", "legolink:40", "cacheblend:15"):
            pe = eng.plan(to_engine_segs(segs, eids), alg)
            po = P.plan(st, to_engine_segs(segs, oids), alg)
            assert pe["n_tokens"] == po.N
            assert np.array_equal(pe["sel"], po.sel), (alg, segs)
            assert np.array_equal(pe["tok"], po.tokens)
            assert np.array_equal(pe["src"], po.src)
            assert pe["chunks"].tolist() == [[s, n, dl] for _, s, n, dl in po.chunks]
            bt = alloc.peek(P.n_blocks(po.N)) if hasattr(alloc, "peek") else sorted(alloc.free)[:P.n_blocks(po.N)]
            assert pe["block_table"].tolist() == bt
            assert np.array_equal(pe["slot"], P.slot_map(bt, po.sel))


def test_plan_errors_and_expiry():
    w = sg.cfg1()
    eng = host_engine()
    ids = eng.generate_context_cache(w.chunks)
    with pytest.raises(B.PicError) as e:
        eng.plan([("cached", 99)], "naive")
    assert e.value.name == "PIC_E_MISSING_CACHE"
    with pytest.raises(B.PicError) as e:
        eng.plan([], "naive")
    assert e.value.name == "PIC_E_EMPTY_INPUT"
    with pytest.raises(B.PicError) as e:
        eng.plan([("tokens", np.array([], dtype=np.int32))], "naive")
    assert e.value.name == "PIC_E_EMPTY_INPUT"
    with pytest.raises(B.PicError) as e:
        eng.plan([("tokens", np.array([300], dtype=np.int32))], "naive")
    assert e.value.name == "PIC_E_TOKEN"
    with pytest.raises(B.PicError) as e:
        eng.plan([("tokens", np.zeros(2000, dtype=np.int32))], "naive")
    assert e.value.name == "PIC_E_CAPACITY"
    with pytest.raises(ValueError):
        eng.plan([("cached", ids[0])], "bogus")
    # expiry is idempotent; ids are never reused; freed blocks return to the pool
    free0 = eng.stats()["free_blocks"]
    assert eng.expire(ids[1]) is True
    assert eng.expire(ids[1]) is False
    assert eng.stats()["free_blocks"] == free0 + 2
    with pytest.raises(B.PicError) as e:
        eng.plan([("cached", ids[1])], "naive")
    assert e.value.name == "PIC_E_MISSING_CACHE"
    new = eng.generate_context_cache([w.chunks[1]])
    assert new == [4]
    assert eng.cache_blocks(4).tolist() == [2, 3]          # lowest free ids reused
    # host-only engines refuse compute
    with pytest.raises(B.PicError) as e:
        eng.link([("cached", ids[0])], "naive")
    assert e.value.name == "PIC_E_NO_DEVICE"


def test_compile_all_or_nothing():
    eng = host_engine(blocks=4)
    with pytest.raises(B.PicError) as e:
        eng.generate_context_cache([np.ones(32, np.int32), np.array([], np.int32)])
    assert e.value.name == "PIC_E_EMPTY_INPUT" and e.value.err_index == 1
    with pytest.raises(B.PicError) as e:
        eng.generate_context_cache([np.ones(48, np.int32), np.ones(48, np.int32)])   # 6 blocks > 4
    assert e.value.name == "PIC_E_CAPACITY"
    assert eng.stats()["free_blocks"] == 4 and eng.stats()["n_cached_chunks"] == 0
    assert eng.generate_context_cache([np.ones(48, np.int32)]) == [1]


def test_block_allocator_model_sequence():
    """A seeded sequence of compile / expire operations: engine block lists == oracle model."""
    eng = host_engine(blocks=64)
    alloc = P.BlockAllocator(64)
    live = {}
    u = sg.U(42, 1, np.arange(200, dtype=np.uint64))
    for step in range(60):
        op = int(u[step] % np.uint64(3))
        if op < 2 or not live:
            n = 1 + int(u[step + 100] % np.uint64(60))
            if not alloc.free or len(alloc.free) < P.n_blocks(n):
                continue
            cid = eng.generate_context_cache([np.ones(n, np.int32)])[0]
            live[cid] = alloc.alloc(P.n_blocks(n))
            assert eng.cache_blocks(cid).tolist() == live[cid]
        else:
            cid = sorted(live)[int(u[step + 50] % np.uint64(len(live)))]
            assert eng.expire(cid)
            alloc.release(live.pop(cid))
    assert eng.stats()["free_blocks"] == len(alloc.free)


def test_legolink0_planner_and_variant_error():
    """Dummy-prefix compile on a host-only engine: same blocks as a plain compile (the scratch blocks
    are returned), Δ = s_c − m in the plan, and LegoLink-0 over a plain chunk is PIC_E_VARIANT."""
    w = sg.cfg1()
    eng = host_engine()
    eids = eng.generate_context_cache(w.chunks, dummy_prefix=4)
    st = P.Store(M.Weights(sg.TINY))
    oids = st.compile(w.chunks, compiled_override=[(None, None)] * len(w.chunks), dummy_prefix=4)
    assert eng.stats()["free_blocks"] == 256 - sum(P.n_blocks(len(c)) for c in w.chunks)
    for segs in [w.requests[0]] + sg.permuted_requests(w, 20):
        pe = eng.plan(to_engine_segs(segs, eids), "legolink0")
        po = P.plan(st, to_engine_segs(segs, oids), "legolink0")
        assert np.array_equal(pe["sel"], po.sel)
        assert pe["chunks"].tolist() == [[s, n, dl] for _, s, n, dl in po.chunks]
    plain = eng.generate_context_cache([w.chunks[0]])
    with pytest.raises(B.PicError) as e:
        eng.plan([("cached", plain[0]), ("cached", eids[1])], "legolink0")
    assert e.value.name == "PIC_E_VARIANT"


def test_shared_block_plan_bit_exact_vs_oracle():
    """f3 shared-block link (kv_share): the planner's block table / per-block Δ equal the oracle's
    layout model (share_blocks + lowest-free-first fresh blocks) on cfg1 and 100 permutations
    (dynamic-first, interleaved, repeated ids), for every algorithm; CacheBlend and FR share nothing."""
    w = sg.cfg1()
    eng = host_engine()
    eids = eng.generate_context_cache(w.chunks)
    st, oids = oracle_store(sg.TINY, w.chunks)
    alloc = P.BlockAllocator(256)
    chunk_blocks = {oid: alloc.alloc(P.n_blocks(len(c))) for oid, c in zip(oids, w.chunks)}
    n_shared_total = 0
    for segs in [w.requests[0]] + sg.permuted_requests(w, 100):
        for alg in ("naive", "fr", "legolink:4", "legolink:16", "legolink:40", "cacheblend:15"):
            pe = eng.plan(to_engine_segs(segs, eids), alg, kv_share=True)
            po = P.plan(st, to_engine_segs(segs, oids), alg)
            shared, delta = P.share_blocks(po, chunk_blocks)
            n_fresh = sum(b < 0 for b in shared)
            fresh = iter(alloc.peek(n_fresh))
            bt = [b if b >= 0 else next(fresh) for b in shared]
            assert pe["block_table"].tolist() == bt, (alg, segs)
            assert pe["block_delta"].tolist() == delta
            assert pe["n_shared"] == len(shared) - n_fresh
            assert np.array_equal(pe["slot"], P.slot_map(bt, po.sel))
            if alg in ("fr", "cacheblend:15"):
                assert pe["n_shared"] == 0
            n_shared_total += pe["n_shared"]
            # without kv_share the plan is the copy layout
            assert eng.plan(to_engine_segs(segs, eids), alg)["n_shared"] == 0
    assert n_shared_total > 0


def test_shared_block_plan_alignment_rules():
    """A chunk placed at a 16-misaligned start shares nothing; a chunk's partial last block is never
    shared; Naive shares every full block of an aligned chunk with Δ = s_c (0 for the index-0 chunk)."""
    eng = host_engine()
    ids = eng.generate_context_cache([np.ones(40, np.int32), np.ones(32, np.int32)])
    blocks = [eng.cache_blocks(i).tolist() for i in ids]
    # [C0 (40 rows: 2 full blocks + 8), C1 at 40 (misaligned), 5 dynamic]
    pe = eng.plan([("cached", ids[0]), ("cached", ids[1]), ("tokens", np.ones(5, np.int32))], "naive",
                  kv_share=True)
    assert pe["block_table"][:2].tolist() == blocks[0][:2] and pe["block_delta"].tolist()[:2] == [0, 0]
    assert pe["n_shared"] == 2
    # [16 dynamic, C1 at 16 (aligned), C0 at 48 (aligned), query]
    pe = eng.plan([("tokens", np.ones(16, np.int32)), ("cached", ids[1]), ("cached", ids[0]),
                   ("tokens", np.ones(3, np.int32))], "naive", kv_share=True)
    assert pe["block_table"][1:3].tolist() == blocks[1] and pe["block_delta"][1:3].tolist() == [16, 16]
    assert pe["block_table"][3:5].tolist() == blocks[0][:2] and pe["block_delta"][3:5].tolist() == [48, 48]
    assert pe["n_shared"] == 4
    # LegoLink-16 recomputes the first block of each non-initial chunk
    pe = eng.plan([("tokens", np.ones(16, np.int32)), ("cached", ids[1]), ("cached", ids[0]),
                   ("tokens", np.ones(3, np.int32))], "legolink:16", kv_share=True)
    assert pe["block_delta"].tolist() == [0, 0, 16, 0, 48, 0]
    assert pe["n_shared"] == 2
