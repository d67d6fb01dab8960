"""End-to-end parity of the linked-prefill path (compile + link through the C ABI) against the
fp64 oracle on the same seeded inputs (SURVEY §8(c).8 protocol).

Tolerances: bf16 build — hidden state of the selected rows after every layer, linked K/V per
layer and logits each within 2e-2 relative L2 (BASELINE north_star).  Indexing is bit-exact:
selected sets, block tables, V rows of unselected cached tokens and K rows with Δ = 0 are
compared bit for bit against the GPU's own compiled store."""
import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
TOL = 2e-2


def f32(bits):
    return B.bf16_bits_to_f32(bits).astype(np.float64)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def check_first_token(gpu_tok, logits_gpu, ref_logits):
    top = np.argsort(-ref_logits)[:2]
    gap = ref_logits[top[0]] - ref_logits[top[1]]
    err = np.abs(logits_gpu - ref_logits).max()
    if gap > 4 * err:
        assert gpu_tok == top[0]
    else:
        assert gpu_tok in top


class Setup:
    def __init__(self, cfg, w, max_rows=1024, blocks=512):
        self.cfg, self.w = cfg, w
        self.eng = B.Engine(cfg, num_blocks=blocks, max_rows=max_rows, max_tokens=4096, max_requests=4, device=0)
        self.eids = self.eng.generate_context_cache(w.chunks)
        self.store = P.Store(M.Weights(cfg))
        self.oids = self.store.compile(w.chunks)

    def segs(self, segs, which):
        ids = self.eids if which == "gpu" else self.oids
        return [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]


@pytest.fixture(scope="module", params=[sg.TINY, sg.TINY_GQA, sg.TINY_D128], ids=lambda c: c.name)
def setup(request):
    s = Setup(request.param, sg.cfg1(model=request.param))
    yield s
    s.eng.close()


def test_compile_matches_oracle(setup):
    s = setup
    for c, (eid, oid) in enumerate(zip(s.eids, s.oids)):
        for l in range(s.cfg.n_layers):
            k, v = s.eng.cache_export(eid, l)
            ch = s.store.chunks[oid]
            assert rel(f32(k), ch.K[l]) < TOL, (c, l)
            assert rel(f32(v), ch.V[l]) < TOL, (c, l)


@pytest.mark.parametrize("alg", ["naive", "fr", "legolink:4", "legolink:0", "legolink:32", "cacheblend:15"])
def test_link_parity_canonical(setup, alg):
    s = setup
    if alg.startswith("cacheblend") and s.cfg.head_dim != 128:
        pytest.skip("CacheBlend runs on the tcgen05 attention path (head_dim 128)")
    segs = s.w.requests[0]
    out = s.eng.link(s.segs(segs, "gpu"), alg, keep_linked=True, debug_hidden=True, want_selected=True)
    try:
        if alg.startswith("cacheblend"):
            ref0 = P.link(s.store, s.segs(segs, "oracle"), alg)
            gsel = out.selected
            osel = ref0.sel_per_layer[-1]
            assert len(gsel) == len(osel)
            # protocol (i): differences only among near-threshold deviations
            diff = set(gsel.tolist()) ^ set(osel.tolist())
            if diff:
                dev = ref0.dev
                T = P.cacheblend_count(ref0.plan)
                cand = sorted([i for i in range(ref0.plan.N) if dev[i] >= 0 and i not in set(ref0.plan.dynamic)
                               and i != ref0.plan.N - 1], key=lambda i: (-dev[i], i))
                thr = dev[cand[T - 1]]
                for i in diff:
                    assert abs(dev[i] - thr) <= 0.05 * thr, (i, dev[i], thr)
            # protocol (ii): oracle re-run with the GPU's selection
            ref = P.link(s.store, s.segs(segs, "oracle"), alg, sel_override=gsel)
        else:
            ref = P.link(s.store, s.segs(segs, "oracle"), alg)
            assert np.array_equal(out.selected, ref.sel_per_layer[-1])
        assert out.n_tokens == ref.plan.N
        assert out.n_selected == len(ref.sel_per_layer[-1])
        assert rel(out.logits, ref.logits) < TOL
        check_first_token(out.first_token, out.logits, ref.logits)
        for l in range(s.cfg.n_layers):
            k, v = s.eng.linked_export(out.linked, l)
            assert rel(f32(k), ref.K[l]) < TOL, l
            assert rel(f32(v), ref.V[l]) < TOL, l
            sel = ref.sel_per_layer[l]
            assert rel(out.hidden[l, :len(sel)], ref.hidden[l]) < TOL, l
        # bit-exact: unselected cached rows are the GPU store's rows (V copied, K re-based; Δ=0 exact)
        sel_set = set(out.selected.tolist()) if not alg.startswith("cacheblend") else set()
        lo = 1 if alg.startswith("cacheblend") else 0
        for l in range(lo, s.cfg.n_layers):
            k, v = s.eng.linked_export(out.linked, l)
            for c, eid in enumerate(s.eids):
                ck, cv = s.eng.cache_export(eid, l)
                for j in range(32):
                    i = 32 * c + j
                    if i in sel_set or (alg.startswith("cacheblend") and i in set(out.selected.tolist())):
                        continue
                    assert np.array_equal(v[i], cv[j]), (l, i)
                    if c == 0:
                        assert np.array_equal(k[i], ck[j]), (l, i)
    finally:
        s.eng.release(out.linked)


def test_link_permutations_and_graph_reuse(setup):
    s = setup
    for segs in sg.permuted_requests(s.w, 6):
        ref = P.link(s.store, s.segs(segs, "oracle"), "legolink:4")
        a = s.eng.link(s.segs(segs, "gpu"), "legolink:4", use_graph=True)
        b = s.eng.link(s.segs(segs, "gpu"), "legolink:4", use_graph=True)   # graph replay
        c = s.eng.link(s.segs(segs, "gpu"), "legolink:4", use_graph=False)
        assert rel(a.logits, ref.logits) < TOL
        assert np.array_equal(a.logits, b.logits) and np.array_equal(a.logits, c.logits)   # deterministic
    assert s.eng.stats()["free_blocks"] == 512 - 6                          # linked blocks returned


def test_link_batch_matches_single(setup):
    s = setup
    reqs = [s.segs(r, "gpu") for r in sg.permuted_requests(s.w, 3)]
    outs = s.eng.link_batch(reqs, "legolink:4")
    for r, o in zip(reqs, outs):
        single = s.eng.link(r, "legolink:4")
        assert rel(o.logits, single.logits) < 1e-5
        assert o.first_token == single.first_token


def test_errors_on_device(setup):
    s = setup
    with pytest.raises(B.PicError) as e:
        s.eng.link([("cached", 12345)], "naive")
    assert e.value.name == "PIC_E_MISSING_CACHE"
    free = s.eng.stats()["free_blocks"]
    with pytest.raises(B.PicError):
        s.eng.link([("tokens", np.array([1, 2, 99999], np.int32))], "naive")
    assert s.eng.stats()["free_blocks"] == free


def test_expire_does_not_corrupt_live_linked_cache():
    cfg = sg.TINY_D128
    w = sg.cfg1(model=cfg)
    eng = B.Engine(cfg, num_blocks=256, max_rows=512, max_tokens=1024, device=0)
    ids = eng.generate_context_cache(w.chunks)
    segs = [("cached", i) for i in ids] + [("tokens", w.requests[0][-1].tokens)]
    out = eng.link(segs, "legolink:4", keep_linked=True)
    k0, v0 = eng.linked_export(out.linked, 1)
    assert eng.expire(ids[1])
    eng.generate_context_cache([w.chunks[2], w.chunks[0]])    # reuses the freed blocks
    k1, v1 = eng.linked_export(out.linked, 1)
    assert np.array_equal(k0, k1) and np.array_equal(v0, v1)
    eng.release(out.linked)
    eng.close()


@pytest.mark.parametrize("which", ["cfg2"])
def test_full_width_truncated_depth(which):
    """Mistral-7B / Llama-3.1-8B width at L = 2: compile + LegoLink link vs the oracle."""
    w = sg.cfg2(n_layers=2) if which == "cfg2" else sg.cfg3(n_layers=2)
    cfg = w.model
    eng = B.Engine(cfg, num_blocks=1024, max_rows=6144, max_tokens=6144, device=0)
    eids = eng.generate_context_cache(w.chunks)
    Wt = M.Weights(cfg)
    store = P.Store(Wt)
    # oracle compile of every chunk is the expensive part (fp64, full width): check two chunks
    for c in (0, len(w.chunks) - 1):
        _, K, V, _ = M.full_prefill(Wt, w.chunks[c])
        for l in range(2):
            k, v = eng.cache_export(eids[c], l)
            assert rel(f32(k), K[l]) < TOL and rel(f32(v), V[l]) < TOL
    # link on identical compiled inputs (the GPU's own chunks)
    over = []
    for eid in eids:
        ks, vs = zip(*[eng.cache_export(eid, l) for l in range(2)])
        over.append((np.stack([f32(k) for k in ks]), np.stack([f32(v) for v in vs])))
    oids = store.compile(w.chunks, compiled_override=over)
    segs = w.requests[0]
    gs = [("cached", eids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]
    os_ = [("cached", oids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]
    out = eng.link(gs, w.alg, keep_linked=True, debug_hidden=True)
    ref = P.link(store, os_, w.alg)
    assert rel(out.logits, ref.logits) < TOL
    for l in range(2):
        k, v = eng.linked_export(out.linked, l)
        assert rel(f32(k), ref.K[l]) < TOL and rel(f32(v), ref.V[l]) < TOL
        assert rel(out.hidden[l, :len(ref.sel_per_layer[l])], ref.hidden[l]) < TOL
    eng.release(out.linked)
    eng.close()


def test_link_batch_logits_into_caller_buffers():
    """pic_link_batch fills caller-owned logits buffers: a page-locked [n][vocab] array (one direct
    device-to-host copy), a pageable one, and the default allocation all give the same logits and first tokens."""
    import torch
    cfg = sg.TINY_D128
    w = sg.cfg1(model=cfg)
    eng = B.Engine(cfg, num_blocks=256, max_rows=512, max_tokens=1024, max_requests=4, device=0)
    try:
        ids = eng.generate_context_cache(w.chunks)
        reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r]
                for r in [w.requests[0]] + sg.permuted_requests(w, 2)]
        ref = eng.link_batch(reqs, "legolink:4")
        pinned = torch.empty((len(reqs), cfg.vocab), dtype=torch.float32, pin_memory=True).numpy()
        pageable = np.empty((len(reqs), cfg.vocab), dtype=np.float32)
        for buf in (pinned, pageable):
            buf[:] = np.nan
            out = eng.link_batch(reqs, "legolink:4", logits_out=buf)
            for a, b in zip(ref, out):
                assert np.array_equal(a.logits, b.logits) and a.first_token == b.first_token
            assert np.array_equal(buf, np.stack([a.logits for a in ref]))
        with pytest.raises(ValueError):
            eng.link_batch(reqs, "legolink:4", logits_out=np.empty((1, cfg.vocab), np.float32))
    finally:
        eng.close()
