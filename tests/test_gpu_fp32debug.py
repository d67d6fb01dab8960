"""The fp32 debug build (pic_model_config.dtype = 1, BASELINE north star: <= 1e-4): fp32 activations,
Q/K/V, paged KV pools and P/O, CUDA-core projections with exact bf16-weight products.  Every output
(logits, linked K/V of every layer, hidden state of the selected rows after every layer) must be within
1e-4 relative L2 of the fp64 oracle, and CacheBlend's device-side selection must equal the oracle's
exactly — at this precision the algorithms are separated far beyond the tolerance."""
from dataclasses import replace

import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", params=[sg.TINY, sg.TINY_GQA, sg.TINY_D128], ids=lambda c: c.name)
def env(request):
    cfg = replace(request.param, dtype=1)
    w = sg.cfg1(model=request.param)
    eng = B.Engine(cfg, num_blocks=512, max_rows=1024, max_tokens=2048, device=0)
    eids = eng.generate_context_cache(w.chunks)
    store = P.Store(M.Weights(request.param))
    oids = store.compile(w.chunks)
    yield cfg, w, eng, store, eids, oids
    eng.close()


def test_compile_fp32(env):
    cfg, w, eng, store, eids, oids = env
    for eid, oid in zip(eids, oids):
        for l in range(cfg.n_layers):
            k, v = eng.cache_export(eid, l)
            assert k.dtype == np.float32
            assert rel(k, store.chunks[oid].K[l]) < TOL and rel(v, store.chunks[oid].V[l]) < TOL


@pytest.mark.parametrize("alg", ["naive", "legolink:2", "legolink:4", "fr", "cacheblend:15"])
def test_link_fp32_within_1e4(env, alg):
    cfg, w, eng, store, eids, oids = env
    segs = w.requests[0]
    g = [("cached", eids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]
    o = [("cached", oids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]
    out = eng.link(g, alg, keep_linked=True, debug_hidden=True, want_selected=True)
    ref = P.link(store, o, alg)
    assert np.array_equal(out.selected, ref.sel_per_layer[-1])        # exact, CacheBlend included
    assert out.first_token == ref.first_token
    assert rel(out.logits, ref.logits) < TOL, rel(out.logits, ref.logits)
    for l in range(cfg.n_layers):
        k, v = eng.linked_export(out.linked, l)
        assert rel(k, ref.K[l]) < TOL and rel(v, ref.V[l]) < TOL, l
        assert rel(out.hidden[l, :len(ref.sel_per_layer[l])], ref.hidden[l]) < TOL, l
    eng.release(out.linked)


def test_fp32_separates_neighbouring_algorithms(env):
    """LegoLink-2 vs LegoLink-4 differ by far more than the fp32 tolerance (C13 discrimination)."""
    cfg, w, eng, store, eids, oids = env
    g = [("cached", eids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
    a = eng.link(g, "legolink:2").logits
    b = eng.link(g, "legolink:4").logits
    assert rel(a, b) > 100 * TOL
