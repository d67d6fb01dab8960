"""LegoLink-0 on the GPU path: dummy-prefix compile (a0 variant) and
the zero-recompute link, against the oracle — bf16 build at 2e-2, fp32 debug build at 1e-4."""
from dataclasses import replace

import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
DUMMY = 4


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def f64(x):
    return B.bf16_bits_to_f32(x).astype(np.float64) if x.dtype == np.uint16 else x.astype(np.float64)


@pytest.fixture(scope="module", params=[(sg.TINY, 0), (sg.TINY_GQA, 0), (sg.TINY_D128, 0), (sg.TINY_D128, 1)],
                ids=lambda p: f"{p[0].name}-{'fp32' if p[1] else 'bf16'}")
def env(request):
    base, dt = request.param
    cfg = replace(base, dtype=dt)
    tol = 1e-4 if dt else 2e-2
    w = sg.cfg1(model=base)
    eng = B.Engine(cfg, num_blocks=512, max_rows=1024, max_tokens=2048, device=0)
    eids = eng.generate_context_cache(w.chunks, dummy_prefix=DUMMY)
    plain = eng.generate_context_cache(w.chunks[:1])
    store = P.Store(M.Weights(base))
    oids = store.compile(w.chunks, dummy_prefix=DUMMY)
    yield cfg, w, eng, store, eids, oids, plain, tol
    eng.close()


def test_dummy_prefix_compile_matches_oracle(env):
    cfg, w, eng, store, eids, oids, plain, tol = env
    for eid, oid in zip(eids, oids):
        for l in range(cfg.n_layers):
            k, v = eng.cache_export(eid, l)
            assert rel(f64(k), store.chunks[oid].K[l]) < tol and rel(f64(v), store.chunks[oid].V[l]) < tol, l


def test_legolink0_link_matches_oracle(env):
    cfg, w, eng, store, eids, oids, plain, tol = env
    for segs in [w.requests[0]] + sg.permuted_requests(w, 2):
        g = [("cached", eids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]
        o = [("cached", oids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]
        out = eng.link(g, "legolink0", keep_linked=True, want_selected=True)
        ref = P.link(store, o, "legolink0")
        assert np.array_equal(out.selected, ref.plan.sel)
        assert rel(out.logits, ref.logits) < tol
        for l in range(cfg.n_layers):
            k, v = eng.linked_export(out.linked, l)
            assert rel(f64(k), ref.K[l]) < tol and rel(f64(v), ref.V[l]) < tol, l
        eng.release(out.linked)


def test_legolink0_variant_error_and_distinct_from_naive(env):
    cfg, w, eng, store, eids, oids, plain, tol = env
    with pytest.raises(B.PicError) as e:
        eng.link([("cached", plain[0]), ("cached", eids[1])], "legolink0")
    assert e.value.name == "PIC_E_VARIANT"
    g = [("cached", eids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
    gp = eng.generate_context_cache(w.chunks)
    gn = [("cached", gp[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
    a = eng.link(g, "legolink0").logits
    b = eng.link(gn, "naive").logits
    assert rel(a, b.astype(np.float64)) > 5 * tol                      # the dummies change the result
    for c in gp:
        eng.expire(c)
