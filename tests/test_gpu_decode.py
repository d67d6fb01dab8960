"""Decode over the linked cache on the GPU path: steps after a
link, against the oracle's decode (bf16 2e-2, fp32 debug 1e-4), batched = single bit-exactly, block
growth across 16-token boundaries, error contract."""
from dataclasses import replace

import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
STEPS = 20


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
    eng = B.Engine(cfg, num_blocks=512, max_rows=1024, max_tokens=2048, max_requests=4, device=0)
    eids = eng.generate_context_cache(w.chunks)
    Wt = M.Weights(base)
    store = P.Store(Wt)
    oids = store.compile(w.chunks)
    yield cfg, w, eng, Wt, store, eids, oids, tol
    eng.close()


def segs_for(segs, ids):
    return [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in segs]


@pytest.mark.parametrize("alg", ["legolink:4", "naive", "fr", "cacheblend:15", "legolink0"])
def test_decode_steps_match_oracle(env, alg):
    cfg, w, eng, Wt, store, eids, oids, tol = env
    if alg == "legolink0":                                   # chunks compiled behind 4 dummies (f2)
        eids = eng.generate_context_cache(w.chunks, dummy_prefix=4)
        store = P.Store(Wt)
        oids = store.compile(w.chunks, dummy_prefix=4)
    out = eng.link(segs_for(w.requests[0], eids), alg, keep_linked=True, want_selected=True)
    # CacheBlend: the oracle continues from the GPU's own device-side selection (near-threshold swaps
    # are a selection question, pinned separately; SURVEY §8(c).8 protocol (ii))
    ref = P.link(store, segs_for(w.requests[0], oids), alg,
                 sel_override=out.selected if alg.startswith("cacheblend") else None)
    K, V = ref.K, ref.V
    toks = sg.tokens(0xDEC0DE, 7, STEPS, cfg.vocab, None)
    N0 = out.n_tokens
    for i, t in enumerate(toks):
        d = eng.decode([out.linked], [int(t)])
        lg, K, V = P.decode(Wt, K, V, int(t))
        assert d.n_tokens[0] == N0 + i + 1
        assert rel(d.logits[0], lg) < tol, (i, rel(d.logits[0], lg))
        assert d.next_token[0] == int(np.argmax(d.logits[0]))
    for l in range(cfg.n_layers):
        k, v = eng.linked_export(out.linked, l)
        assert k.shape[0] == N0 + STEPS
        assert rel(f64(k), K[l]) < tol and rel(f64(v), V[l]) < tol, l
    eng.release(out.linked)


def test_batched_decode_equals_single_and_greedy(env):
    cfg, w, eng, Wt, store, eids, oids, tol = env
    reqs = [w.requests[0]] + sg.permuted_requests(w, 1)
    a = [eng.link(segs_for(r, eids), "legolink:4", keep_linked=True) for r in reqs]
    b = [eng.link(segs_for(r, eids), "legolink:4", keep_linked=True) for r in reqs]
    ta = [x.first_token for x in a]
    for step in range(18):                                   # crosses a 16-token block boundary
        batch = eng.decode([x.linked for x in a], ta)
        singles = [eng.decode([x.linked], [t]) for x, t in zip(b, ta)]
        for j in range(len(a)):
            assert np.array_equal(batch.logits[j], singles[j].logits[0]), (step, j)
        ta = [int(t) for t in batch.next_token]              # greedy
    for x, y in zip(a, b):
        for l in (0, cfg.n_layers - 1):
            ka, va = eng.linked_export(x.linked, l)
            kb, vb = eng.linked_export(y.linked, l)
            assert np.array_equal(ka, kb) and np.array_equal(va, vb)
        eng.release(x.linked)
        eng.release(y.linked)


def test_decode_errors(env):
    cfg, w, eng, Wt, store, eids, oids, tol = env
    out = eng.link(segs_for(w.requests[0], eids), "naive", keep_linked=True)
    with pytest.raises(B.PicError) as e:
        eng.decode([out.linked, out.linked], [1, 2])
    assert e.value.name == "PIC_E_INVALID_ARG"
    with pytest.raises(B.PicError) as e:
        eng.decode([out.linked], [cfg.vocab])
    assert e.value.name == "PIC_E_TOKEN"
    k, _ = eng.linked_export(out.linked, 0)
    assert k.shape[0] == out.n_tokens                         # failed calls changed nothing
    eng.release(out.linked)
