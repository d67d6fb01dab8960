"""Parity at the bench's sizes and launch configuration (VERDICT r1 "close parity at bench sizes").

1. cfg2 END TO END, FULL DEPTH: the fp64 oracle links the same request through all 32 layers from its
   own state (§4.2: the layer-by-layer recomputation of Eq. (1)), starting only from
   the GPU's compiled chunks (compiled_override, SURVEY §8(c).8 "full-depth large configs") — no GPU
   hidden state is fed back.  Logits, the selected rows' hidden state after every layer and the linked
   K/V of every layer are held to the north star's 2e-2 relative L2; the first token follows §8(c).8.
2. cfg4 WAVE: one 32-request pic_link_batch with graphs and the shared-block link (exactly what
   bench.py times).  Graph and eager (debug) batches are bit-identical; for 4 requests spread over the
   wave the oracle recomputes layers 0 and L-1 on sampled rows from the GPU's layer input and linked
   K/V, re-bases their unselected cached keys, and applies the LM head to their last row.
3. cfg5 (Llama-3-70B shape, G = 8 query heads per kv-head, N = 32832) at truncated depth L = 2, full
   width, on sampled rows of both layers.
"""
import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
TOL = 2e-2          # north star: bf16 hidden states and logits, relative L2
LAYER_TOL = 5e-3    # one layer from identical inputs: bf16 GEMM/attention rounding only


def f64(bits):
    return B.bf16_bits_to_f32(bits).astype(np.float64)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def n_tok(w, r):
    return sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r)


def first_token_ok(gpu_logits, ref_logits):
    """the GPU argmax equals the oracle's when the oracle's top-1/top-2 gap exceeds 4x the
    measured logit error; otherwise either of the oracle's top two is accepted."""
    g = int(np.argmax(gpu_logits))
    top = np.argsort(-ref_logits)[:2]
    gap = ref_logits[top[0]] - ref_logits[top[1]]
    err = float(np.max(np.abs(gpu_logits - ref_logits)))
    return g == top[0] if gap > 4 * err else g in set(top.tolist())


def test_cfg2_full_depth_end_to_end_vs_oracle():
    w = sg.cfg2()
    cfg = w.model
    L = cfg.n_layers
    N = n_tok(w, w.requests[0])
    eng = B.Engine(cfg, num_blocks=(sum(len(c) for c in w.chunks) + 3 * N) // 16 + 64, max_rows=4096,
                   max_tokens=N + 16, device=0)
    eng.kv_share = 3                                           # the bench's configuration (chunk-frame link)
    try:
        ids = eng.generate_context_cache(w.chunks)
        segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
        g = eng.link(segs, w.alg, keep_linked=True, want_selected=True)
        d = eng.link(segs, w.alg, keep_linked=True, debug_hidden=True, use_graph=False, want_selected=True)
        assert np.array_equal(g.logits, d.logits) and np.array_equal(g.selected, d.selected)
        sel = g.selected
        assert len(sel) == 4 * 16 + 64                         # k' = 128 (SURVEY §8 legend)
        # oracle from the GPU's compiled chunks only (compile is compared separately at truncated depth)
        over = []
        for cid in ids:
            ks, vs = zip(*[eng.cache_export(cid, l) for l in range(L)])
            over.append((np.stack([f64(k) for k in ks]), np.stack([f64(v) for v in vs])))
        store = P.Store(M.Weights(cfg, cache_layers=1))
        oids = store.compile(w.chunks, compiled_override=over)
        del over
        ref = P.link(store, [("cached", oids[s.chunk]) if s.cached else ("tokens", s.tokens)
                             for s in w.requests[0]], w.alg)
        assert np.array_equal(ref.plan.sel, sel)
        errs = []
        for l in range(L):
            eh = rel(d.hidden[l, :len(sel)], ref.hidden[l])
            kg, vg = eng.linked_export(g.linked, l)
            ek, ev = rel(f64(kg), ref.K[l]), rel(f64(vg), ref.V[l])
            errs.append((l, eh, ek, ev))
            assert eh < TOL and ek < TOL and ev < TOL, errs[-1]
        el = rel(g.logits, ref.logits)
        print(f"cfg2 full depth: logits rel-L2 {el:.2e}; hidden after layer 0/15/31 "
              f"{errs[0][1]:.2e}/{errs[15][1]:.2e}/{errs[31][1]:.2e}; max K {max(e[2] for e in errs):.2e} "
              f"V {max(e[3] for e in errs):.2e}")
        assert el < TOL, el
        assert first_token_ok(g.logits, ref.logits)
        eng.release(g.linked)
        eng.release(d.linked)
    finally:
        eng.close()


@pytest.mark.parametrize("kv_share", [1, 3])
def test_cfg4_wave_sampled_rows_vs_oracle(kv_share):
    w = sg.cfg4(n_requests=32)
    cfg = w.model
    L = cfg.n_layers
    Ns = [n_tok(w, r) for r in w.requests]
    eng = B.Engine(cfg, num_blocks=sum(len(c) for c in w.chunks) // 16 + (sum(Ns) + 2 * max(Ns)) // 16 + 256,
                   max_rows=8192, max_tokens=max(Ns) + 16, max_requests=32, device=0)
    eng.kv_share = kv_share                                    # 3 is the bench default
    try:
        ids = eng.generate_context_cache(w.chunks)
        reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
        g = eng.link_batch(reqs, w.alg, keep_linked=True)                      # bench configuration
        d = eng.link_batch(reqs, w.alg, keep_linked=True, use_graph=False, debug_hidden=True)
        if kv_share == 3:  # the bench path: the persistent chunk-frame attention kernel (1792 items per layer)
            assert B.last_attention_kernel() == 4, B.last_attention_kernel()
        for a, b in zip(g, d):
            assert np.array_equal(a.logits, b.logits) and a.first_token == b.first_token
        plans = [eng.plan(r, w.alg) for r in reqs]
        r0 = np.cumsum([0] + [len(p["sel"]) for p in plans])
        hid = d[0].hidden
        Wt = M.Weights(cfg, cache_layers=1)
        for l in (0, L - 1):
            for q in (0, 9, 22, 31):
                pl, sel = plans[q], plans[q]["sel"]
                assert len(sel) == 9 * 16 + 64 and sel[-1] == Ns[q] - 1     # k' = 208
                sub = np.unique(np.r_[np.arange(0, len(sel), 8), len(sel) - 1])
                kg, vg = eng.linked_export(g[q].linked, l)
                kd, vd = eng.linked_export(d[q].linked, l)
                assert np.array_equal(kg, kd) and np.array_equal(vg, vd), (l, q)
                h_in = (Wt.embed_rows(pl["tok"][sel[sub]]) if l == 0
                        else hid[l - 1, r0[q] + sub].astype(np.float64))
                K, V = f64(kg), f64(vg)
                h_out = M.layer_rows(Wt.layer(l), cfg, h_in, sel[sub], sel[sub], K, V)
                e = rel(hid[l, r0[q] + sub], h_out)
                assert e < LAYER_TOL, (l, q, e)
                assert rel(f64(kg)[sel[sub]], K[sel[sub]]) < LAYER_TOL, (l, q)
                assert rel(f64(vg)[sel[sub]], V[sel[sub]]) < LAYER_TOL, (l, q)
                # unselected cached rows: R(Δ)·K_chunk of the GPU's own compiled chunk, V bit-equal
                for (start, n, delta), seg in list(zip(pl["chunks"], [s for s in reqs[q] if s[0] == "cached"]))[1:3]:
                    ck, cv = eng.cache_export(seg[1], l)
                    rows = np.arange(16, n)
                    assert np.array_equal(vg[start + rows], cv[rows]), (l, q)
                    refk = P.rebase(f64(ck[rows]), int(delta), cfg.head_dim, cfg.rope_theta)
                    assert rel(f64(kg[start + rows]), refk) < 4e-3, (l, q)
        for q in (0, 9, 22, 31):
            logits = M.logits_of(Wt, hid[L - 1, r0[q + 1] - 1].astype(np.float64))
            assert rel(g[q].logits, logits) < LAYER_TOL, q
        for o in g + d:
            eng.release(o.linked)
    finally:
        eng.close()


def test_cfg5_truncated_depth_sampled_rows_vs_oracle():
    w = sg.cfg5(n_layers=2)
    cfg = w.model
    N = n_tok(w, w.requests[0])
    assert N == 32832 and cfg.n_heads // cfg.n_kv_heads == 8
    eng = B.Engine(cfg, num_blocks=(sum(len(c) for c in w.chunks) + 3 * N) // 16 + 64, max_rows=4096,
                   max_tokens=N + 16, device=0)
    eng.kv_share = 3
    try:
        ids = eng.generate_context_cache(w.chunks)
        segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
        g = eng.link(segs, w.alg, keep_linked=True, want_selected=True)
        d = eng.link(segs, w.alg, keep_linked=True, debug_hidden=True, use_graph=False, want_selected=True)
        assert np.array_equal(g.logits, d.logits) and np.array_equal(g.selected, d.selected)
        sel = g.selected
        assert len(sel) == 63 * 16 + 64                         # k' = 1072 (SURVEY §8 legend)
        pl = eng.plan(segs, w.alg)
        Wt = M.Weights(cfg, cache_layers=1)
        sub = np.unique(np.r_[np.arange(0, len(sel), 16), len(sel) - 1])
        for l in range(2):
            kg, vg = eng.linked_export(g.linked, l)
            h_in = Wt.embed_rows(pl["tok"][sel[sub]]) if l == 0 else d.hidden[l - 1, sub].astype(np.float64)
            K, V = f64(kg), f64(vg)
            h_out = M.layer_rows(Wt.layer(l), cfg, h_in, sel[sub], sel[sub], K, V)
            e = rel(d.hidden[l, sub], h_out)
            assert e < LAYER_TOL, (l, e)
            assert rel(f64(kg)[sel[sub]], K[sel[sub]]) < LAYER_TOL
            (start, n, delta), cid = pl["chunks"][-1], ids[-1]
            ck, cv = eng.cache_export(cid, l)
            rows = np.arange(16, n)
            assert np.array_equal(vg[start + rows], cv[rows])
            refk = P.rebase(f64(ck[rows]), int(delta), cfg.head_dim, cfg.rope_theta)
            assert rel(f64(kg[start + rows]), refk) < 4e-3
        logits = M.logits_of(Wt, d.hidden[1, len(sel) - 1].astype(np.float64))
        assert rel(g.logits, logits) < LAYER_TOL
        eng.release(g.linked)
        eng.release(d.linked)
    finally:
        eng.close()
