"""Full-size parity at BASELINE.json's sizes, in the launch configuration bench.py times
(CUDA graphs on, full depth).  The fp64 oracle cannot run 32 full-width layers, so it checks
SAMPLED outputs one by one:

  1. the graph run and an eager debug run (which also exports every layer's hidden state) are
     bit-identical (logits and linked K/V), so the debug hidden states describe the graph run;
  2. for sampled layers l the oracle recomputes layer l from the GPU's layer input (embeddings or
     hidden[l-1]) and the GPU's linked K/V of layer l, and compares the output residual and the
     recomputed rows' K/V;
  3. unselected cached rows of the linked cache equal R(Δ)·K_chunk (V bit-equal) of the GPU's own
     compiled chunks; the oracle's LM head on the GPU's final hidden state reproduces the logits;
  4. CacheBlend at full size: the selection count is exact and the GPU's selection agrees with the
     oracle's selection recomputed from the GPU's layer-0 output, up to near-threshold swaps.
"""
import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu
TOL = 2e-2
LAYER_TOL = 5e-3    # one layer from identical inputs: bf16 GEMM/attention rounding only


def f32(bits):
    return B.bf16_bits_to_f32(bits).astype(np.float64)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def build(w, max_rows=4096):
    m = w.model
    N = sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in w.requests[0])
    eng = B.Engine(m, num_blocks=(sum(len(c) for c in w.chunks) + 3 * N) // 16 + 64, max_rows=max(max_rows, N),
                   max_tokens=N + 16, device=0)
    ids = eng.generate_context_cache(w.chunks)
    segs = [("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in w.requests[0]]
    return eng, ids, segs, N


def oracle_layer(Wt, l, h_in, pos, sel, K_gpu, V_gpu):
    """Oracle layer l on the GPU's inputs; returns (h_out, K_l, V_l) (K/V rows at sel recomputed)."""
    K = K_gpu.copy()
    V = V_gpu.copy()
    h = M.layer_rows(Wt.layer(l), Wt.cfg, h_in, pos, sel, K, V)
    return h, K, V


@pytest.mark.parametrize("which", ["cfg2", "cfg3"])
def test_fullsize_legolink_sampled_layers(which):
    w = sg.cfg2() if which == "cfg2" else sg.cfg3()
    cfg = w.model
    eng, ids, segs, N = build(w)
    g = eng.link(segs, w.alg, keep_linked=True, want_selected=True)            # bench configuration (graph)
    d = eng.link(segs, w.alg, keep_linked=True, debug_hidden=True, use_graph=False, want_selected=True)
    assert np.array_equal(g.logits, d.logits) and g.first_token == d.first_token
    sel = g.selected
    assert np.array_equal(sel, d.selected)
    L = cfg.n_layers
    Wt = M.Weights(cfg, cache_layers=1)
    pl = eng.plan(segs, w.alg)
    tok = pl["tok"]
    for l in sorted({0, 1, L // 2, L - 1}):
        kg, vg = eng.linked_export(g.linked, l)
        kd, vd = eng.linked_export(d.linked, l)
        assert np.array_equal(kg, kd) and np.array_equal(vg, vd), l
        h_in = Wt.embed_rows(tok[sel]) if l == 0 else d.hidden[l - 1, :len(sel)].astype(np.float64)
        h_out, K, V = oracle_layer(Wt, l, h_in, sel, sel, f32(kg), f32(vg))
        assert rel(d.hidden[l, :len(sel)], h_out) < LAYER_TOL, (l, rel(d.hidden[l, :len(sel)], h_out))
        assert rel(f32(kg)[sel], K[sel]) < LAYER_TOL and rel(f32(vg)[sel], V[sel]) < LAYER_TOL, l
        # K2 rows: re-based copies of the GPU's compiled chunks
        for (start, n, delta), cid in zip(pl["chunks"], ids):
            ck, cv = eng.cache_export(cid, l)
            rows = [j for j in range(n) if start + j not in set(sel.tolist())]
            lin = np.asarray([start + j for j in rows])
            assert np.array_equal(vg[lin], cv[rows]), (l, cid)
            ref = P.rebase(f32(ck[rows]), int(delta), cfg.head_dim, cfg.rope_theta)
            assert rel(f32(kg[lin]), ref) < 4e-3, (l, cid)
    logits = M.logits_of(Wt, d.hidden[L - 1, len(sel) - 1].astype(np.float64))
    assert rel(g.logits, logits) < LAYER_TOL
    eng.release(g.linked)
    eng.release(d.linked)
    eng.close()


def test_fullsize_cacheblend_selection_cfg3():
    w = sg.cfg3("cacheblend:15")
    cfg = w.model
    eng, ids, segs, N = build(w, max_rows=N_rows(w))
    g = eng.link(segs, w.alg, keep_linked=True, want_selected=True)
    d = eng.link(segs, w.alg, keep_linked=True, debug_hidden=True, use_graph=False, want_selected=True)
    assert np.array_equal(g.logits, d.logits) and np.array_equal(g.selected, d.selected)
    assert g.n_selected_layer0 == N == 5120 and g.n_selected == 769          # ⌈0.15·5120⌉ + forced last
    gsel = g.selected
    assert gsel[-1] == N - 1 and np.all(np.diff(gsel) > 0)
    # oracle deviation at the check layer from the GPU's layer-0 output and the GPU's compiled chunks
    Wt = M.Weights(cfg, cache_layers=1)
    pl = eng.plan(segs, w.alg)
    h0 = d.hidden[0, :N].astype(np.float64)
    _, k_new, v_new = M.qkv(Wt.layer(1), cfg, h0, np.arange(N))
    Kc, Vc = np.zeros_like(k_new), np.zeros_like(v_new)
    for (start, n, delta), cid in zip(pl["chunks"], ids):
        ck, cv = eng.cache_export(cid, 1)
        Kc[start:start + n] = P.rebase(f32(ck), int(delta), cfg.head_dim, cfg.rope_theta)
        Vc[start:start + n] = f32(cv)
    dev = ((k_new - Kc) ** 2).sum(axis=(1, 2)) + ((v_new - Vc) ** 2).sum(axis=(1, 2))
    cand = sorted(range(N - 1), key=lambda i: (-dev[i], i))
    T = 768
    osel = set(cand[:T]) | {N - 1}
    diff = set(gsel.tolist()) ^ osel
    thr = dev[cand[T - 1]]
    assert len(diff) <= 0.02 * T, len(diff)
    for i in diff:
        assert abs(dev[i] - thr) <= 0.05 * thr, (i, dev[i], thr)
    # post-selection layers on the GPU's selection: sampled layer L-1 recomputed by the oracle
    L = cfg.n_layers
    kg, vg = eng.linked_export(g.linked, L - 1)
    h_out, K, V = oracle_layer(Wt, L - 1, d.hidden[L - 2, :len(gsel)].astype(np.float64), gsel, gsel, f32(kg), f32(vg))
    assert rel(d.hidden[L - 1, :len(gsel)], h_out) < LAYER_TOL
    eng.release(g.linked)
    eng.release(d.linked)
    eng.close()


def N_rows(w):
    return sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in w.requests[0])


def test_long_context_16k_legolink_sampled_rows():
    """f3 long-context point: N = 16448 (32 x 512 + 64), LegoLink-16 on the
    Llama-3.1-8B shape.  Graph = eager bit-identically; layer 0 and L-1 recomputed by the oracle for
    every 8th selected row from the GPU's inputs; unselected cached keys are R(Δ)·K_chunk."""
    w = sg.long_context(32)
    cfg = w.model
    eng, ids, segs, N = build(w)
    assert N == 16448
    g = eng.link(segs, w.alg, keep_linked=True, want_selected=True)
    d = eng.link(segs, w.alg, keep_linked=True, debug_hidden=True, use_graph=False, want_selected=True)
    assert np.array_equal(g.logits, d.logits) and np.array_equal(g.selected, d.selected)
    sel = g.selected
    assert len(sel) == 31 * 16 + 64
    Wt = M.Weights(cfg, cache_layers=1)
    pl = eng.plan(segs, w.alg)
    L = cfg.n_layers
    sub = np.arange(0, len(sel), 8)
    for l in (0, L - 1):
        kg, vg = eng.linked_export(g.linked, l)
        h_in = Wt.embed_rows(pl["tok"][sel[sub]]) if l == 0 else d.hidden[l - 1, sub].astype(np.float64)
        K, V = f32(kg), f32(vg)
        h_out = M.layer_rows(Wt.layer(l), cfg, h_in, sel[sub], sel[sub], K, V)
        assert rel(d.hidden[l, sub], h_out) < LAYER_TOL, (l, rel(d.hidden[l, sub], h_out))
        assert rel(f32(kg)[sel[sub]], K[sel[sub]]) < LAYER_TOL
        (start, n, delta), cid = pl["chunks"][-1], ids[-1]
        ck, cv = eng.cache_export(cid, l)
        rows = np.arange(16, n)                                  # past the recomputed first 16
        assert np.array_equal(vg[start + rows], cv[rows])
        ref = P.rebase(f32(ck[rows]), int(delta), cfg.head_dim, cfg.rope_theta)
        assert rel(f32(kg[start + rows]), ref) < 4e-3
    eng.release(g.linked)
    eng.release(d.linked)
    eng.close()


@pytest.mark.parametrize("kernel,mode", [(1, 1), (2, 1), (2, 2)])
@pytest.mark.parametrize("which", ["cfg2", "cfg3", "cfg4"])
def test_fullsize_shared_block_link_bit_identical(which, kernel, mode):
    """f3 shared-block link at full size in the bench's launch configuration (graphs, batched link for
    cfg4): logits, first tokens and sampled layers' linked K/V are bit-identical to the copy path, which
    the sampled-layer tests above hold to the oracle — on the same attention kernel for both paths
    (1 = one q-tile per CTA, 2 = ping-pong: the engine picks per link, so it is forced here)."""
    B.set_attention_kernel(kernel)
    w = {"cfg2": sg.cfg2, "cfg3": sg.cfg3}.get(which, lambda: sg.cfg4(n_requests=4))()
    m = w.model
    Ns = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]
    eng = B.Engine(m, num_blocks=(sum(len(c) for c in w.chunks) + 2 * sum(Ns)) // 16 + 64, max_rows=4096,
                   max_tokens=max(Ns) + 16, max_requests=len(w.requests), device=0)
    try:
        ids = eng.generate_context_cache(w.chunks)
        reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
        outs = [eng.link_batch(reqs, w.alg, keep_linked=True, kv_share=share) for share in (0, mode)]
        shared = 0
        for a, b in zip(*outs):
            assert np.array_equal(a.logits, b.logits) and a.first_token == b.first_token
            shared += eng.linked_sharing(b.linked)[0]
            for l in (0, m.n_layers // 2, m.n_layers - 1):
                ka, va = eng.linked_export(a.linked, l)
                kb, vb = eng.linked_export(b.linked, l)
                assert np.array_equal(ka, kb) and np.array_equal(va, vb), l
        assert shared > 0
    finally:
        B.set_attention_kernel(0)
        eng.close()


@pytest.mark.parametrize("which", ["cfg2", "cfg4"])
def test_fullsize_chunkframe_qrot_link(which):
    """kv_share 3 at full size: every 128-key tile of these links lies inside one 512-token chunk, so the
    attention re-bases by rotating Q per chunk frame (QROT).  Held to the copy path (itself held to the
    oracle above) at the north star's 2e-2: logits, first tokens, and sampled layers' linked K/V exports."""
    w = sg.cfg2() if which == "cfg2" else sg.cfg4(n_requests=4)
    m = w.model
    Ns = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]
    eng = B.Engine(m, num_blocks=(sum(len(c) for c in w.chunks) + 2 * sum(Ns)) // 16 + 64, max_rows=4096,
                   max_tokens=max(Ns) + 16, max_requests=len(w.requests), device=0)
    try:
        ids = eng.generate_context_cache(w.chunks)
        reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
        outs = [eng.link_batch(reqs, w.alg, keep_linked=True, kv_share=share) for share in (0, 3)]
        for a, b in zip(*outs):
            assert rel(b.logits, a.logits) < 2e-2
            # different re-base arithmetic (Q rotated instead of K): the argmax is held to the copy path's
            # unless its top-1/top-2 gap is within 4x the measured logit error (SURVEY §8(c).8 near ties)
            assert b.first_token == int(np.argmax(b.logits))
            top = np.argsort(-a.logits)[:2]
            err = float(np.max(np.abs(np.asarray(b.logits, np.float64) - a.logits)))
            if a.logits[top[0]] - a.logits[top[1]] > 4 * err:
                assert b.first_token == a.first_token
            else:
                assert b.first_token in set(top.tolist())
            for l in (0, m.n_layers // 2, m.n_layers - 1):
                ka, va = eng.linked_export(a.linked, l)
                kb, vb = eng.linked_export(b.linked, l)
                assert rel(f32(kb), f32(ka)) < 2e-2, l
                assert rel(f32(vb), f32(va)) < 2e-2, l
    finally:
        eng.close()


def test_fullsize_qrot_persistent_bit_identical():
    """cfg4 (4 requests, full depth, eager): the persistent QROT attention kernel (default for kv_share 3)
    equals the one-CTA-per-item QROT kernel bit for bit (logits, sampled layers' linked K/V)."""
    import os
    w = sg.cfg4(n_requests=4)
    m = w.model
    Ns = [sum(len(w.chunks[s.chunk]) if s.cached else len(s.tokens) for s in r) for r in w.requests]
    eng = B.Engine(m, num_blocks=(sum(len(c) for c in w.chunks) + 3 * sum(Ns)) // 16 + 64, max_rows=4096,
                   max_tokens=max(Ns) + 16, max_requests=len(w.requests), device=0)
    try:
        ids = eng.generate_context_cache(w.chunks)
        reqs = [[("cached", ids[s.chunk]) if s.cached else ("tokens", s.tokens) for s in r] for r in w.requests]
        outs = []
        for key in ("PIC_ATTN_PERSIST", "PIC_NO_ATTN_PERSIST"):  # 224 items: force either kernel
            os.environ[key] = "1"
            try:
                outs.append(eng.link_batch(reqs, w.alg, keep_linked=True, kv_share=3, use_graph=False))
                assert B.last_attention_kernel() == (4 if key == "PIC_ATTN_PERSIST" else 3)
            finally:
                os.environ.pop(key, None)
        for a, b in zip(*outs):
            assert np.array_equal(a.logits, b.logits)
            for l in (0, m.n_layers - 1):
                ka, va = eng.linked_export(a.linked, l)
                kb, vb = eng.linked_export(b.linked, l)
                assert np.array_equal(ka, kb) and np.array_equal(va, vb), l
    finally:
        eng.close()
