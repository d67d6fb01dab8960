"""Pins of the fp64 oracle against things other than itself (SURVEY §8(c).4, C1–C13).

Independent references used here:
  * HuggingFace ``transformers`` LlamaForCausalLM in float64 (a library implementation of
    the Llama decoder: RMSNorm, rotate-half RoPE, GQA, SwiGLU, causal softmax attention)
    loaded with the oracle's weights — pins the decoder, full prefill, and (through its
    KV-cache API) the Naive construction C6;
  * scipy.special.softmax brute force per query (C1);
  * complex-number RoPE (C7, C12);
  * torch's bfloat16 conversion (generator rounding), published SplitMix64 outputs;
  * closed-form plan arithmetic printed in SPEC/SURVEY (C10) and causality identities
    (C3, C4, C8, C9, C11).
"""
import numpy as np
import pytest
import scipy.special

import seedgen as sg
from oracle import model as M
from oracle import pic as P


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ----------------------------------------------------------------------------
# generator pins
# ----------------------------------------------------------------------------
def test_splitmix64_published_vectors():
    # SplitMix64 seeded with 0 (Steele/Lea/Flood; Vigna's reference C): the first outputs.
    outs, state = [], 0
    for _ in range(3):
        outs.append(sg.sm64_int(state))
        state = (state + sg.GOLDEN) & sg.M64
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    # the numpy path agrees with the integer path
    x = np.arange(1000, dtype=np.uint64) * np.uint64(0x123456789)
    assert all(int(a) == sg.sm64_int(int(b)) for a, b in zip(sg._sm64_np(x), x))


def test_bf16_rounding_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32),
                        sg.uniform_pm1(sg.U(1, 2, np.arange(100000, dtype=np.uint64)))])
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(sg.bf16_rne(x), ref)


def test_uniform_exact_and_range():
    u = sg.U(7, 3, np.arange(1 << 16, dtype=np.uint64))
    f = sg.uniform_pm1(u)
    assert f.min() >= -1.0 and f.max() < 1.0
    # exactness: float64 evaluation gives the same numbers
    f64 = (u >> np.uint64(40)).astype(np.float64) * 2.0 ** -23 - 1.0
    assert np.array_equal(f.astype(np.float64), f64)
    w = sg.matrix(5, 9, 64, 4096)
    assert np.array_equal(w, sg.bf16_rne(w))                      # bf16-exact
    assert abs(np.var(w) * 4096 - 1.0) < 0.5                      # variance ≈ 1/fan_in


# ----------------------------------------------------------------------------
# decoder pinned against HuggingFace Llama (float64)
# ----------------------------------------------------------------------------
HF_TOL = 2e-6   # float32 internals of HF's RMSNorm / softmax (see hf_model)


def test_rms_norm_matches_torch_and_silu():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    x = rng.standard_normal((7, 64)) * 3
    g = rng.standard_normal(64)
    ref = torch.nn.functional.rms_norm(torch.from_numpy(x), (64,), torch.from_numpy(g), eps=1e-5).numpy()
    assert np.abs(M.rms_norm(x, g, 1e-5) - ref).max() < 1e-14
    ref = torch.nn.functional.silu(torch.from_numpy(x)).numpy()
    assert np.abs(M.silu(x) - ref).max() < 1e-14


def hf_model(cfg: sg.ModelConfig, Wt: M.Weights):
    torch = pytest.importorskip("torch")
    tf = pytest.importorskip("transformers")
    c = tf.LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model, intermediate_size=cfg.ffn_dim,
                       num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
                       num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, rms_norm_eps=cfg.rms_eps,
                       rope_theta=cfg.rope_theta, tie_word_embeddings=False, attention_bias=False,
                       mlp_bias=False, max_position_embeddings=cfg.max_pos)
    c._attn_implementation = "eager"
    m = tf.LlamaForCausalLM(c).double().eval()
    # HF evaluates RoPE angles, RMSNorm and the softmax in float32 even for a float64
    # model.  The angles are re-evaluated in float64 here (θ^(−2j/D)·p, pinned again by
    # the complex-rotation test); the float32 norm/softmax bound the comparison to
    # HF_TOL.  RMSNorm and softmax are pinned separately at 1e-14 against
    # torch.nn.functional.rms_norm and scipy.
    rot = m.model.rotary_emb

    def rot_forward(x, position_ids):
        j = torch.arange(0, cfg.head_dim, 2, dtype=torch.float64)
        inv = cfg.rope_theta ** (-j / cfg.head_dim)
        fr = position_ids.to(torch.float64)[..., None] * inv
        emb = torch.cat([fr, fr], dim=-1)
        return emb.cos().to(x.dtype), emb.sin().to(x.dtype)

    rot.forward = rot_forward
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(T(Wt.embed))
        m.lm_head.weight.copy_(T(Wt.lm_head))
        m.model.norm.weight.copy_(T(Wt.g_final))
        for l, layer in enumerate(m.model.layers):
            W = Wt.layer(l)
            layer.self_attn.q_proj.weight.copy_(T(W["q"]))
            layer.self_attn.k_proj.weight.copy_(T(W["k"]))
            layer.self_attn.v_proj.weight.copy_(T(W["v"]))
            layer.self_attn.o_proj.weight.copy_(T(W["o"]))
            layer.mlp.gate_proj.weight.copy_(T(W["gate"]))
            layer.mlp.up_proj.weight.copy_(T(W["up"]))
            layer.mlp.down_proj.weight.copy_(T(W["down"]))
            layer.input_layernorm.weight.copy_(T(W["g1"]))
            layer.post_attention_layernorm.weight.copy_(T(W["g2"]))
    return m


@pytest.mark.parametrize("cfg", [sg.TINY, sg.TINY_GQA, sg.TINY_D128], ids=lambda c: c.name)
def test_full_prefill_matches_hf_llama(cfg):
    torch = pytest.importorskip("torch")
    Wt = M.Weights(cfg)
    w = sg.cfg1(model=cfg)
    tok = np.concatenate([w.chunks[0], w.requests[0][-1].tokens])
    logits, K, V, _ = M.full_prefill(Wt, tok)
    m = hf_model(cfg, Wt)
    with torch.no_grad():
        out = m(torch.from_numpy(tok.astype(np.int64))[None], use_cache=True)
    assert rel(logits, out.logits[0, -1].numpy()) < HF_TOL
    # cached keys/values of HF are post-RoPE [B, H_kv, T, D]
    kv = out.past_key_values
    for l in range(cfg.n_layers):
        k_hf = kv.layers[l].keys[0].numpy().transpose(1, 0, 2)
        v_hf = kv.layers[l].values[0].numpy().transpose(1, 0, 2)
        assert rel(K[l], k_hf) < HF_TOL
        assert rel(V[l], v_hf) < HF_TOL


# ----------------------------------------------------------------------------
# C1 / C2: attention
# ----------------------------------------------------------------------------
def test_C1_attention_brute_force():
    rng = np.random.default_rng(1)
    n, Hq, Hkv, D = 9, 4, 2, 8
    q = rng.standard_normal((n, Hq, D))
    k = rng.standard_normal((n, Hkv, D))
    v = rng.standard_normal((n, Hkv, D))
    pos = np.arange(n)
    out = M.causal_attention(q, k, v, pos)
    for h in range(Hq):
        g = h // (Hq // Hkv)
        for i in range(n):
            s = np.array([q[i, h] @ k[j, g] / np.sqrt(D) for j in range(i + 1)])
            p = scipy.special.softmax(s)
            ref = sum(p[j] * v[j, g] for j in range(i + 1))
            assert np.allclose(out[i, h], ref, atol=1e-12, rtol=0)
        A = M.attention_matrix_dense(q[:, h], k[:, g])
        assert np.allclose(A.sum(1), 1.0, atol=1e-12)
        assert np.all(A[np.triu_indices(n, 1)] == 0.0)
    # closed forms: zero query → uniform average of visible values; first row → v[0]
    out0 = M.causal_attention(np.zeros_like(q), k, v, pos)
    for i in range(n):
        assert np.allclose(out0[i, 0], v[: i + 1, 0].mean(0), atol=1e-12)
    assert np.allclose(out[0, :, :], v[0, np.arange(Hq) // 2], atol=1e-12)


def test_C2_sparse_query_rows_equal_dense_rows():
    rng = np.random.default_rng(2)
    n, H, D = 40, 2, 8
    q = rng.standard_normal((n, H, D))
    k = rng.standard_normal((n, H, D))
    v = rng.standard_normal((n, H, D))
    dense = M.causal_attention(q, k, v, np.arange(n))
    sel = np.array([3, 7, 8, 20, 39])
    sparse = M.causal_attention(q[sel], k, v, sel)
    assert np.abs(sparse - dense[sel]).max() <= 1e-12


# ----------------------------------------------------------------------------
# RoPE pins (C7, C12)
# ----------------------------------------------------------------------------
def complex_rope(x, pos, theta):
    D = x.shape[-1]
    h = D // 2
    z = x[..., :h] + 1j * x[..., h:]
    ang = np.outer(pos, theta ** (-np.arange(h) * 2.0 / D))
    z = z * np.exp(1j * ang)[:, None, :]
    return np.concatenate([z.real, z.imag], axis=-1)


def test_rope_matches_complex_rotation_and_preserves_norm():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((50, 3, 128))
    pos = rng.integers(0, 32832, 50)
    y = M.rope(x, pos, 5e5)
    assert np.abs(y - complex_rope(x, pos, 5e5)).max() < 1e-12
    n1 = x[..., :64] ** 2 + x[..., 64:] ** 2
    n2 = y[..., :64] ** 2 + y[..., 64:] ** 2
    assert np.abs(n1 - n2).max() < 1e-12                         # C12 pair norms


def test_C7_rebase_identity():
    rng = np.random.default_rng(4)
    k = rng.standard_normal((16, 2, 128))
    p = np.arange(16)
    for delta in (0, 1, 512, 31232):
        lhs = P.rebase(M.rope(k, p, 1e4), delta, 128, 1e4)
        rhs = M.rope(k, p + delta, 1e4)
        assert np.abs(lhs - rhs).max() < 1e-10
    assert np.array_equal(P.rebase(k, 0, 128, 1e4), k)            # Δ = 0 is exact


# ----------------------------------------------------------------------------
# link pins on cfg1
# ----------------------------------------------------------------------------
@pytest.fixture(scope="module", params=[sg.TINY, sg.TINY_GQA], ids=lambda c: c.name)
def tiny(request):
    cfg = request.param
    w = sg.cfg1(model=cfg)
    Wt = M.Weights(cfg)
    store = P.Store(Wt)
    ids = store.compile(w.chunks)
    segs = [("cached", ids[0]), ("cached", ids[1]), ("cached", ids[2]), ("tokens", w.requests[0][-1].tokens)]
    tok = np.concatenate(w.chunks + [w.requests[0][-1].tokens])
    ref = M.full_prefill(Wt, tok)
    return cfg, w, Wt, store, ids, segs, tok, ref


def test_C3_fr_equals_full_prefill(tiny):
    cfg, w, Wt, store, ids, segs, tok, (logits, K, V, _) = tiny
    r = P.link(store, segs, "fr")
    assert rel(r.logits, logits) < 1e-12
    assert rel(r.K, K) < 1e-12 and rel(r.V, V) < 1e-12
    assert len(r.plan.sel) == 112


def test_C4_saturated_legolink_equals_fr(tiny):
    cfg, w, Wt, store, ids, segs, tok, (logits, K, V, _) = tiny
    r = P.link(store, segs, "legolink:32")
    assert len(r.plan.sel) == 112 - 32                           # index-0 chunk exempt
    assert rel(r.logits, logits) < 1e-12
    assert rel(r.K, K) < 1e-12 and rel(r.V, V) < 1e-12
    r2 = P.link(store, segs, "legolink:1000")
    assert rel(r2.logits, logits) < 1e-12


def test_C5_legolink0_equals_naive(tiny):
    cfg, w, Wt, store, ids, segs, *_ = tiny
    a = P.link(store, segs, "legolink:0")
    b = P.link(store, segs, "naive")
    assert np.array_equal(a.plan.sel, b.plan.sel)
    assert np.array_equal(a.logits, b.logits)


def test_C6_naive_equals_hf_prefill_over_rebased_prefix(tiny):
    """Independent construction: HF Llama's KV cache filled with the re-based chunk KV
    (the 'prefix'), then an ordinary HF forward of only the dynamic tokens."""
    torch = pytest.importorskip("torch")
    tf = pytest.importorskip("transformers")
    cfg, w, Wt, store, ids, segs, tok, _ = tiny
    r = P.link(store, segs, "naive")
    m = hf_model(cfg, Wt)
    cache = tf.DynamicCache(config=m.config)
    n_pre = 96
    for l in range(cfg.n_layers):
        ks, vs = [], []
        for c, cid in enumerate(ids):
            ch = store.chunks[cid]
            ks.append(P.rebase(ch.K[l], 32 * c, cfg.head_dim, cfg.rope_theta))
            vs.append(ch.V[l])
        k = torch.from_numpy(np.concatenate(ks).transpose(1, 0, 2)[None].copy())
        v = torch.from_numpy(np.concatenate(vs).transpose(1, 0, 2)[None].copy())
        cache.update(k, v, l)
    q = w.requests[0][-1].tokens.astype(np.int64)
    with torch.no_grad():
        out = m(torch.from_numpy(q)[None], past_key_values=cache, use_cache=True,
                position_ids=torch.arange(n_pre, n_pre + len(q))[None])
    assert rel(r.logits, out.logits[0, -1].numpy()) < HF_TOL
    for l in range(cfg.n_layers):
        k_hf = out.past_key_values.layers[l].keys[0].numpy().transpose(1, 0, 2)
        assert rel(r.K[l], k_hf) < HF_TOL


def test_C8_layer0_kv_equals_prefill_for_every_algorithm(tiny):
    cfg, w, Wt, store, ids, segs, tok, (logits, K, V, _) = tiny
    for alg in ("naive", "legolink:4", "cacheblend:15", "fr"):
        r = P.link(store, segs, alg)
        assert rel(r.K[0], K[0]) < 1e-12, alg
        assert rel(r.V[0], V[0]) < 1e-12, alg


def test_C9_prefix_equivalence(tiny):
    cfg, w, Wt, store, ids, segs, tok, _ = tiny
    q = w.requests[0][-1].tokens
    logits, K, V, _ = M.full_prefill(Wt, np.concatenate([w.chunks[1], q]))
    for alg in ("naive", "legolink:4", "cacheblend:15", "fr"):
        r = P.link(store, [("cached", ids[1]), ("tokens", q)], alg)
        assert rel(r.logits, logits) < 1e-12, alg
        assert rel(r.K, K) < 1e-12, alg


def test_C10_plan_arithmetic():
    cfg = sg.TINY
    Wt = M.Weights(cfg)
    store = P.Store(Wt)
    w = sg.cfg1()
    # planning needs only the store's token lists: use zero KV placeholders
    ids = store.compile(w.chunks, compiled_override=[(None, None)] * 3)
    q = w.requests[0][-1].tokens
    segs = [("cached", i) for i in ids] + [("tokens", q)]
    pl = P.plan(store, segs, "legolink:4")
    assert pl.sel.tolist() == list(range(32, 36)) + list(range(64, 68)) + list(range(96, 112))
    assert len(P.plan(store, segs, "fr").sel) == 112
    assert P.plan(store, segs, "naive").sel.tolist() == list(range(96, 112))
    # SPEC S:326 example: 3 chunks × 48 + 16-token query, LegoLink-16
    ids48 = store.compile([np.arange(48, dtype=np.int32) + 2] * 3, compiled_override=[(None, None)] * 3)
    segs48 = [("cached", i) for i in ids48] + [("tokens", np.arange(16, dtype=np.int32) + 5)]
    pl = P.plan(store, segs48, "legolink:16")
    assert pl.sel.tolist() == list(range(48, 64)) + list(range(96, 112)) + list(range(144, 160))
    # CacheBlend-15 on that layout: 160 rows at layer 0, then 16 + ⌈0.15·144⌉ = 38
    cb = P.plan(store, segs48, "cacheblend:15")
    assert P.cacheblend_count(cb) == 22
    dev = np.arange(160, dtype=np.float64)
    sel = P.cacheblend_select(cb, dev)
    assert len(sel) == 38 and sel[-1] == 159
    # cfg1 CB-15: 112 → 15 + 16 = 31; cfg3 CB-15 (no dynamic): 5120 → 768 + forced last = 769
    cb1 = P.plan(store, segs, "cacheblend:15")
    assert len(P.cacheblend_select(cb1, np.zeros(112))) == 31
    # dynamic-first order: no chunk is exempt
    pl = P.plan(store, [("tokens", q)] + [("cached", i) for i in ids], "legolink:4")
    assert pl.sel.tolist() == list(range(16)) + [16, 17, 18, 19, 48, 49, 50, 51, 80, 81, 82, 83] + [111]
    # chunk deltas
    assert [c[3] for c in pl.chunks] == [16, 48, 80]
    # ties → lower index
    dev = np.zeros(160)
    assert P.cacheblend_select(cb, dev)[:22].tolist() == list(range(22))


def test_C11_cacheblend_index0_deviation_zero_and_count(tiny):
    cfg, w, Wt, store, ids, segs, *_ = tiny
    r = P.link(store, segs, "cacheblend:15")
    assert r.dev is not None
    assert np.abs(r.dev[:32]).max() <= 1e-20 * max(1.0, np.abs(r.dev).max())
    assert r.dev[32:96].min() > 0
    assert len(r.sel_per_layer[0]) == 112 and len(r.sel_per_layer[1]) == 31
    # selection override reproduces the oracle's own selection
    r2 = P.link(store, segs, "cacheblend:15", sel_override=r.sel_per_layer[1])
    assert np.array_equal(r2.logits, r.logits)


def test_C12_unselected_cached_v_rows_bit_equal(tiny):
    cfg, w, Wt, store, ids, segs, *_ = tiny
    r = P.link(store, segs, "legolink:4")
    sel = set(r.plan.sel.tolist())
    for c, cid in enumerate(ids):
        for j in range(32):
            i = 32 * c + j
            if i in sel:
                continue
            assert np.array_equal(r.V[:, i], store.chunks[cid].V[:, j])
            if c == 0:
                assert np.array_equal(r.K[:, i], store.chunks[cid].K[:, j])   # Δ = 0 exact


def test_C13_algorithms_distinguishable(tiny):
    cfg, w, Wt, store, ids, segs, tok, (logits, *_ ) = tiny
    naive = P.link(store, segs, "naive").logits
    lego = P.link(store, segs, "legolink:4").logits
    assert rel(naive, logits) > 5 * 2e-2
    assert rel(lego, logits) > 2e-2
    assert rel(naive, lego) > 2e-2


def test_rebase_off_reading_differs(tiny):
    cfg, w, Wt, store, ids, segs, tok, (logits, K, V, _) = tiny
    r = P.link(store, segs, "naive", rebase_keys=False)
    assert rel(r.K[0], K[0]) > 0.1          # SPEC's no-rebase reading is a different method


def test_allocator_and_slot_map():
    a = P.BlockAllocator(10)
    assert a.alloc(3) == [0, 1, 2]
    assert a.alloc(2) == [3, 4]
    a.release([1, 3])
    assert a.alloc(3) == [1, 3, 5]
    with pytest.raises(MemoryError):
        a.alloc(10)
    assert P.slot_map([7, 2], [0, 15, 16, 31]).tolist() == [112, 127, 32, 47]


def test_C14_legolink0_after_literal_dummies_equals_prefill(tiny):
    """LegoLink-0: a chunk compiled behind m dummy tokens, linked right after m literal
    dummies, lands at Δ = s_c − m = 0 and needs no recomputation — the result is exactly an ordinary
    prefill of dummy^m ‖ chunk (the compile's own computation seen from the link side)."""
    cfg, w, Wt, *_ = tiny
    m = 4
    store = P.Store(Wt)
    chunk = w.chunks[1]
    (cid,) = store.compile([chunk], dummy_prefix=m)
    assert store.chunks[cid].c0 == m and store.chunks[cid].K.shape[1] == len(chunk)
    bos = np.full(m, cfg.bos_id, np.int32)
    r = P.link(store, [("tokens", bos), ("cached", cid)], "legolink0")
    logits, K, V, _ = M.full_prefill(Wt, np.concatenate([bos, chunk]))
    assert r.plan.chunks[0][3] == 0
    assert r.plan.sel.tolist() == list(range(m)) + [m + len(chunk) - 1]
    assert rel(r.logits, logits) < 1e-12
    assert rel(r.K, K) < 1e-12 and rel(r.V, V) < 1e-12


def test_C15_legolink0_variant_check_and_negative_delta(tiny):
    """S:324 variant mismatch; Δ = s_c − m (negative for the chunk placed first, R21) is undone by R(+m)."""
    cfg, w, Wt, *_ = tiny
    m = 4
    store = P.Store(Wt)
    plain = store.compile([w.chunks[0]])
    dummy = store.compile(w.chunks, dummy_prefix=m)
    # the dummies change what the chunk's KV encodes (attention sink removed in advance)
    assert rel(store.chunks[dummy[0]].K, store.chunks[plain[0]].K) > 1e-3
    with pytest.raises(ValueError):
        P.plan(store, [("cached", plain[0]), ("cached", dummy[1])], "legolink0")
    segs = [("cached", c) for c in dummy] + [("tokens", w.requests[0][-1].tokens)]
    r = P.link(store, segs, "legolink0")
    nv = P.plan(store, segs, "naive")
    assert np.array_equal(r.plan.sel, nv.sel)                          # "skips recomputation entirely"
    assert [d for *_, d in r.plan.chunks] == [s - m for _, s, _, _ in r.plan.chunks]
    assert r.plan.chunks[0][3] == -m
    c = store.chunks[dummy[0]]
    n = len(c.tokens)
    for l in range(cfg.n_layers):
        back = P.rebase(r.K[l, :n], m, cfg.head_dim, cfg.rope_theta)
        assert rel(back, c.K[l]) < 1e-12
        assert np.array_equal(r.V[l, :n], c.V[l])


def test_C16_decode_after_fr_equals_prefill_of_extended_prompt(tiny):
    """Decode (f1): FR link of the prompt, then two decode steps, equals an ordinary prefill of
    prompt ‖ t1 ‖ t2 (logits of the last row and every K/V row)."""
    cfg, w, Wt, store, ids, segs, tok, _ = tiny
    r = P.link(store, segs, "fr")
    t1, t2 = 17, 201
    lg1, K, V = P.decode(Wt, r.K, r.V, t1)
    lg2, K, V = P.decode(Wt, K, V, t2)
    ref1 = M.full_prefill(Wt, np.concatenate([tok, [t1]]))
    ref2 = M.full_prefill(Wt, np.concatenate([tok, [t1, t2]]))
    assert rel(lg1, ref1[0]) < 1e-12 and rel(lg2, ref2[0]) < 1e-12
    assert rel(K, ref2[1]) < 1e-12 and rel(V, ref2[2]) < 1e-12


def test_C17_decode_equals_link_with_the_token_as_literal(tiny):
    """For Naive / LegoLink requests that end with literal tokens, decoding t after the link equals
    linking the same message list with t appended as one more literal token (the new row is dynamic,
    every earlier row is computed exactly as before)."""
    cfg, w, Wt, store, ids, segs, tok, _ = tiny
    for alg in ("naive", "legolink:4"):
        r = P.link(store, segs, alg)
        lg, K, V = P.decode(Wt, r.K, r.V, 99)
        q = np.concatenate([segs[-1][1], [99]]).astype(np.int32)
        r2 = P.link(store, segs[:-1] + [("tokens", q)], alg)
        assert rel(lg, r2.logits) < 1e-12, alg
        assert rel(K, r2.K) < 1e-12 and rel(V, r2.V) < 1e-12, alg


# ----------------------------------------------------------------------------
# C18: LegoLink with 0 < k < n_c by an independent construction
# ----------------------------------------------------------------------------
def _complex_rebase(k_post, delta, cfg):
    """R(Δ) on post-RoPE keys [H, n, D] as complex multiplication of the rotate-half pairs
    (x_j + i·x_{j+D/2})·e^{iΔθ_j}, θ_j = rope_theta^(−2j/D) — the definition pinned by C7."""
    D = cfg.head_dim
    th = cfg.rope_theta ** (-np.arange(0, D, 2, dtype=np.float64) / D)
    z = (k_post[..., : D // 2] + 1j * k_post[..., D // 2:]) * np.exp(1j * delta * th)
    return np.concatenate([z.real, z.imag], axis=-1)


def hf_legolink(cfg, Wt, parts, k):
    """PAPER.md:213 (LegoLink, §4.2) built from HuggingFace Llama alone, in message order: a cached chunk
    at message index 0 is linked as is; every later cached chunk contributes its first k tokens as an
    ordinary HF forward over the KV cache built so far, then its remaining rows' KV from a standalone HF
    prefill of the chunk (positions 0..n−1) re-based to their linked positions; dynamic tokens are an
    ordinary forward.  The recomputed rows therefore attend to every earlier cached and recomputed row,
    layer by layer (Eq. 1).  Returns the last forward's final logits and the per-layer K/V
    [L][N][H_kv][D] of the whole linked cache."""
    torch = pytest.importorskip("torch")
    tf = pytest.importorskip("transformers")
    m = hf_model(cfg, Wt)
    cache = tf.DynamicCache(config=m.config)
    pos, logits = 0, None

    def fwd(tok, p0):
        with torch.no_grad():
            return m(torch.from_numpy(np.asarray(tok, np.int64))[None], past_key_values=cache, use_cache=True,
                     position_ids=torch.arange(p0, p0 + len(tok))[None])

    for idx, (kind, tok) in enumerate(parts):
        n = len(tok)
        if kind == "tokens":
            logits = fwd(tok, pos).logits[0, -1].numpy()
        else:
            kk = 0 if idx == 0 else min(k, n)  # the message-index-0 chunk is exempt (reading R9, SPEC)
            # the prompt's last token is always recomputed (its logits give the first token)
            ke = n - 1 if idx == len(parts) - 1 else n
            if kk:
                logits = fwd(tok[:kk], pos).logits[0, -1].numpy()
            if kk < ke:
                with torch.no_grad():
                    alone = m(torch.from_numpy(np.asarray(tok, np.int64))[None], use_cache=True).past_key_values
                for l in range(cfg.n_layers):
                    kc = alone.layers[l].keys[0].numpy()[:, kk:ke]        # [H_kv, ke - kk, D] at kk..ke-1
                    vc = alone.layers[l].values[0].numpy()[:, kk:ke]
                    kr = _complex_rebase(kc, pos, cfg)
                    cache.update(torch.from_numpy(kr[None].copy()), torch.from_numpy(vc[None].copy()), l)
            if ke < n and kk < n:
                logits = fwd(tok[n - 1:], pos + n - 1).logits[0, -1].numpy()
        pos += n
    K = [cache.layers[l].keys[0].numpy().transpose(1, 0, 2) for l in range(cfg.n_layers)]
    V = [cache.layers[l].values[0].numpy().transpose(1, 0, 2) for l in range(cfg.n_layers)]
    return logits, K, V


@pytest.mark.parametrize("cfg", [sg.TINY, sg.TINY_GQA, sg.TINY_D128], ids=lambda c: c.name)
@pytest.mark.parametrize("k", [1, 4, 16])
def test_C18_legolink_equals_hf_sequential_construction(cfg, k):
    """Pins LegoLink for 0 < k < n_c (previously 'parity unpinned'): the oracle's layer-by-layer
    recomputation of the selected rows over the linked cache equals the HF construction above, for the
    canonical request and a permuted one (dynamic tokens first, chunks out of order, the prompt ending in a
    cached chunk whose last token is recomputed)."""
    w = sg.cfg1(model=cfg)
    Wt = M.Weights(cfg)
    store = P.Store(Wt)
    ids = store.compile(w.chunks)
    q = w.requests[0][-1].tokens
    for order in ([0, 1, 2, "q"], ["q", 2, 0, 1]):
        segs = [("tokens", q) if c == "q" else ("cached", ids[c]) for c in order]
        parts = [("tokens", q) if c == "q" else ("chunk", w.chunks[c]) for c in order]
        r = P.link(store, segs, f"legolink:{k}")
        logits, K, V = hf_legolink(cfg, Wt, parts, k)
        assert rel(r.logits, logits) < HF_TOL
        for l in range(cfg.n_layers):
            assert rel(r.K[l], K[l]) < HF_TOL, l
            assert rel(r.V[l], V[l]) < HF_TOL, l


# ----------------------------------------------------------------------------
# C19: CacheBlend with a non-trivial selection by an independent construction
# ----------------------------------------------------------------------------
class _PrefixKV:
    """Duck-typed HF cache for one decoder-layer call: keys/values already in the linked cache (any
    order: the mask carries the positions) followed by the rows the call computes."""

    def __init__(self, k, v):
        self.k, self.v = k, v

    def update(self, k, v, layer_idx, *args, **kwargs):
        return torch_cat(self.k, k), torch_cat(self.v, v)


def torch_cat(a, b):
    import torch
    return b if a is None else torch.cat([a, b], dim=2)


def hf_cacheblend(cfg, Wt, parts, r_pct, check_layer=1):
    """PAPER.md:170 (CacheBlend, as the paper describes it) built from HuggingFace Llama's own decoder
    layers, RoPE and LM head: layer 0 recomputed for all N rows (ordinary causal prefill layer); at the
    check layer the fresh K/V of every row (the layer's own projections + RoPE) are compared with the
    linked cached K/V (standalone HF prefill of each chunk, keys re-based by complex rotation) by
    squared L2 (reading R10); the T = ⌈r·N_cached/100⌉ most deviating cached rows (ties: lower index,
    R13; the forced last row excluded, R11), every dynamic row and the last row are recomputed from the
    check layer on, attending to the cached K/V of all other rows (explicit position mask).  Returns
    (logits, selected rows, per-layer linked K)."""
    import torch
    m = hf_model(cfg, Wt)
    tok = np.concatenate([t for _, t in parts]).astype(np.int64)
    N = len(tok)
    pos = torch.arange(N)
    Kc = np.zeros((cfg.n_layers, cfg.n_kv_heads, N, cfg.head_dim))
    Vc = np.zeros_like(Kc)
    dyn = np.zeros(N, bool)
    s = 0
    for kind, t in parts:
        if kind == "tokens":
            dyn[s:s + len(t)] = True
        else:
            with torch.no_grad():
                alone = m(torch.from_numpy(t.astype(np.int64))[None], use_cache=True).past_key_values
            for l in range(cfg.n_layers):
                Kc[l, :, s:s + len(t)] = _complex_rebase(alone.layers[l].keys[0].numpy(), s, cfg)
                Vc[l, :, s:s + len(t)] = alone.layers[l].values[0].numpy()
        s += len(t)
    rot = m.model.rotary_emb

    def mask(qpos, kpos):
        ok = kpos[None, :] <= qpos[:, None]
        return torch.where(ok, 0.0, float("-inf")).to(torch.float64)[None, None]

    K = Kc.copy()
    with torch.no_grad():
        h = m.model.embed_tokens(torch.from_numpy(tok)[None])
        sel = np.arange(N)
        for l, layer in enumerate(m.model.layers):
            if l == check_layer:
                x = layer.input_layernorm(h)
                cs, sn = rot(x, pos[None])
                k_new = layer.self_attn.k_proj(x).view(1, N, cfg.n_kv_heads, cfg.head_dim).transpose(1, 2)
                v_new = layer.self_attn.v_proj(x).view(1, N, cfg.n_kv_heads, cfg.head_dim).transpose(1, 2)
                _, k_new = _hf_rope(k_new, k_new, cs, sn)
                dev = ((k_new[0].numpy() - Kc[l]) ** 2).sum(axis=(0, 2)) + ((v_new[0].numpy() - Vc[l]) ** 2).sum(axis=(0, 2))
                n_cached = int((~dyn).sum())
                T = (r_pct * n_cached + 99) // 100
                cand = sorted((i for i in range(N) if not dyn[i] and i != N - 1), key=lambda i: (-dev[i], i))[:T]
                sel = np.asarray(sorted(set(cand) | set(np.nonzero(dyn)[0].tolist()) | {N - 1}))
                h = h[:, torch.from_numpy(sel)]
            unsel = np.setdiff1d(np.arange(N), sel)
            cache = _PrefixKV(torch.from_numpy(Kc[l][:, unsel][None].copy()), torch.from_numpy(Vc[l][:, unsel][None].copy()))
            qpos = pos[torch.from_numpy(sel)]
            cs, sn = rot(h, qpos[None])
            x = layer.input_layernorm(h)
            kq = layer.self_attn.k_proj(x).view(1, len(sel), cfg.n_kv_heads, cfg.head_dim).transpose(1, 2)
            _, kq = _hf_rope(kq, kq, cs, sn)
            K[l][:, sel] = kq[0].numpy()
            h = layer(h, attention_mask=mask(qpos, torch.cat([pos[torch.from_numpy(unsel)], qpos])), past_key_values=cache,
                      position_embeddings=(cs, sn))
            if isinstance(h, tuple):
                h = h[0]
        logits = m.lm_head(m.model.norm(h))[0, -1].numpy()
    return logits, sel, [K[l].transpose(1, 0, 2) for l in range(cfg.n_layers)]


def _hf_rope(q, k, cos, sin):
    from transformers.models.llama.modeling_llama import apply_rotary_pos_emb
    return apply_rotary_pos_emb(q, k, cos, sin)


@pytest.mark.parametrize("cfg", [sg.TINY, sg.TINY_GQA, sg.TINY_D128], ids=lambda c: c.name)
@pytest.mark.parametrize("r_pct", [15, 40])
def test_C19_cacheblend_equals_hf_layerwise_construction(cfg, r_pct):
    """Pins CacheBlend with a real selection (previously 'parity unpinned'): the selected set, the
    logits and every layer's linked K equal the HF construction above, canonical and permuted orders."""
    w = sg.cfg1(model=cfg)
    Wt = M.Weights(cfg)
    store = P.Store(Wt)
    ids = store.compile(w.chunks)
    q = w.requests[0][-1].tokens
    for order in ([0, 1, 2, "q"], ["q", 2, 0, 1]):
        segs = [("tokens", q) if c == "q" else ("cached", ids[c]) for c in order]
        parts = [("tokens", q) if c == "q" else ("chunk", w.chunks[c]) for c in order]
        r = P.link(store, segs, f"cacheblend:{r_pct}")
        logits, sel, K = hf_cacheblend(cfg, Wt, parts, r_pct)
        assert np.array_equal(r.sel_per_layer[-1], sel)
        assert 0 < len(sel) < r.plan.N
        assert rel(r.logits, logits) < HF_TOL
        for l in range(cfg.n_layers):
            assert rel(r.K[l], K[l]) < HF_TOL, l
