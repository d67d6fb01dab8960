"""Kernel-level parity on a B200: each hot-path kernel through the C ABI (libpic.so) against
the fp64 oracle (or exact integer expectations) on the same seeded inputs."""
import numpy as np
import pytest

import seedgen as sg
from oracle import model as M
from oracle import pic as P
from paper_2410_15332_b200 import pic as B

pytestmark = pytest.mark.gpu


def bf16_bits(x):
    return (sg.bf16_rne(np.asarray(x, dtype=np.float32)).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def f32(bits):
    return B.bf16_bits_to_f32(bits).astype(np.float64)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def rand_bf16(seed, shape, scale=1.0):
    u = sg.uniform_pm1(sg.U(seed, 77, np.arange(int(np.prod(shape)), dtype=np.uint64))).reshape(shape)
    return bf16_bits(u * scale)


# ------------------------------------------------------------------ K15 generator (bit-exact)
@pytest.fixture(scope="module")
def tiny_engine():
    import torch  # noqa: F401
    eng = B.Engine(sg.TINY_D128, num_blocks=256, max_rows=512, max_tokens=1024, max_requests=4, device=0)
    yield eng
    eng.close()


@pytest.mark.parametrize("which,tag,rows,cols_attr", [
    (0, sg.TAG_Q, "q", None), (1, sg.TAG_K, "k", None), (2, sg.TAG_V, "v", None), (3, sg.TAG_O, "o", None),
    (4, sg.TAG_GATE, "gate", None), (5, sg.TAG_UP, "up", None), (6, sg.TAG_DOWN, "down", None)])
def test_weights_bit_exact(tiny_engine, which, tag, rows, cols_attr):
    cfg = sg.TINY_D128
    W = M.Weights(cfg)
    for l in range(cfg.n_layers):
        ref = W.layer(l)[rows].astype(np.float32)
        got = tiny_engine.read_weights(which, l, 0, ref.shape[0])
        assert np.array_equal(got, bf16_bits(ref)), (which, l)


def test_embed_lm_gains_bit_exact(tiny_engine):
    cfg = sg.TINY_D128
    W = M.Weights(cfg)
    assert np.array_equal(tiny_engine.read_weights(7, 0, 0, cfg.vocab), bf16_bits(W.embed))
    assert np.array_equal(tiny_engine.read_weights(8, 0, 0, cfg.vocab), bf16_bits(W.lm_head))
    assert np.array_equal(tiny_engine.read_weights(9, 1), W.layer(1)["g1"].astype(np.float32))
    assert np.array_equal(tiny_engine.read_weights(10, 0), W.layer(0)["g2"].astype(np.float32))
    assert np.array_equal(tiny_engine.read_weights(11), W.g_final.astype(np.float32))


# ------------------------------------------------------------------ tcgen05 GEMM
@pytest.mark.parametrize("M_,N_,K_,bn,splits", [
    (128, 256, 128, 128, 1), (100, 192, 64, 64, 1), (1, 512, 4096, 256, 3), (300, 512, 640, 128, 2),
    (128, 6144, 4096, 256, 6), (609, 256, 1024, 256, 1), (17, 96, 192, 64, 3),
    (96, 512, 256, 64, 2), (96, 512, 256, 256, 2),
    # CTA pair (cta_group::2, 256-row M-tiles; negative bn): ragged M, several units per pair, split-K
    (256, 512, 256, -256, 1), (609, 1024, 512, -256, 2), (300, 768, 640, -128, 1), (100, 384, 128, -192, 1),
    (1000, 448, 256, -224, 3), (3000, 2048, 256, -256, 1)])
def test_gemm_vs_fp64(M_, N_, K_, bn, splits):
    A = rand_bf16(M_ * 7 + K_, (M_, K_))
    Bm = rand_bf16(N_ * 3 + K_, (N_, K_), 0.05)
    got = B.test_gemm(A, Bm, bn, splits)
    ref = f32(A) @ f32(Bm).T
    assert rel(got, ref) < 1e-5, rel(got, ref)


@pytest.mark.parametrize("M_,F,K_,bn", [(128, 14336 // 8, 512, 224), (37, 256, 128, 64), (300, 512, 256, 256),
                                       (5, 64, 64, 32), (600, 14336 // 8, 512, -224), (300, 512, 256, -256)])
def test_gemm_swiglu_vs_fp64(M_, F, K_, bn):
    g = abs(bn) // 2
    A = rand_bf16(M_ + K_, (M_, K_))
    Wg = rand_bf16(F + 1, (F, K_), 0.05)
    Wu = rand_bf16(F + 2, (F, K_), 0.05)
    Bi = np.concatenate([np.concatenate([Wg[n * g:(n + 1) * g], Wu[n * g:(n + 1) * g]]) for n in range(F // g)])
    got = f32(B.test_gemm_swiglu(A, Bi, bn))
    a = f32(A)
    gate, up = a @ f32(Wg).T, a @ f32(Wu).T
    ref = gate / (1 + np.exp(-gate)) * up
    assert rel(got, ref) < 1e-2, rel(got, ref)


# ------------------------------------------------------------------ attention
@pytest.mark.parametrize("Hq,Hkv,n_keys,M_,splits", [
    (4, 4, 300, 40, 1), (8, 2, 257, 70, 2), (32, 8, 700, 128, 3), (64, 8, 1000, 33, 4), (8, 1, 130, 130, 1),
    (2, 1, 112, 96, 1), (2, 1, 2624, 128, 5)])
@pytest.mark.parametrize("version,grid,contig", [(2, 0, False), (2, 3, True), (1, 0, False)])
def test_attention_vs_oracle(Hq, Hkv, n_keys, M_, splits, version, grid, contig):
    """version 2 = the engine's persistent ping-pong kernel (grid 3: several items per CTA; contig: the
    8-block TMA box path), version 1 = one q-tile per CTA."""
    D = 128
    Q = rand_bf16(1 + Hq, (M_, Hq, D))
    K = rand_bf16(2 + Hq, (n_keys, Hkv, D))
    V = rand_bf16(3 + Hq, (n_keys, Hkv, D))
    # scattered sorted query positions including the ends
    u = sg.U(9, Hq, np.arange(M_, dtype=np.uint64))
    pos = np.unique(np.concatenate([[0, n_keys - 1], (u % np.uint64(n_keys)).astype(np.int64)]))[:M_]
    M_ = len(pos)
    Q = Q[:M_]
    nb = (n_keys + 15) // 16
    perm = np.argsort(sg.U(5, nb, np.arange(nb + 5, dtype=np.uint64)))[:nb].astype(np.int32)  # distinct ids
    if contig:
        perm = np.arange(2, nb + 2, dtype=np.int32)
    got = B.test_attention(Q, K, V, pos, perm, nb + 5, splits, version=version, grid=grid)
    ref = M.causal_attention(f32(Q), f32(K), f32(V), pos)
    assert rel(f32(got), ref) < 1e-2, rel(f32(got), ref)
    # per-row check too (a wrong causal limit shows up on one row)
    err = np.linalg.norm(f32(got) - ref, axis=(1, 2)) / np.linalg.norm(ref, axis=(1, 2))
    assert err.max() < 3e-2, (err.argmax(), err.max())


# ------------------------------------------------------------------ KV link (gather + re-base)
def test_kv_link_tags_and_rebase():
    L, NB, Hkv, D = 3, 12, 2, 128
    K = rand_bf16(11, (L, NB, Hkv, 16, D))
    V = np.arange(L * NB * Hkv * 16 * D, dtype=np.uint64).astype(np.uint16).reshape(L, NB, Hkv, 16, D)  # tags
    src = np.array([0, 5, 17, 33, 40, 47], dtype=np.int32)
    dst = np.array([100, 101, 130, 131, 150, 191], dtype=np.int32)
    delta = np.array([0, 0, 31, 512, 3000, 0], dtype=np.int32)
    K2, V2 = B.test_kv_link(K.copy(), V.copy(), src, dst, delta, layer0=1, theta=1e4, max_pos=4096)

    def row(a, l, s):
        return a[l, s // 16, :, s % 16, :]

    for l in range(L):
        for s, d, dl in zip(src, dst, delta):
            if l == 0:                                   # below layer0: untouched
                assert np.array_equal(row(K2, l, d), row(K, l, d))
                continue
            assert np.array_equal(row(V2, l, d), row(V, l, s))          # bit copy
            if dl == 0:
                assert np.array_equal(row(K2, l, d), row(K, l, s))      # Δ = 0 exact
            else:
                ref = P.rebase(f32(row(K, l, s))[None], int(dl), D, 1e4)[0]
                got = f32(row(K2, l, d))
                ulp = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)
                assert np.all((ulp <= 2 ** -7) | (np.abs(got - ref) < 1e-6)), ulp.max()
