"""Attention kernel error vs fp64 (bench-only debug): rel-L2 of the v2 kernel on random inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import seedgen as sg
from oracle import model as M
from paper_2410_15332_b200 import pic as B

def rand_bf16(seed, shape):
    u = sg.U(seed, 1, np.arange(int(np.prod(shape)), dtype=np.uint64))
    f = ((u >> np.uint64(40)).astype(np.float64) / 2**24 * 2 - 1).astype(np.float32)
    return (f.view(np.uint32) >> 16).astype(np.uint16).reshape(shape)
f32 = lambda b: (b.astype(np.uint32) << 16).view(np.float32)
for (Hq, Hkv, n, M_) in [(32, 8, 2624, 128), (32, 8, 1000, 64)]:
    Q = rand_bf16(1, (M_, Hq, 128)); K = rand_bf16(2, (n, Hkv, 128)); V = rand_bf16(3, (n, Hkv, 128))
    pos = np.sort(np.random.default_rng(0).choice(n, M_, replace=False)).astype(np.int32)
    nb = (n + 15) // 16
    perm = np.arange(nb, dtype=np.int32)
    ref = M.causal_attention(f32(Q), f32(K), f32(V), pos)
    for v in (1, 2):
        got = f32(B.test_attention(Q, K, V, pos, perm, nb + 4, 1, version=v))
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        print(f"Hq={Hq} n={n} M={M_} version {v}: rel-L2 {err:.3e}")
