"""Attention kernel timing vs KV length (fixed cost + per-KV-tile cost)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_15332_b200 import pic as B

rng = np.random.default_rng(0)
for Hq, Hkv, M in ((4, 1, 32), (32, 8, 32), (32, 8, 128)):
    for nt in (1, 2, 4, 8, 16):
        n = 128 * nt
        Q = (rng.integers(0, 1 << 14, (M, Hq, 128)) | 0x3c00).astype(np.uint16) & 0xBFFF
        K = (rng.integers(0, 1 << 14, (n, Hkv, 128)) | 0x3c00).astype(np.uint16) & 0xBFFF
        V = K.copy()
        pos = np.arange(n - M, n)
        nb = n // 16
        perm = np.arange(nb) if os.environ.get("CONTIG", "1") == "1" else np.argsort(rng.random(nb))
        us = B.bench_attention(Q, K, V, pos, perm, nb, 1, 30)
        print(f"Hq={Hq} Hkv={Hkv} M={M} kv_tiles={nt:3d} {us:8.2f} us  ({us/nt:.2f} us/tile)", flush=True)
