"""Skinny (k' = 128) weight-streaming GEMMs: N-tile / split-K pairs that fill ~148 SMs (random operands)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_15332_b200 import pic as B

for (N, K) in [(4096, 4096), (4096, 14336), (6144, 4096)]:
    for bn, sp in [(128, 148 // ((N + 127) // 128)), (144, 5), (176, 6), (208, 7), (256, 9), (256, 6), (192, 6), (160, 5)]:
        tiles = (N + bn - 1) // bn
        if tiles * sp > 148 or sp > K // 256:
            continue
        try:
            us = B.bench_gemm(128, N, K, bn, sp, iters=50)
            print(N, K, bn, sp, tiles * sp, f"{us:.2f} us", f"{(N * K * 2) / us / 1e3:.0f} GB/s", flush=True)
        except Exception as e:
            print(N, K, bn, sp, "ERR", e, flush=True)
