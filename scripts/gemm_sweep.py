"""Sweep GEMM tile/split choices for the cfg2 link shapes (M = k' = 128) on a B200."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_15332_b200 import pic as B

shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gateup": (28672, 4096), "down": (4096, 14336), "lm": (32000, 4096)}
M = int(sys.argv[1]) if len(sys.argv) > 1 else 128
for name, (N, K) in shapes.items():
    best = None
    for bn in (64, 128, 256):
        for s in (1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 16):
            if s > K // 64:
                continue
            ctas = ((N + bn - 1) // bn) * ((M + 127) // 128) * s
            if ctas > 600:
                continue
            us = B.bench_gemm(M, N, K, bn, s, 30)
            gbs = (N * K * 2 + M * K * 2) / us / 1e3
            print(f"{name:7s} M={M} N={N} K={K} bn={bn:3d} s={s:2d} ctas={ctas:4d} {us:8.2f} us {gbs:7.0f} GB/s", flush=True)
            if best is None or us < best[0]:
                best = (us, bn, s, gbs)
    print(f"BEST {name}: bn={best[1]} s={best[2]} {best[0]:.2f} us {best[3]:.0f} GB/s", flush=True)
