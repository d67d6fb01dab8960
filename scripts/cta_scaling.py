"""Does weight-stream bandwidth scale with the number of streaming CTAs (per-SM limit) or saturate (HBM)?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_15332_b200 import pic as B

K = 8192
for tiles in (64, 96, 112, 128, 136, 144, 148):
    N = tiles * 128
    us = B.bench_gemm(128, N, K, 128, 1, 50)
    print(f"ctas={tiles:4d} N={N} K={K} {us:7.2f} us  {N*K*2/us/1e3:6.0f} GB/s  per-CTA {N*K*2/us/1e3/tiles:5.1f} GB/s", flush=True)
