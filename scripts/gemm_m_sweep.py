"""Does activation (A) traffic limit weight streaming?  Same weights, M in {1, 32, 64, 128}."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_15332_b200 import pic as B

for name, N, K, bn, s in (("down", 4096, 14336, 128, 4), ("gateup", 28672, 4096, 256, 1), ("qkv", 6144, 4096, 128, 3)):
    for M in (1, 32, 64, 128):
        us = B.bench_gemm(M, N, K, bn, s, 30)
        print(f"{name} M={M:3d} bn={bn} s={s} {us:7.2f} us  weights {N*K*2/us/1e3:6.0f} GB/s", flush=True)
