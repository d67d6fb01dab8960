"""Traffic ablations of the GEMM (PIC_GEMM_DBG, set by the caller): weight-stream rate per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_15332_b200 import pic as B

dbg = os.environ.get("PIC_GEMM_DBG", "0")
cases = [("qkv", 128, 6144, 4096, 128, 3), ("o", 128, 4096, 4096, 128, 4), ("down", 128, 4096, 14336, 128, 4),
         ("gateup", 128, 28672, 4096, 256, 1), ("big128", 128, 18944, 8192, 128, 1), ("big256", 128, 37888, 4096, 256, 1),
         ("big64", 128, 9472, 16384, 64, 1)]
for name, M, N, K, bn, s in cases:
    us = B.bench_gemm(M, N, K, bn, s, 50)
    print(f"dbg={dbg} {name:7s} M={M} N={N} K={K} bn={bn} s={s} {us:8.2f} us  W {N*K*2/us/1e3:6.0f} GB/s  W+A/CTA {(N*K*2 + M*K*2*N//bn)/us/1e3:6.0f} GB/s", flush=True)
