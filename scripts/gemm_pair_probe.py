"""One-CTA (M = 128) vs CTA-pair (cta_group::2, M = 256) tcgen05 GEMM on the link's tensor-bound shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_15332_b200 import pic as B

for (M, N, K) in [(6656, 6144, 4096), (6656, 4096, 4096), (6656, 4096, 14336), (1072, 8192, 8192), (608, 4096, 4096),
                  (2048, 6144, 4096)]:
    for bn in (256, -256, -192, -128):
        try:
            us = B.bench_gemm(M, N, K, bn, 1, iters=20)
            print(M, N, K, bn, f"{us:.1f} us", f"{2 * M * N * K / us / 1e6:.0f} TFLOP/s", flush=True)
        except Exception as e:
            print(M, N, K, bn, "ERR", e, flush=True)
