import sys; sys.path.insert(0, '/root/repo')
from paper_2410_15332_b200 import pic as B
for (M,N,K,bn) in [(6656,6144,4096,256),(1072,8192,8192,256),(1024,8192,8192,256),(1152,8192,8192,256),(1072,8192,4096,256),(1072,10240,8192,256),(4096,8192,8192,256),(1072,8192,28672,256)]:
    us = B.bench_gemm(M,N,K,bn,1,iters=20)
    print(M,N,K,bn, f"{us:.1f} us", f"{2*M*N*K/us/1e6:.0f} TFLOP/s", flush=True)
