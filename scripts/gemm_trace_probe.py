import sys; sys.path.insert(0, '/root/repo')
from paper_2410_15332_b200 import pic as B
for (M,N,K,bn,sp) in [(128,6144,4096,128,3),(128,4096,4096,128,4),(128,4096,14336,128,4)]:
    print(M,N,K,bn,sp, B.bench_gemm(M,N,K,bn,sp,iters=30), flush=True)
