timeout 300 python scripts/gemm_m_sweep.py 2>&1 | grep "M=128"
PIC_BENCH_PACK=128 timeout 300 python scripts/gemm_m_sweep.py 2>&1 | grep "M=128"
PIC_BENCH_PACK=64 timeout 300 python scripts/gemm_m_sweep.py 2>&1 | grep "M=128"
