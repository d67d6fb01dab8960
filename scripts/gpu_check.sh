timeout 300 python scripts/gemm_m_sweep.py 2>&1
