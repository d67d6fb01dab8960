timeout 900 python -m pytest tests/test_gpu_fp32debug.py -q -x --timeout 600 --timeout_method thread 2>&1 | tail -20
timeout 900 python -m pytest tests/ -m gpu -q -x --timeout 600 --timeout_method thread -k "not fullsize" 2>&1 | tail -3
