timeout 900 python -m pytest tests/test_gpu_edges.py -q -x --timeout 600 --timeout_method thread 2>&1 | tail -15
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 1400 --timeout_method thread 2>&1 | tail -15
