timeout 1200 python -m pytest tests/test_gpu_legolink0.py -q -x --timeout 900 --timeout_method thread 2>&1 | tail -15
