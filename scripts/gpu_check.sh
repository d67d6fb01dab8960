timeout 900 python -m pytest tests/test_gpu_decode.py -q -x --timeout 800 --timeout_method thread 2>&1 | tail -5
