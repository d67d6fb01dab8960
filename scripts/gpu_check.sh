timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k long_context --timeout 1400 --timeout_method thread 2>&1 | tail -5
