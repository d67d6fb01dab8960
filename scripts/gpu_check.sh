timeout 600 python -m pytest tests/test_serve.py -q -x --timeout 500 --timeout_method thread 2>&1 | tail -3
timeout 1500 python scripts/serve_sweep.py --out gpurun_out/serve_r1.md 2>&1 | tail -32
