PIC_CHAIN=1 timeout 900 python -m pytest tests/test_gpu_link.py tests/test_gpu_fullsize.py tests/test_gpu_decode.py -q -x --timeout 600 --timeout_method thread 2>&1 | tail -2
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('default', json.loads(sys.stdin.read())['ms_per_step'])"
