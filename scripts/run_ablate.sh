timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2
PIC_ATTN_TRACE=1 timeout 300 python scripts/attn_trace.py 2>&1 | tail -15
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 2>&1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])"
