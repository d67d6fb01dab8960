timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 60 --timeout_method thread 2>&1 | tail -3
timeout 600 python -m pytest tests/ -m gpu -q -x --timeout 300 --timeout_method thread 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'tok/s', d['value']); print(d['roofline']['frac']); [print(k, v) for k,v in d['kernel_breakdown'].items()]"
