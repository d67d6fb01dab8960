mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 60 --timeout_method thread 2>&1 | tail -2
timeout 600 python -m pytest tests/ -m gpu -q -x --timeout 300 --timeout_method thread 2>&1 | tail -2
for c in cfg2 cfg3 cfg4; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c ms/step %.3f tok/s %.0f'%(d['ms_per_step'], d['value']), d['roofline']['bound'], '%.1f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']), {k: round(v['ms_per_step'],3) for k,v in d['kernel_breakdown'].items()})"
done
