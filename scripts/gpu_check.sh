timeout 1200 python -m pytest tests/ -m gpu -q -x --timeout 900 --timeout_method thread 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>gpurun_out/b2.err | tail -1 > gpurun_out/bench_cfg2.json
python -c "import json; d=json.load(open('gpurun_out/bench_cfg2.json')); print(d['ms_per_step'], d['value'], d['decode'], d['roofline']['frac'])"
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --decode-steps 16 2>gpurun_out/b4.err | tail -1 > gpurun_out/bench_cfg4.json
python -c "import json; d=json.load(open('gpurun_out/bench_cfg4.json')); print(d['ms_per_step'], d['value'], d['decode'])"
timeout 300 python bench.py --alg legolink0 --steps 20 --warmup 5 --no-cpu-baseline --decode-steps 0 2>gpurun_out/b0.err | tail -1 > gpurun_out/bench_cfg2_ll0.json
python -c "import json; d=json.load(open('gpurun_out/bench_cfg2_ll0.json')); print('legolink0', d['ms_per_step'], d['value'])"
