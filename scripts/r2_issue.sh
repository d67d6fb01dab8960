#!/bin/bash
# convergent elect.sync MMA issue in the GEMM and one-lane attention: tests + cfg4 bench + cfg2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_share.py -x -q -k "attention or shared" > gpurun_out/is_t.log 2>&1; tail -1 gpurun_out/is_t.log
for i in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/is.json 2> gpurun_out/is.err
python -c "import json;d=json.loads(open('gpurun_out/is.json').read().strip().splitlines()[-1]);print('cfg4', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/is.err
done
timeout 900 python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu-baseline --decode-steps 0 > gpurun_out/is2.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/is2.json').read().strip().splitlines()[-1]);print('cfg2', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernel_breakdown'].items()})"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share 0 > gpurun_out/is3.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/is3.json').read().strip().splitlines()[-1]);print('cfg4 copy', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])"
