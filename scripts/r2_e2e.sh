#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_link.py -q -k "caller_buffers or batched" > gpurun_out/e2e_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/e2e_tests.log)"; grep -A15 "^E " gpurun_out/e2e_tests.log | head -20
for i in 1 2; do
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/e2e.json 2> gpurun_out/e2e.err
python -c "import json;d=json.loads(open('gpurun_out/e2e.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), round(d['value']), round(d['e2e']['value']), d['e2e']['ms_per_step_host'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/e2e.err
done
