#!/bin/bash
# kv_share 2 (V by reference, re-based key copies): tests, cfg4 bench vs kv_share 1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_share.py tests/test_gpu_fullsize.py tests/test_gpu_decode.py tests/test_gpu_link.py tests/test_gpu_fp32debug.py -x -q > gpurun_out/vs_t.log 2>&1; tail -1 gpurun_out/vs_t.log
for ks in 2 1 2 1; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share $ks > gpurun_out/vs.json 2> gpurun_out/vs.err
  python -c "import json;d=json.loads(open('gpurun_out/vs.json').read().strip().splitlines()[-1]);print('ks=$ks', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/vs.err
done
