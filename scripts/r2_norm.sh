#!/bin/bash
# fused RMSNorm across GEMM boundaries: tests, bench A/B (cfg4 shared default, cfg3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fused.py -x -q -s > gpurun_out/norm_tests.log 2>&1; tail -3 gpurun_out/norm_tests.log; grep "fused-norm" gpurun_out/norm_tests.log
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_NO_NORM_FUSE=1; else unset PIC_NO_NORM_FUSE; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/norm.json 2> gpurun_out/norm.err
  python -c "import json;d=json.loads(open('gpurun_out/norm.json').read().strip().splitlines()[-1]);print('cfg4 nonormfuse=$v', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/norm.err
done
