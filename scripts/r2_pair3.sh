#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused.py tests/test_gpu_parity_bench.py tests/test_gpu_link.py -x -q > gpurun_out/pa_t.log 2>&1; tail -1 gpurun_out/pa_t.log
for v in def nopf def nopf; do
  unset PIC_NO_PAIR_FUSED
  if [ $v = nopf ]; then export PIC_NO_PAIR_FUSED=1; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/pa.json 2> gpurun_out/pa.err
  python -c "import json;d=json.loads(open('gpurun_out/pa.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pa.err
done
