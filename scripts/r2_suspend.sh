#!/bin/bash
# mbarrier try_wait with a suspend-time hint (libpic_s.so) vs plain spin (libpic.so): cfg4 step A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PIC_LIB_NAME=libpic_s.so timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > gpurun_out/su_t.log 2>&1; tail -1 gpurun_out/su_t.log
for lib in libpic_s.so libpic.so libpic_s.so libpic.so; do
  PIC_LIB_NAME=$lib timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/su.json 2> gpurun_out/su.err
  python -c "import json;d=json.loads(open('gpurun_out/su.json').read().strip().splitlines()[-1]);print('$lib', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/su.err
done
