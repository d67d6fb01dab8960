#!/bin/bash
# persistent QROT attention: exponential split (PIC_V1_POLY8 pairs of 8 on the FMA polynomial) 1 (default) vs 0/2/3
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for L in libpic.so libpic_p0.so libpic_p2.so libpic_p3.so; do
  PIC_LIB_NAME=$L timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/pq.json 2> gpurun_out/pq.err
  python -c "import json;d=json.loads(open('gpurun_out/pq.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pq.err
done
done
