#!/bin/bash
# CTA-pair residual / QKV GEMMs (PIC_PAIR_FUSED=1) vs one-CTA (default) on the session-3 build
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_PAIR_FUSED=1; else unset PIC_PAIR_FUSED; fi
  timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/pf.json 2> gpurun_out/pf.err
  python -c "import json;d=json.loads(open('gpurun_out/pf.json').read().strip().splitlines()[-1]);print('pair_fused=$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pf.err
done
done
