#!/bin/bash
# kv_share 3 with the Q-side re-base (QROT): tests and cfg4 bench vs kv_share 1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
true
true
for ks in 3 1 3 1; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share $ks > gpurun_out/qr.json 2> gpurun_out/qr.err
  python -c "import json;d=json.loads(open('gpurun_out/qr.json').read().strip().splitlines()[-1]);print('ks=$ks', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/qr.err
done
