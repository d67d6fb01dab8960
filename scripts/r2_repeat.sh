#!/bin/bash
# three back-to-back runs of the driver's bench command on one box (run-to-run spread)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/rep
for i in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/rep/bench_$i.json 2> gpurun_out/rep/bench_$i.err
  python -c "import json;d=json.loads(open('gpurun_out/rep/bench_$i.json').read().strip().splitlines()[-1]);print('run $i', round(d['ms_per_step'],2), round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['decode']['tpot_ms'])"
done
