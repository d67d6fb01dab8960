#!/bin/bash
# full GPU suite, then cfg4 copy (side-stream a2 at 148 CTAs) vs shared, and the no-overlap copy path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab3_suite.log 2>&1; tail -3 gpurun_out/ab3_suite.log
for v in "0" "1" "0 nooverlap"; do
  set -- $v
  if [ "$2" = nooverlap ]; then export PIC_NO_K2_OVERLAP=1; else unset PIC_NO_K2_OVERLAP; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share $1 > gpurun_out/ab3.json 2> gpurun_out/ab3.err
  python -c "import json;d=json.loads(open('gpurun_out/ab3.json').read().strip().splitlines()[-1]);print('cfg4 ks=$v', round(d['ms_per_step'],2), round(d['value']), {k:(round(v['ms_per_step'],2), round(v['GB/s'])) for k,v in d['kernel_breakdown'].items()})" || tail -5 gpurun_out/ab3.err
done
