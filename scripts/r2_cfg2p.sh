#!/bin/bash
# cfg2 / cfg3 / cfg5: persistent QROT attention (default) vs one CTA per item (PIC_NO_ATTN_PERSIST=1)
cd $GRAFT_REPO_ROOT
for C in cfg2 cfg3; do
for r in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_NO_ATTN_PERSIST=1; else unset PIC_NO_ATTN_PERSIST; fi
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --decode-steps 0 > gpurun_out/c2.json 2> gpurun_out/c2.err
  python -c "import json;d=json.loads(open('gpurun_out/c2.json').read().strip().splitlines()[-1]);print('$C no_persist=$v', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/c2.err
done
done
done
unset PIC_NO_ATTN_PERSIST
