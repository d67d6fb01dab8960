#!/bin/bash
# ncu --set full of the ping-pong attention at cfg4 (wave of 32, layer 0), shared and copy path; bench A/B copy path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N="ncu --profile-from-start off --clock-control none"
timeout 900 $N --set full --import-source on -k regex:attn_pp -c 1 -o gpurun_out/pp_attn_cfg4 python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/pp_ncu1.log 2>&1
timeout 900 $N --set full --import-source on -k regex:attn_pp -c 1 -o gpurun_out/pp_attn_cfg4_copy python scripts/ncu_link.py --config cfg4 --layers 2 --kv-share 0 > gpurun_out/pp_ncu2.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share 0"
for v in 2 1; do
  if [ $v = 1 ]; then export PIC_ATTN_V1=1; else unset PIC_ATTN_V1; fi
  timeout 600 $B > gpurun_out/pp_bench_copy_v$v.json 2> gpurun_out/pp_bench_copy_v$v.err
  python -c "import json;d=json.loads(open('gpurun_out/pp_bench_copy_v$v.json').read().strip().splitlines()[-1]);print('copy v=$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()})" || tail -5 gpurun_out/pp_bench_copy_v$v.err
done
