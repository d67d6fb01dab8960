#!/bin/bash
# ping-pong attention (attention_pp.cu): kernel parity, engine parity, cfg4/cfg2 bench A/B vs the one-lane kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/pp_kern.log 2>&1
tail -5 gpurun_out/pp_kern.log
timeout 900 python -m pytest tests/test_gpu_link.py tests/test_gpu_share.py tests/test_gpu_fused.py -x -q > gpurun_out/pp_link.log 2>&1
tail -5 gpurun_out/pp_link.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 0"
for v in 2 1 2; do
  if [ $v = 1 ]; then export PIC_ATTN_V1=1; else unset PIC_ATTN_V1; fi
  timeout 600 $B > gpurun_out/pp_bench_v$v.json 2> gpurun_out/pp_bench_v$v.err
  python -c "import json;d=json.loads(open('gpurun_out/pp_bench_v$v.json').read().strip().splitlines()[-1]);print('v=$v', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()})" || tail -5 gpurun_out/pp_bench_v$v.err
done
for v in 2 1; do
  if [ $v = 1 ]; then export PIC_ATTN_V1=1; else unset PIC_ATTN_V1; fi
  timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu-baseline --decode-steps 0 > gpurun_out/pp_cfg2_v$v.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/pp_cfg2_v$v.json').read().strip().splitlines()[-1]);print('cfg2 v=$v', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernel_breakdown'].items()})" || tail -5 gpurun_out/pp_cfg2_v$v.json
done
