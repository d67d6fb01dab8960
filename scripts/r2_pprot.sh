#!/bin/bash
# ping-pong kernel with the rotation warpgroup (shared-block link): parity, trace, bench with it forced
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_share.py -x -q -k "attention or shared" > gpurun_out/pr_t.log 2>&1; tail -1 gpurun_out/pr_t.log
for ks in 0 1; do
PIC_ATTN_PP_ROT=1 PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share $ks > gpurun_out/pr_tr$ks.log 2>&1
echo "== ks $ks"; grep "attn_pp" gpurun_out/pr_tr$ks.log | tail -21 | grep -v " 0 (0.0%\|steps\|items\|Q-empty\|wait Q\|O-free\|epilogue"
done
for v in 1 0; do
  if [ $v = 1 ]; then export PIC_ATTN_PP_ROT=1; else unset PIC_ATTN_PP_ROT; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/pr.json 2> gpurun_out/pr.err
  python -c "import json;d=json.loads(open('gpurun_out/pr.json').read().strip().splitlines()[-1]);print('cfg4 pprot=$v', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/pr.err
done
