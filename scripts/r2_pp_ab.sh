#!/bin/bash
# cfg4 bench: shared-block link vs copy path (per-layer side-stream a2), v2 attention; link parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_link.py tests/test_gpu_share.py tests/test_gpu_fused.py tests/test_gpu_parity_bench.py -x -q > gpurun_out/ab_tests.log 2>&1; tail -2 gpurun_out/ab_tests.log
for ks in 0 1; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share $ks > gpurun_out/ab_ks$ks.json 2> gpurun_out/ab_ks$ks.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_ks$ks.json').read().strip().splitlines()[-1]);print('cfg4 ks=$ks', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()})" || tail -5 gpurun_out/ab_ks$ks.err
done
