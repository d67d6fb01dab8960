#!/bin/bash
# kv_link v2 + v2 attention for non-rotating links: tests, cfg4/cfg2 bench copy vs shared
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_link.py tests/test_gpu_share.py tests/test_gpu_legolink0.py tests/test_gpu_decode.py -x -q > gpurun_out/ab2_tests.log 2>&1; tail -2 gpurun_out/ab2_tests.log
for ks in 0 1; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share $ks > gpurun_out/ab2_ks$ks.json 2> gpurun_out/ab2_ks$ks.err
  python -c "import json;d=json.loads(open('gpurun_out/ab2_ks$ks.json').read().strip().splitlines()[-1]);print('cfg4 ks=$ks', round(d['ms_per_step'],2), round(d['value']), {k:(round(v['ms_per_step'],2), round(v['GB/s'])) for k,v in d['kernel_breakdown'].items()})" || tail -5 gpurun_out/ab2_ks$ks.err
  timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu-baseline --decode-steps 0 --kv-share $ks > gpurun_out/ab2_cfg2_ks$ks.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab2_cfg2_ks$ks.json').read().strip().splitlines()[-1]);print('cfg2 ks=$ks', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernel_breakdown'].items()})" || tail -3 gpurun_out/ab2_cfg2_ks$ks.json
done
