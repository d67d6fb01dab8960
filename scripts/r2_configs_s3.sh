#!/bin/bash
# session-3 lines for the other configurations + the --gpus 2 self-spawn dry run (2 ranks sharing one GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3cfg
B="timeout 900 python bench.py --no-cpu-baseline"
$B --config cfg2 --steps 20 --warmup 5 > gpurun_out/s3cfg/cfg2.json 2> gpurun_out/s3cfg/cfg2.err
$B --config cfg3 --steps 10 --warmup 3 --decode-steps 0 > gpurun_out/s3cfg/cfg3_ll32.json 2> gpurun_out/s3cfg/cfg3_ll32.err
$B --config cfg3 --alg cacheblend:15 --steps 10 --warmup 3 --decode-steps 0 > gpurun_out/s3cfg/cfg3_cb15.json 2> gpurun_out/s3cfg/cfg3_cb15.err
$B --config cfg5 --steps 3 --warmup 3 --decode-steps 0 > gpurun_out/s3cfg/cfg5.json 2> gpurun_out/s3cfg/cfg5.err
$B --gpus 2 --requests 64 --steps 2 --warmup 3 --decode-steps 0 > gpurun_out/s3cfg/dp2_dry.json 2> gpurun_out/s3cfg/dp2_dry.err
$B --config cfg5 --gpus 2 --layers 4 --steps 2 --warmup 3 --decode-steps 0 > gpurun_out/s3cfg/tp2_dry.json 2> gpurun_out/s3cfg/tp2_dry.err
for f in cfg2 cfg3_ll32 cfg3_cb15 cfg5 dp2_dry tp2_dry; do
  python -c "
import json
d=json.loads(open('gpurun_out/s3cfg/$f.json').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step'],3), round(d['value']), d['n_gpus'], d['config'].get('parallelism'), d['config'].get('shared_gpu'), {k:round(v['ms_per_step'],3) for k,v in list(d['kernel_breakdown'].items())[:5]}, (d.get('decode') or {}).get('tpot_ms'))
" || (echo "$f failed"; tail -3 gpurun_out/s3cfg/$f.err)
done
