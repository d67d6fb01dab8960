#!/bin/bash
# skinny GEMMs (one m-tile: decode batch 32, cfg2) unsplit with fused epilogues (PIC_SKINNY_NOSPLIT=1) vs split-K
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PIC_SKINNY_NOSPLIT=1 timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_link.py -q -x > gpurun_out/sk_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/sk_tests.log)"
for r in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_SKINNY_NOSPLIT=1; else unset PIC_SKINNY_NOSPLIT; fi
  timeout 600 python scripts/decode_profile.py 32 32 > gpurun_out/sk.log 2>&1; echo "nosplit=$v $(head -1 gpurun_out/sk.log)"
  timeout 900 python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu-baseline --decode-steps 16 > gpurun_out/sk.json 2> gpurun_out/sk.err
  python -c "import json;d=json.loads(open('gpurun_out/sk.json').read().strip().splitlines()[-1]);print('cfg2 nosplit=$v', round(d['ms_per_step'],3), d['decode']['tpot_ms'], {k:round(v['ms_per_step'],3) for k,v in d['kernel_breakdown'].items()})" || tail -3 gpurun_out/sk.err
done
done
unset PIC_SKINNY_NOSPLIT
