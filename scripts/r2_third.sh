#!/bin/bash
# fused epilogues + direct attention output: GPU suite, then bench A/B (fused vs separate kernels)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_kernels.py tests/test_gpu_link.py -x -q > gpurun_out/r3_quick.log 2>&1
tail -3 gpurun_out/r3_quick.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 0"
for v in 0 1 0; do
  if [ $v = 1 ]; then export PIC_NO_EPI_FUSE=1; else unset PIC_NO_EPI_FUSE; fi
  timeout 600 $B > gpurun_out/r3_bench_nofuse$v.json 2> gpurun_out/r3_bench_nofuse$v.err
  python -c "import json;d=json.loads(open('gpurun_out/r3_bench_nofuse$v.json').read().strip().splitlines()[-1]);print('nofuse=$v', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()})"
done
unset PIC_NO_EPI_FUSE
timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu-baseline --decode-steps 0 > gpurun_out/r3_cfg2.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/r3_cfg2.json').read().strip().splitlines()[-1]);print('cfg2', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernel_breakdown'].items()})"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3_gpu_all.log 2>&1
tail -3 gpurun_out/r3_gpu_all.log
