#!/bin/bash
# CTA-pair gate/up GEMM: grouped m-unit raster (PIC_PAIR_RASTER = group size) vs m-fastest (default)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PIC_PAIR_RASTER=8 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused.py -q -x > gpurun_out/pr_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/pr_tests.log)"
for g in 8 0 4; do
  PIC_PAIR_RASTER=$g timeout 900 ncu --profile-from-start off --clock-control none -k regex:gemm_pair -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum --csv python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/pr_ncu_$g.csv 2>/dev/null
  echo "raster=$g $(grep -o '"dram__bytes_read.sum","[a-zA-Z]*","[0-9.,]*"\|"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/pr_ncu_$g.csv | tr '\n' ' ')"
done
for r in 1 2; do
for g in 0 8; do
  PIC_PAIR_RASTER=$g timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/pr.json 2> gpurun_out/pr.err
  python -c "import json;d=json.loads(open('gpurun_out/pr.json').read().strip().splitlines()[-1]);print('raster=$g', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pr.err
done
done
