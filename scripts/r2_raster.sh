#!/bin/bash
# grouped GEMM raster for large-A GEMMs: down-proj DRAM traffic and step time
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_kernels.py -x -q -k "gemm or fused" > gpurun_out/ra_t.log 2>&1; tail -1 gpurun_out/ra_t.log
for i in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/ra.json 2> gpurun_out/ra.err
python -c "import json;d=json.loads(open('gpurun_out/ra.json').read().strip().splitlines()[-1]);print('cfg4', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/ra.err
done
N="ncu --profile-from-start off --clock-control none"
timeout 900 $N --set full -k regex:gemm -c 4 -o gpurun_out/ra_gemm python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/ra_g.log 2>&1
python scripts/ncu_detail.py gpurun_out/ra_gemm.ncu-rep > gpurun_out/ra_gemm.md 2>&1
grep -h "^## \|time_duration\|dram__bytes\|tensor_cycles" gpurun_out/ra_gemm.md
