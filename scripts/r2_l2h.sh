#!/bin/bash
# GEMM L2 policy A/B (PIC_GEMM_L2HINT: activations evict_last + weights evict_first for unsplit GEMMs whose
# A fits in L2): GEMM tests, cfg4 bench alternating, per-GEMM DRAM bytes of one wave-layer under ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PIC_GEMM_L2HINT=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused.py -q -x > gpurun_out/l2h_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/l2h_tests.log)"
for r in 1 2; do
for h in 0 1; do
  PIC_GEMM_L2HINT=$h timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/l2h.json 2> gpurun_out/l2h.err
  python -c "import json;d=json.loads(open('gpurun_out/l2h.json').read().strip().splitlines()[-1]);print('hint=$h', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/l2h.err
done
done
for h in 0 1; do
  PIC_GEMM_L2HINT=$h timeout 900 ncu --profile-from-start off --clock-control none -k regex:gemm -c 4 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --csv python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/l2h_ncu_$h.csv 2> gpurun_out/l2h_ncu_$h.err
  echo "== hint=$h"; grep -o '"[a-z_]*gemm[^"]*"\|"dram__bytes_[a-z]*.sum","[A-Za-z]*","[0-9.,]*"\|"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/l2h_ncu_$h.csv | head -24
done
