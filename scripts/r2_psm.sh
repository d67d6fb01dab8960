#!/bin/bash
# persistent QROT attention: P in smem + SS PV MMA (libpic_psm.so) vs P in TMEM (default)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PIC_LIB_NAME=libpic_psm.so timeout 900 python -m pytest tests/test_gpu_qrot.py "tests/test_gpu_fullsize.py::test_fullsize_qrot_persistent_bit_identical" -q > gpurun_out/psm_tests.log 2>&1
echo "psm tests rc=$? $(tail -1 gpurun_out/psm_tests.log)"; grep "^FAILED" gpurun_out/psm_tests.log | head -5; grep -m3 -A8 "^E " gpurun_out/psm_tests.log | head -20
for r in 1 2; do
for L in libpic.so libpic_psm.so; do
  PIC_LIB_NAME=$L timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/psm.json 2> gpurun_out/psm.err
  python -c "import json;d=json.loads(open('gpurun_out/psm.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/psm.err
done
done
