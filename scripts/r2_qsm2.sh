#!/bin/bash
# persistent QROT attention: R(-Δ)Q in smem (libpic_qsm.so, SS MMA, 2-slot V ring) vs TMEM (default)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PIC_LIB_NAME=libpic_qsm.so timeout 900 python -m pytest tests/test_gpu_qrot.py "tests/test_gpu_fullsize.py::test_fullsize_qrot_persistent_bit_identical" "tests/test_gpu_fullsize.py::test_fullsize_chunkframe_qrot_link" -q > gpurun_out/qsm2_tests.log 2>&1
echo "qsm tests rc=$? $(tail -1 gpurun_out/qsm2_tests.log)"; grep "^FAILED" gpurun_out/qsm2_tests.log | head -5
for r in 1 2; do
for L in libpic.so libpic_qsm.so; do
  PIC_LIB_NAME=$L timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/qsm2.json 2> gpurun_out/qsm2.err
  python -c "import json;d=json.loads(open('gpurun_out/qsm2.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/qsm2.err
done
done
