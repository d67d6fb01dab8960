#!/bin/bash
# persistent QROT attention: O epilogue by the rotation warps (default) vs by the softmax warps (libpic_nooff.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qrot.py "tests/test_gpu_fullsize.py::test_fullsize_qrot_persistent_bit_identical" "tests/test_gpu_fullsize.py::test_fullsize_chunkframe_qrot_link" -q -x > gpurun_out/off_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/off_tests.log)"; grep -B2 -A10 "^E " gpurun_out/off_tests.log | head -30
for r in 1 2; do
for L in libpic.so libpic_nooff.so; do
  PIC_LIB_NAME=$L timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/off.json 2> gpurun_out/off.err
  python -c "import json;d=json.loads(open('gpurun_out/off.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/off.err
done
done
