#!/bin/bash
# persistent QROT attention (attention_qp.cu): bit-identity tests, QROT tests, cfg4 bench A/B vs one CTA per item
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qrot.py "tests/test_gpu_fullsize.py::test_fullsize_qrot_persistent_bit_identical" "tests/test_gpu_fullsize.py::test_fullsize_chunkframe_qrot_link" -q -x > gpurun_out/qp_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/qp_tests.log)"; grep -B3 -A12 "^E " gpurun_out/qp_tests.log | head -40
for r in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_NO_ATTN_PERSIST=1; else unset PIC_NO_ATTN_PERSIST; fi
  timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/qp.json 2> gpurun_out/qp.err
  python -c "import json;d=json.loads(open('gpurun_out/qp.json').read().strip().splitlines()[-1]);print('no_persist=$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/qp.err
done
done
unset PIC_NO_ATTN_PERSIST
