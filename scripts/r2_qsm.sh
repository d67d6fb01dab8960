#!/bin/bash
# QROT with R(-Δ)Q in smem (SS MMA, default build) vs in TMEM (TS MMA, libpic_qtm.so): new QROT tests,
# cfg4 bench A/B on one box, attention trace of both
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qrot.py "tests/test_gpu_fullsize.py::test_fullsize_chunkframe_qrot_link" -q > gpurun_out/qsm_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/qsm_tests.log)"; grep "^FAILED" gpurun_out/qsm_tests.log | head
for L in libpic.so libpic_qtm.so libpic.so libpic_qtm.so; do
  PIC_LIB_NAME=$L timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/qsm.json 2> gpurun_out/qsm.err
  python -c "import json;d=json.loads(open('gpurun_out/qsm.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/qsm.err
done
for L in libpic.so libpic_qtm.so; do
  PIC_LIB_NAME=$L PIC_ATTN_TRACE=1 timeout 600 python scripts/attn_trace4.py 16 2 3 > gpurun_out/trace_$L.log 2>&1
  echo "== $L"; grep "per-tile\|softmax cycles\|arrive ->\|frames" gpurun_out/trace_$L.log | tail -12
done
