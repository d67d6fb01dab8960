#!/bin/bash
# QROT variants: R(-Δ)Q in TMEM (default, 4 warps) vs smem with 4 / 2 / 1 rotation warps; tests, cfg4 A/B,
# per-phase softmax traces (PIC_ATTN_PHASES builds) of copy / TMEM QROT / smem QROT 1 warp
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in libpic_sm2.so libpic_sm1.so; do
  PIC_LIB_NAME=$L timeout 900 python -m pytest tests/test_gpu_qrot.py "tests/test_gpu_fullsize.py::test_fullsize_chunkframe_qrot_link" -q > gpurun_out/qw_tests.log 2>&1
  echo "$L tests rc=$? $(tail -1 gpurun_out/qw_tests.log)"; grep "^FAILED" gpurun_out/qw_tests.log | head -3
done
for r in 1 2; do
for L in libpic.so libpic_sm4.so libpic_sm2.so libpic_sm1.so; do
  PIC_LIB_NAME=$L timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/qw.json 2> gpurun_out/qw.err
  python -c "import json;d=json.loads(open('gpurun_out/qw.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/qw.err
done
done
PIC_LIB_NAME=libpic_ph.so PIC_ATTN_TRACE=1 timeout 600 python scripts/attn_trace4.py 16 2 0,3 > gpurun_out/trace_ph.log 2>&1
echo "== TMEM QROT build, modes 0 (copy) and 3"; grep "^---\|per-tile\|softmax cycles\|arrive ->" gpurun_out/trace_ph.log | tail -26
PIC_LIB_NAME=libpic_phsm1.so PIC_ATTN_TRACE=1 timeout 600 python scripts/attn_trace4.py 16 2 3 > gpurun_out/trace_phsm1.log 2>&1
echo "== smem QROT 1 warp"; grep "^---\|per-tile\|softmax cycles\|arrive ->" gpurun_out/trace_phsm1.log | tail -13
