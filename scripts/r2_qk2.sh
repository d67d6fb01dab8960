#!/bin/bash
# QROT with R(-Δ)Q in smem and a 2-slot K / 3-slot V ring (libpic_smk2*.so) vs TMEM QROT (default)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PIC_LIB_NAME=libpic_smk2.so timeout 900 python -m pytest tests/test_gpu_qrot.py "tests/test_gpu_fullsize.py::test_fullsize_chunkframe_qrot_link" -q > gpurun_out/qk2_tests.log 2>&1
echo "smk2 tests rc=$? $(tail -1 gpurun_out/qk2_tests.log)"; grep "^FAILED" gpurun_out/qk2_tests.log | head -3
for r in 1 2; do
for L in libpic.so libpic_smk2.so libpic_smk2w2.so; do
  PIC_LIB_NAME=$L timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/qk2.json 2> gpurun_out/qk2.err
  python -c "import json;d=json.loads(open('gpurun_out/qk2.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/qk2.err
done
done
PIC_LIB_NAME=libpic_phsmk2.so PIC_ATTN_TRACE=1 timeout 600 python scripts/attn_trace4.py 16 2 3 > gpurun_out/trace_phsmk2.log 2>&1
echo "== smem QROT K2/V3 4 warps"; grep "^---\|per-tile\|softmax cycles\|arrive ->" gpurun_out/trace_phsmk2.log | tail -13
