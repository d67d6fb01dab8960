#!/bin/bash
# f1 decode attention kernel: tests, decode breakdown new vs old kernel, bench TPOT
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode_attn.py tests/test_gpu_decode.py -q -x > gpurun_out/da_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/da_tests.log)"; grep -B5 "Error\|assert" gpurun_out/da_tests.log | head -40
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_NO_ATTN_DECODE=1; else unset PIC_NO_ATTN_DECODE; fi
  timeout 600 python scripts/decode_profile.py 32 8 > gpurun_out/da_prof_$v.log 2>&1; echo "== PIC_NO_ATTN_DECODE=$v rc=$?"; tail -8 gpurun_out/da_prof_$v.log
done
unset PIC_NO_ATTN_DECODE
