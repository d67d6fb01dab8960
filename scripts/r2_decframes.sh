#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode_attn.py tests/test_gpu_decode.py tests/test_gpu_share.py -q > gpurun_out/df_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/df_tests.log)"; grep "^FAILED" gpurun_out/df_tests.log | head; grep -m2 -B3 -A15 "^E " gpurun_out/df_tests.log | head -40
