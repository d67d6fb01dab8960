#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode_attn.py tests/test_gpu_decode.py tests/test_gpu_share.py -q -x > gpurun_out/dm_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/dm_tests.log)"; grep -B2 -A12 "^E " gpurun_out/dm_tests.log | head -30
for i in 1 2; do timeout 600 python scripts/decode_profile.py 32 8 > gpurun_out/dm_prof.log 2>&1; echo "rc=$?"; head -9 gpurun_out/dm_prof.log; done
