#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode_attn.py tests/test_gpu_decode.py -q > gpurun_out/dns_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/dns_tests.log)"; grep -B3 -A15 "^E " gpurun_out/dns_tests.log | head -40
for i in 1 2; do timeout 600 python scripts/decode_profile.py 32 32 > gpurun_out/dns.log 2>&1; head -1 gpurun_out/dns.log; grep "attention\|combine" gpurun_out/dns.log; done
