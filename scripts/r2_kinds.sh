#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_qrot.py tests/test_gpu_decode_attn.py tests/test_gpu_fullsize.py tests/test_gpu_share.py tests/test_gpu_decode.py -q > gpurun_out/kinds_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/kinds_tests.log)"; grep "^FAILED" gpurun_out/kinds_tests.log | head; grep -B3 -A12 "^E " gpurun_out/kinds_tests.log | head -40
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/k.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/k.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])"
