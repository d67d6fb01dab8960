#!/bin/bash
# one-lane attention softmax: exponential split (PIC_V1_POLY8 = 0..3 pairs of 8 on the FMA polynomial), cfg4 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_share.py -x -q -k "attention or chunkframe or shared" > gpurun_out/p1_t.log 2>&1; echo "tests: $(tail -1 gpurun_out/p1_t.log)"
PIC_LIB_NAME=libpic_ph.so PIC_ATTN_TRACE=1 timeout 600 python scripts/attn_trace4.py 16 2 0,3 > gpurun_out/trace4_ph.log 2>&1
grep "softmax cycles\|^---" gpurun_out/trace4_ph.log | tail -4
for r in 1 2; do
for lib in libpic.so libpic_p0.so libpic_p2.so libpic_p3.so; do
  PIC_LIB_NAME=$lib timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/p1.json 2> gpurun_out/p1.err
  python -c "import json;d=json.loads(open('gpurun_out/p1.json').read().strip().splitlines()[-1]);print('$lib', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/p1.err
done
done
