#!/bin/bash
# batched (one elect.sync per 8 MMAs) vs per-MMA issue in the one-lane attention: kernel tests, trace, cfg4 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_share.py -x -q -k "attention or chunkframe or shared" > gpurun_out/is_t.log 2>&1; echo "tests: $(tail -1 gpurun_out/is_t.log)"
for lib in libpic.so libpic_permma.so; do
  PIC_LIB_NAME=$lib PIC_ATTN_TRACE=1 timeout 600 python scripts/attn_trace4.py 16 2 0,3 > gpurun_out/trace4_$lib.log 2>&1
  echo "$lib"; grep "arrive\|softmax cycles\|^---" gpurun_out/trace4_$lib.log | tail -6
done
for lib in libpic.so libpic_permma.so libpic.so libpic_permma.so; do
  PIC_LIB_NAME=$lib timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/is.json 2> gpurun_out/is.err
  python -c "import json;d=json.loads(open('gpurun_out/is.json').read().strip().splitlines()[-1]);print('$lib', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/is.err
done
