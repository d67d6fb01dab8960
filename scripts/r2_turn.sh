#!/bin/bash
# ping-pong attention with strict softmax turns (default) vs without (libpic_noturn.so): kernel tests,
# cfg4 copy-path bench A/B (the ping-pong kernel's path), PP trace of both
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_share.py -q -x > gpurun_out/turn_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/turn_tests.log)"; grep "^FAILED" gpurun_out/turn_tests.log | head
for L in libpic.so libpic_noturn.so libpic.so libpic_noturn.so; do
  PIC_LIB_NAME=$L timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share 0 > gpurun_out/turn.json 2> gpurun_out/turn.err
  python -c "import json;d=json.loads(open('gpurun_out/turn.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/turn.err
done
for L in libpic.so libpic_noturn.so; do
PIC_LIB_NAME=$L PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share 0 > gpurun_out/pp_trace_$L.log 2>&1
echo "== $L"; tail -24 gpurun_out/pp_trace_$L.log | grep "span\|smA\|smB\|mma wait"
done
