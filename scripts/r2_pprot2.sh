#!/bin/bash
# ROT ping-pong: tests; trace with rotation work ablated (debug 2) vs full
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_share.py -x -q -k "attention or shared" > gpurun_out/pr_t.log 2>&1; tail -1 gpurun_out/pr_t.log
for dbg in 2 0; do
PIC_ATTN_DEBUG=$dbg PIC_ATTN_PP_ROT=1 PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share 1 > gpurun_out/pr2_$dbg.log 2>&1
echo "== debug $dbg"; grep "attn_pp" gpurun_out/pr2_$dbg.log | tail -21 | grep -v " 0 (0.0%\|steps\|items\|Q-empty\|wait Q\|O-free\|epilogue\|tiles"
done
