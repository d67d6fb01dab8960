#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_share.py -x -q -k "shared" > gpurun_out/pr_t.log 2>&1; tail -1 gpurun_out/pr_t.log
for dbg in 0 2; do
PIC_ATTN_DEBUG=$dbg PIC_ATTN_PP_ROT=1 PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share 1 > gpurun_out/pr3_$dbg.log 2>&1
echo "== debug $dbg"; grep "attn_pp" gpurun_out/pr3_$dbg.log | tail -21 | grep "span\|compute\|wait S\|wait P\|rot"
done
