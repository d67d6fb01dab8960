#!/bin/bash
# one-lane attention accounting at a cfg4 batch (copy / Q-side re-base), finer softmax phases; MMA probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out

PIC_ATTN_TRACE=1 timeout 600 python scripts/attn_trace4.py 16 2 ${MODES:-0,3} > gpurun_out/trace4.log 2>&1
echo "trace rc=$?"
grep "softmax cycles\|arrive ->\|per-tile\|^---" gpurun_out/trace4.log | tail -24
