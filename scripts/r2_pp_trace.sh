#!/bin/bash
# ping-pong attention cycle accounting at cfg4 (wave of 32, last layer of a 2-layer link), copy and shared
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for ks in 0 1; do
PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share $ks > gpurun_out/pp_trace_ks$ks.log 2>&1
echo "== kv_share $ks"; tail -24 gpurun_out/pp_trace_ks$ks.log
done
