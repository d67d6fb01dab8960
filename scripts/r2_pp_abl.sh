#!/bin/bash
# ping-pong attention ablation: softmax skipped (MMA + TMA pipeline alone) vs full, cfg4 copy path, ncu durations
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N="ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for dbg in 0 1; do
PIC_ATTN_DEBUG=$dbg timeout 600 $N -k regex:attn -c 2 --csv python scripts/ncu_link.py --config cfg4 --layers 2 --kv-share 0 > gpurun_out/abl_$dbg.csv 2>&1
echo "== debug $dbg"; grep -h "attn_pp" gpurun_out/abl_$dbg.csv | awk -F'","' '{print $(NF-2), $NF}'
PIC_ATTN_DEBUG=$dbg PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share 0 2>&1 | grep "attn_pp" | tail -21 | grep -v " 0 (0.0%\|steps\|items\|Q-empty\|wait Q\|O-free\|epilogue"
done
