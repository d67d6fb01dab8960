#!/bin/bash
# copy path (no a2 overlap): one-lane vs ping-pong attention, step-time A/B; ncu durations of both kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PIC_NO_K2_OVERLAP=1
for v in 2 1 2 1; do
  if [ $v = 1 ]; then export PIC_ATTN_V1=1; else unset PIC_ATTN_V1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 0 --kv-share 0 > gpurun_out/ab4.json 2> gpurun_out/ab4.err
  python -c "import json;d=json.loads(open('gpurun_out/ab4.json').read().strip().splitlines()[-1]);print('cfg4 copy v$v', round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()}, d['clocks']['sm_mhz'])" || tail -5 gpurun_out/ab4.err
done
unset PIC_ATTN_V1
N="ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
timeout 600 $N -k regex:attn --csv python scripts/ncu_link.py --config cfg4 --layers 4 --kv-share 0 > gpurun_out/ab4_ncu_v2.csv 2>&1
PIC_ATTN_V1=1 timeout 600 $N -k regex:attn --csv python scripts/ncu_link.py --config cfg4 --layers 4 --kv-share 0 > gpurun_out/ab4_ncu_v1.csv 2>&1
grep -h "gpu__time_duration\|tensor" gpurun_out/ab4_ncu_v*.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head -20
