#!/bin/bash
# launch list of the bench command's own timed step (bench.py --ncu-range: cudaProfilerStart/Stop around it),
# the profiling recipe's gpu__time_duration pass; the JSON printed under ncu is not a bench value
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3c
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/s3c/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --decode-steps 0 --ncu-range \
  > gpurun_out/s3c/ncu_bench.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/s3c/ncu_bench.log | cut -c1-300
python scripts/launches_summary.py gpurun_out/s3c/launches_bench.csv > gpurun_out/s3c/launches_bench.md 2>&1; head -14 gpurun_out/s3c/launches_bench.md
