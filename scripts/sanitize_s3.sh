#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_s3.py: the session-3 kernels
# (persistent chunk-frame attention incl. split pieces, split-KV decode attention) plus the default path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 python scripts/sanitize_s3.py > gpurun_out/sanitize_s3_${tool}.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitize_s3_${tool}.log)"
done
