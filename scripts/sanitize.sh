#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_link.py (tiny-D128), with and
# without the CTA-pair GEMM; summaries -> gpurun_out/sanitize_*.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for pair in 0 1; do
    PIC_PAIR=$pair timeout 900 $CS --tool $tool --print-limit 50 python scripts/sanitize_link.py \
      > gpurun_out/sanitize_${tool}_pair${pair}.log 2>&1
    echo "$tool pair=$pair rc=$? $(tail -1 gpurun_out/sanitize_${tool}_pair${pair}.log)"
  done
done
