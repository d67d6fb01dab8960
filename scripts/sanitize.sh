#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_link.py (tiny-D128), with and
# without the CTA-pair residual / QKV GEMMs (the pair gate/up GEMM is the default); summaries -> gpurun_out/sanitize_*.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for pair in 0 1; do
    if [ $pair = 1 ]; then export PIC_PAIR_FUSED=1; else unset PIC_PAIR_FUSED; fi
    timeout 1500 $CS --tool $tool --print-limit 50 python scripts/sanitize_link.py \
      > gpurun_out/sanitize_${tool}_pair${pair}.log 2>&1
    echo "$tool pair=$pair rc=$? $(tail -1 gpurun_out/sanitize_${tool}_pair${pair}.log)"
  done
done
