#!/bin/bash
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_DEC_NOSPLIT=1; else unset PIC_DEC_NOSPLIT; fi
  timeout 600 python scripts/decode_profile.py 32 32 > gpurun_out/ds.log 2>&1; echo "nosplit=$v $(head -1 gpurun_out/ds.log)"; grep "attention\|combine" gpurun_out/ds.log
done
done
