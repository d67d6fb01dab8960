#!/bin/bash
# session-3 build: long-context sweep (Fig. 8 analogue: copy path vs chunk-frame link, the bench default) and
# open-loop serving (Fig. 7 analogue) with the chunk-frame link
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3sweep
timeout 1500 python scripts/long_context_sweep.py --kv-share 0,3 --out gpurun_out/s3sweep/long_context.jsonl > gpurun_out/s3sweep/long_context.log 2>&1
echo "sweep rc=$?"; tail -12 gpurun_out/s3sweep/long_context.log
timeout 1500 python scripts/serve_sweep.py --kv-share 3 --ccr 0.2,0.8 --out gpurun_out/s3sweep/serve.jsonl > gpurun_out/s3sweep/serve.log 2>&1
echo "serve rc=$?"; tail -14 gpurun_out/s3sweep/serve.log
