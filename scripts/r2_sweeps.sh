#!/bin/bash
# round-2 build: long-context sweep (Fig. 8 analogue) and open-loop serving (Fig. 7 analogue)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2sweep
timeout 1500 python scripts/long_context_sweep.py --kv-share 0,1 --out gpurun_out/r2sweep/long_context.jsonl > gpurun_out/r2sweep/long_context.log 2>&1
tail -3 gpurun_out/r2sweep/long_context.log
timeout 1500 python scripts/serve_sweep.py --kv-share 1 --ccr 0.2,0.8 --out gpurun_out/r2sweep/serve.jsonl > gpurun_out/r2sweep/serve.log 2>&1
tail -3 gpurun_out/r2sweep/serve.log
