#!/bin/bash
# round-2 first GPU pass: new cfg4 bench (N=1), --gpus 2 self-spawn dry run, GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/r2_smi.txt
( time timeout 600 python bench.py --steps 5 --warmup 3 ) > gpurun_out/r2_bench_n1.log 2>&1
( time timeout 600 python bench.py --gpus 2 --requests 64 --steps 2 --warmup 3 --no-cpu-baseline --decode-steps 0 ) > gpurun_out/r2_bench_n2dry.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1
tail -3 gpurun_out/r2_pytest.log
