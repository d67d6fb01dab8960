#!/bin/bash
# round-end rehearsal on the current HEAD: full GPU suite, smoke, default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/full_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/full_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$? $(tail -1 gpurun_out/smoke.log)"
( time timeout 900 python bench.py ) > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"; tail -1 gpurun_out/bench_default.json | cut -c1-1500; tail -3 gpurun_out/bench_default.err
