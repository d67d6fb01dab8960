#!/bin/bash
# full GPU suite + smoke (round-end rehearsal); logs -> gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/full_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/full_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$? $(tail -1 gpurun_out/smoke.log)"
