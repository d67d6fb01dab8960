#!/bin/bash
# full GPU suite without -x (every failure listed), then smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=10 ${PYTEST_ARGS} > gpurun_out/full_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/full_gpu.log)"
grep "^FAILED\|^ERROR" gpurun_out/full_gpu.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$? $(tail -1 gpurun_out/smoke.log)"
