#!/bin/bash
# one-m-tile (decode / skinny) GEMMs: N-tile + split that keep the most SMs streaming (PIC_SKINNY_FILL=1) vs bn 128
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PIC_SKINNY_FILL=1 timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_decode_attn.py tests/test_gpu_link.py -q -x > gpurun_out/sf_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/sf_tests.log)"
for r in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_SKINNY_FILL=1; else unset PIC_SKINNY_FILL; fi
  timeout 600 python scripts/decode_profile.py 32 32 > gpurun_out/sf.log 2>&1; echo "fill=$v $(head -1 gpurun_out/sf.log) $(grep gemm gpurun_out/sf.log)"
done
done
unset PIC_SKINNY_FILL
