set -x
mkdir -p gpurun_out
# compile issues 125 GEMM + 31 attention launches before the first link step
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 125 -c 4 -o gpurun_out/prof_gemm_link_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 31 -c 2 -o gpurun_out/prof_attn_link_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_attn.log 2>&1
timeout 900 python -m pytest tests/test_gpu_link.py -q -x --timeout 800 --timeout_method thread -k full_width 2>&1 | tail -20
