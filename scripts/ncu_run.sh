set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_r1_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
# compile issues 125 GEMM launches (31 layers x 3 + 32 QKV) ... skip into the first link step
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -s 97 -c 4 -o gpurun_out/prof_gemm_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 31 -c 2 -o gpurun_out/prof_attn_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_link -s 0 -c 1 -o gpurun_out/prof_kvlink_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu_kvlink.log 2>&1
