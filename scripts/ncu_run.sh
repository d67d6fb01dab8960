set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-steps 1 --decode-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-steps 1 --decode-steps 0 > /dev/null 2>&1
# the compile forward issues 31 x 3 + 32 + 31 = 156 GEMM launches; the link GEMMs follow
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 160 -c 4 -o gpurun_out/prof_gemm_r1b $B > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 40 -c 2 -o gpurun_out/prof_attn_r1b $B > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_link -s 0 -c 1 -o gpurun_out/prof_kvlink_r1b $B > gpurun_out/ncu_kvlink.log 2>&1
