# Round-1 (session 2) evidence: launch list of the default bench (shared-block link) and full captures of
# the shared-block attention kernel (attn_tc_kernel<4,true>, K-tile re-base) and a link-step GEMM.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-steps 1 --decode-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --profile-steps 1 --decode-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 40 -c 2 -o gpurun_out/prof_attn_r1c $B > gpurun_out/ncu_attn_r1c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 160 -c 4 -o gpurun_out/prof_gemm_r1c $B > gpurun_out/ncu_gemm_r1c.log 2>&1
python scripts/launches_summary.py gpurun_out/launches_r1c.csv > gpurun_out/launches_r1c.md 2>&1
python scripts/ncu_summary.py gpurun_out/prof_attn_r1c.ncu-rep > gpurun_out/ncu_attn_r1c.md 2>&1
python scripts/ncu_summary.py gpurun_out/prof_gemm_r1c.ncu-rep > gpurun_out/ncu_gemm_r1c.md 2>&1
