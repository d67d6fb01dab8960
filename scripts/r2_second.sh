#!/bin/bash
# new parity tests (bench sizes), TP 2/4/8 + cfg5 TP8, sanitizer, link-step ncu at cfg4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
free -g > gpurun_out/r2_host_mem.txt; nproc >> gpurun_out/r2_host_mem.txt
timeout 1500 python -m pytest tests/test_gpu_parity_bench.py -x -q -s > gpurun_out/r2_parity_bench.log 2>&1
tail -3 gpurun_out/r2_parity_bench.log
timeout 1500 python -m pytest tests/test_gpu_tp.py tests/test_gpu_share.py -q -s > gpurun_out/r2_tp.log 2>&1
tail -3 gpurun_out/r2_tp.log
bash scripts/sanitize.sh
N="ncu --profile-from-start off --clock-control none"
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2_launches_cfg4_wave.csv python scripts/ncu_link.py --config cfg4 > gpurun_out/r2_ncu_launch.log 2>&1
timeout 900 $N --set full --import-source on -k regex:attn_tc -c 1 -o gpurun_out/r2_attn_cfg4 python scripts/ncu_link.py --config cfg4 > gpurun_out/r2_ncu_attn.log 2>&1
timeout 900 $N --set full --import-source on -k regex:gemm -c 4 -o gpurun_out/r2_gemm_cfg4 python scripts/ncu_link.py --config cfg4 > gpurun_out/r2_ncu_gemm.log 2>&1
timeout 900 $N --set full --import-source on -k regex:"attn_tc|gemm|kv_link|rmsnorm|scatter|combine" -c 10 -o gpurun_out/r2_cfg2 python scripts/ncu_link.py --config cfg2 > gpurun_out/r2_ncu_cfg2.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2_attn_cfg4.ncu-rep > gpurun_out/r2_attn_cfg4.md 2>&1
python scripts/ncu_summary.py gpurun_out/r2_gemm_cfg4.ncu-rep > gpurun_out/r2_gemm_cfg4.md 2>&1
python scripts/ncu_summary.py gpurun_out/r2_cfg2.ncu-rep > gpurun_out/r2_cfg2.md 2>&1
echo done
