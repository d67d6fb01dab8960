# tensor-bound evidence: ncu --set full of cfg4 (32-request wave, Llama-3.1-8B shape) link-step GEMMs and attention
set -x
mkdir -p gpurun_out
B="python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --profile-steps 0 --decode-steps 0"
timeout 1200 ncu --set full --clock-control none -k regex:gemm_bf16 -s 600 -c 3 -o gpurun_out/prof_gemm_cfg4_r1c $B > gpurun_out/ncu_gemm_cfg4.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:attn_tc -s 100 -c 1 -o gpurun_out/prof_attn_cfg4_r1c $B > gpurun_out/ncu_attn_cfg4.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_gemm_cfg4_r1c.ncu-rep > gpurun_out/ncu_gemm_cfg4_r1c.md 2>&1
python scripts/ncu_summary.py gpurun_out/prof_attn_cfg4_r1c.ncu-rep > gpurun_out/ncu_attn_cfg4_r1c.md 2>&1
