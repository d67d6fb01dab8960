#!/bin/bash
# ping-pong attention iteration: kernel + link parity, cycle trace (cfg4 wave, copy and shared), cfg4 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/it_kern.log 2>&1; tail -2 gpurun_out/it_kern.log
timeout 900 python -m pytest tests/test_gpu_link.py tests/test_gpu_share.py -x -q > gpurun_out/it_link.log 2>&1; tail -2 gpurun_out/it_link.log
for ks in 0 1; do
PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share $ks > gpurun_out/it_trace_ks$ks.log 2>&1
echo "== kv_share $ks"; grep "attn_pp" gpurun_out/it_trace_ks$ks.log | tail -21 | grep -v " 0 (0.0%" 
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
python -c "import json;d=json.loads(open('gpurun_out/it_bench.json').read().strip().splitlines()[-1]);print('cfg4', round(d['ms_per_step'],2), round(d['value']), {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()})" || tail -5 gpurun_out/it_bench.err
