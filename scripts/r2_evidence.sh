#!/bin/bash
# round-2 evidence: default bench line (driver command), ncu launch list of one cfg4 link step (32-request
# wave), ncu --set full of the link step's GEMMs (layer 0) and attention (shared v1, copy v2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 900 python bench.py --steps 10 --warmup 3 ) > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
tail -1 gpurun_out/ev_bench.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench', round(d['ms_per_step'],1), round(d['value']), d['e2e']['value'], d['roofline']['frac'], d['clocks'], d.get('cpu_baseline'))"
tail -4 gpurun_out/ev_bench.err
N="ncu --profile-from-start off --clock-control none"
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/ev_launches.csv python scripts/ncu_link.py --config cfg4 > gpurun_out/ev_l.log 2>&1
python scripts/launches_summary.py gpurun_out/ev_launches.csv > gpurun_out/ev_launches.md 2>&1; head -14 gpurun_out/ev_launches.md
timeout 900 $N --set full --import-source on -k regex:gemm -c 4 -o gpurun_out/ev_gemm python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/ev_g.log 2>&1
timeout 900 $N --set full --import-source on -k regex:attn -c 1 -o gpurun_out/ev_attn_shared python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/ev_a.log 2>&1
timeout 900 $N --set full --import-source on -k regex:attn -c 1 -o gpurun_out/ev_attn_copy python scripts/ncu_link.py --config cfg4 --layers 2 --kv-share 0 > gpurun_out/ev_a2.log 2>&1
for f in ev_gemm ev_attn_shared ev_attn_copy; do python scripts/ncu_detail.py gpurun_out/$f.ncu-rep > gpurun_out/$f.md 2>&1; done
grep -h "^## \|time_duration\|dram__bytes\|tensor_cycles" gpurun_out/ev_gemm.md gpurun_out/ev_attn_*.md
