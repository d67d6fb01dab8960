#!/bin/bash
# session-3 evidence on the final build: full GPU suite, smoke, default bench line (driver command),
# ncu launch list of one cfg4 link step (32-request wave), ncu --set full of the link step's QROT attention
# and a GEMM, and of the decode attention kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/s3/full_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/s3/full_gpu.log)"; grep "^FAILED\|^ERROR" gpurun_out/s3/full_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1
echo "smoke rc=$? $(tail -1 gpurun_out/s3/smoke.log)"
( time timeout 900 python bench.py ) > gpurun_out/s3/bench_default.json 2> gpurun_out/s3/bench_default.err
echo "bench rc=$?"; tail -1 gpurun_out/s3/bench_default.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench', round(d['ms_per_step'],1), round(d['value']), d['e2e']['value'], d['roofline'], d['clocks'], d.get('decode'))"
N="ncu --profile-from-start off --clock-control none"
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/s3/launches.csv python scripts/ncu_link.py --config cfg4 > gpurun_out/s3/l.log 2>&1
python scripts/launches_summary.py gpurun_out/s3/launches.csv > gpurun_out/s3/launches.md 2>&1; head -14 gpurun_out/s3/launches.md
timeout 900 $N --set full --import-source on -k regex:attn_tc -c 1 -o gpurun_out/s3/ncu_attn_qrot python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/s3/a.log 2>&1
timeout 900 $N --set full --import-source on -k regex:gemm -c 4 -o gpurun_out/s3/ncu_gemm python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/s3/g.log 2>&1
timeout 900 ncu --clock-control none --set full --import-source on -k regex:attn_decode -s 4 -c 1 -o gpurun_out/s3/ncu_attn_decode python scripts/decode_profile.py 32 1 > gpurun_out/s3/d.log 2>&1
for f in ncu_attn_qrot ncu_gemm ncu_attn_decode; do python scripts/ncu_detail.py gpurun_out/s3/$f.ncu-rep > gpurun_out/s3/$f.md 2>&1; done
grep -h "^## \|time_duration\|dram__bytes\|tensor_cycles" gpurun_out/s3/ncu_*.md
