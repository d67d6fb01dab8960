#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3b
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3b/smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/s3b/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/s3b/bench_default.json 2> gpurun_out/s3b/bench_default.err
echo "bench rc=$?"; tail -1 gpurun_out/s3b/bench_default.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench', round(d['ms_per_step'],1), round(d['value']), d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['decode']['tpot_ms'], {k:round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()})"
N="ncu --profile-from-start off --clock-control none"
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/s3b/launches.csv python scripts/ncu_link.py --config cfg4 > gpurun_out/s3b/l.log 2>&1
python scripts/launches_summary.py gpurun_out/s3b/launches.csv > gpurun_out/s3b/launches.md 2>&1; head -12 gpurun_out/s3b/launches.md
timeout 900 $N --set full --import-source on -k regex:attn_qp -c 1 -o gpurun_out/s3b/ncu_attn_qp python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/s3b/a.log 2>&1
python scripts/ncu_detail.py gpurun_out/s3b/ncu_attn_qp.ncu-rep > gpurun_out/s3b/ncu_attn_qp.md 2>&1; head -24 gpurun_out/s3b/ncu_attn_qp.md
