#!/bin/bash
# decode (batch 32) link-step GEMM launch list: per-GEMM duration and DRAM bytes (ncu, one decode step)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
DECODE_NCU=1 timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size -c 14 --csv python scripts/decode_profile.py 32 1 > gpurun_out/decgemm.csv 2> gpurun_out/decgemm.err
echo "rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/decgemm.csv')) if len(r) > 10]
hdr=rows[0]; data=rows[1:]
ik=hdr.index('Kernel Name'); im=hdr.index('Metric Name'); iv=hdr.index('Metric Value'); iid=hdr.index('ID')
by={}
for r in data:
    by.setdefault(r[iid], {'k': r[ik][:60]})[r[im]] = r[iv]
for k,v in by.items(): print(k, v)
PY
