#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/decode_profile.py 32 8 > gpurun_out/dec_prof.log 2>&1; echo "rc=$?"; tail -14 gpurun_out/dec_prof.log
timeout 900 ncu --profile-from-start on --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:attn -c 2 --csv python scripts/decode_profile.py 32 1 > gpurun_out/dec_ncu.csv 2>&1; grep -o '"attn[^"]*"\|"dram__bytes_read.sum","[A-Za-z]*","[0-9.,]*"\|"gpu__time_duration.sum","[a-z]*","[0-9.,]*"\|"[0-9]*, [0-9]*, [0-9]*"' gpurun_out/dec_ncu.csv | tail -12
