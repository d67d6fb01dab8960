#!/bin/bash
# reference arm (the fp64 oracle on the host cores, bench.py --impl reference) as the driver launches it,
# with its wall clock, then the default bench line again on the same box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3h
( time timeout 900 python bench.py --impl reference ) > gpurun_out/s3h/ref_default.json 2> gpurun_out/s3h/ref_default.err
echo "ref rc=$?"; tail -1 gpurun_out/s3h/ref_default.json | cut -c1-900; tail -3 gpurun_out/s3h/ref_default.err
( time timeout 900 python bench.py ) > gpurun_out/s3h/bench_repeat.json 2> gpurun_out/s3h/bench_repeat.err
echo "bench rc=$?"; tail -1 gpurun_out/s3h/bench_repeat.json | cut -c1-400; tail -3 gpurun_out/s3h/bench_repeat.err
