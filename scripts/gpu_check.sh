mkdir -p gpurun_out
timeout 900 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_ll32.json 2>gpurun_out/bench_cfg3.err; tail -3 gpurun_out/bench_cfg3.err
timeout 900 python bench.py --config cfg3 --alg cacheblend:15 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_cb15.json 2>gpurun_out/bench_cfg3cb.err; tail -3 gpurun_out/bench_cfg3cb.err
timeout 1200 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2>gpurun_out/bench_cfg4.err; tail -3 gpurun_out/bench_cfg4.err
