bash scripts/ncu_run.sh
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_ll32.json 2>/dev/null
timeout 600 python bench.py --config cfg3 --alg cacheblend:15 --steps 10 --warmup 3 --no-cpu-baseline --decode-steps 0 > gpurun_out/bench_cfg3_cb15.json 2>/dev/null
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --decode-steps 16 > gpurun_out/bench_cfg4.json 2>/dev/null
timeout 600 python bench.py --alg legolink0 --steps 20 --warmup 5 --no-cpu-baseline --decode-steps 0 > gpurun_out/bench_cfg2_legolink0.json 2>/dev/null
ls -la gpurun_out/*.json
