# Round-1 (session 2) bench lines, final build: default bench (cfg2, shared-block link), the copy path,
# cfg3 LegoLink-32 / CacheBlend-15, cfg4 wave, LegoLink-0, cfg5 (70B shape on one GPU), the oracle arm.
mkdir -p gpurun_out/bench_r1c
O=gpurun_out/bench_r1c
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --kv-share 0 --decode-steps 0 > $O/bench_cfg2_copy.json 2> $O/bench_cfg2_copy.err
python bench.py --config cfg3 --decode-steps 0 > $O/bench_cfg3_ll32.json 2> $O/bench_cfg3_ll32.err
python bench.py --config cfg3 --alg cacheblend:15 --decode-steps 0 > $O/bench_cfg3_cb15.json 2> $O/bench_cfg3_cb15.err
python bench.py --config cfg4 --steps 10 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python bench.py --alg legolink0 --decode-steps 0 > $O/bench_cfg2_legolink0.json 2> $O/bench_cfg2_legolink0.err
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --decode-steps 0 --no-cpu-baseline > $O/bench_cfg5_1gpu.json 2> $O/bench_cfg5_1gpu.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
