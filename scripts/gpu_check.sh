timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_link.py -q -x --timeout 800 --timeout_method thread 2>&1 | tail -2
for i in 1 2; do
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('cfg3', json.loads(sys.stdin.read())['ms_per_step'])"
PIC_NO_WAVE_FIT=1 timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('cfg3 nofit', json.loads(sys.stdin.read())['ms_per_step'])"
done
