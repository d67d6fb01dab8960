timeout 900 python -m pytest tests/test_gpu_link.py tests/test_gpu_fullsize.py -q -x --timeout 800 --timeout_method thread 2>&1 | tail -2
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export PIC_NO_WAVE_FIT=1; else unset PIC_NO_WAVE_FIT; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('nofit=$v', json.loads(sys.stdin.read())['ms_per_step'])"
done
