timeout 1500 python -m pytest tests/test_gpu_link.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py tests/test_gpu_decode.py -q -x --timeout 1400 --timeout_method thread 2>&1 | tail -2
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export PIC_NO_K2_OVERLAP=1; else unset PIC_NO_K2_OVERLAP; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('nooverlap=$v', json.loads(sys.stdin.read())['ms_per_step'])"
done
unset PIC_NO_K2_OVERLAP
timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('cfg3', json.loads(sys.stdin.read())['ms_per_step'])"
