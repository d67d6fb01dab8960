PIC_GEMM_CPS=2 timeout 900 python -m pytest tests/test_gpu_link.py tests/test_gpu_fullsize.py -q -x --timeout 800 --timeout_method thread 2>&1 | tail -2
for c in 1 2; do
  for cfg in cfg2 cfg3 cfg4; do
    st=20; [ $cfg = cfg4 ] && st=3
    PIC_GEMM_CPS=$c timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('cps=$c $cfg', json.loads(sys.stdin.read())['ms_per_step'])"
  done
done
