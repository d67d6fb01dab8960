timeout 1500 python -m pytest tests/ -m gpu -q -x --timeout 1400 --timeout_method thread 2>&1 | tail -3
for v in 0 1; do
  if [ $v = 1 ]; then export PIC_NO_FUSED_MERGE=1; fi
  for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('nofused=$v', json.loads(sys.stdin.read())['ms_per_step'])"; done
done
