timeout 1500 python -m pytest tests/ -m gpu -q -x --timeout 1400 --timeout_method thread 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('cfg2', json.loads(sys.stdin.read())['ms_per_step'])"; done
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>&1 | tail -1 | python -c "import json,sys; print('cfg4', json.loads(sys.stdin.read())['ms_per_step'])"
