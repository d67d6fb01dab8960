timeout 1200 python -m pytest tests/ -m gpu -q -x --timeout 900 --timeout_method thread 2>&1 | tail -3
for i in 1 2 3; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 2>&1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])"; done
