for m in ${MASKS:-0 47 16 14 2 32}; do
  r=$(PIC_ABLATE=$m timeout 300 python bench.py --config ${CFG:-cfg2} --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "ablate=$m ms_per_step=$r"
done
