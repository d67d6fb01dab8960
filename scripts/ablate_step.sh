# in-graph cost of each kernel class: step time with that class skipped (results invalid)
mkdir -p gpurun_out
for m in ${MASKS:-0 1 2 4 8 16 32 64 12 127}; do
  PIC_ABLATE=$m timeout 300 python bench.py --config ${CFG:-cfg2} --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 > gpurun_out/abl_$m.log 2>&1
  r=$(tail -1 gpurun_out/abl_$m.log | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])" 2>/dev/null)
  echo "ablate=$m ms_per_step=$r"
done
