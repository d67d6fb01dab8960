for cfg in 0,0 1,0 1,8 1,16 1,24 0,16 0,0; do
  for i in 1 2; do
    r=$(PIC_L2PF=$cfg timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --profile-steps 0 --decode-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "l2pf=$cfg ms=$r"
  done
done
