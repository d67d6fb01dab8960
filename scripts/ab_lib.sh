# same-box A/B of two builds (PIC_LIB_NAME): alternate bench runs, 2 rounds
mkdir -p gpurun_out/ab
for r in ${ROUNDS:-1 2}; do
  for L in ${LIBS:-libpic_a5f.so libpic.so}; do
    for C in ${CFGS:-cfg2 cfg3}; do
      PIC_LIB_NAME=$L python bench.py --config $C --decode-steps 0 --no-cpu-baseline --profile-steps 0 > gpurun_out/ab/${L}_${C}_$r.json 2>&1
    done
  done
done
