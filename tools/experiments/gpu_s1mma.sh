# decode chain: stage-1 row dots on the tensor pipe (PG_CHAIN_S1MMA=1) vs FFMA2: interleaved timing
O=gpurun_out; mkdir -p $O; : > $O/s1mma_t.txt
for i in 1 2 3 4; do
  for v in 0 1; do
    PG_CHAIN_S1MMA=$v timeout 120 python tools/experiments/exp_c2_step.py >> $O/s1mma_t.txt 2>&1
  done
done
cat $O/s1mma_t.txt
