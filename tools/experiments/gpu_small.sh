O=gpurun_out; mkdir -p $O; : > $O/s1unroll.txt
for i in 1 2 3; do
for v in "" u8 u6; do
  PG_LIB_VARIANT=$v timeout 120 python tools/experiments/exp_c2_step.py | sed "s/^/V=$v /" >> $O/s1unroll.txt 2>&1
done
done
PG_LIB_VARIANT=u8 timeout 600 python -m pytest tests -m gpu -x -q -k "mlp or chain or module" 2>&1 | tail -1 >> $O/s1unroll.txt
cat $O/s1unroll.txt
