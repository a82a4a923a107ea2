O=gpurun_out; mkdir -p $O; : > $O/mbar.txt
for i in 1 2; do
for v in "" poll hint; do
  echo "variant=$v" >> $O/mbar.txt
  PG_LIB_VARIANT=$v EXP_ONLY=o EXP_SHAPE="256 256 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py >> $O/mbar.txt 2>&1
  PG_LIB_VARIANT=$v EXP_ONLY=o EXP_SHAPE="4096 4096 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py >> $O/mbar.txt 2>&1
  PG_LIB_VARIANT=$v timeout 120 python tools/experiments/exp_c2_step.py >> $O/mbar.txt 2>&1
done
done
cat $O/mbar.txt
