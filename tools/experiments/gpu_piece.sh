# decode chain: weight copies split into smaller bulk copies (PG_CHAIN_PIECE bytes)
O=gpurun_out; mkdir -p $O; : > $O/piece.txt
for p in 0 1024 2048 4096 8192; do
  PG_CHAIN_PIECE=$p EXP_ONLY=o EXP_SHAPE="4096 4096 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py >> $O/piece.txt 2>&1
  PG_CHAIN_PIECE=$p EXP_ONLY=o timeout 120 python tools/experiments/exp_c5_qkvo.py >> $O/piece.txt 2>&1
  PG_CHAIN_PIECE=$p timeout 120 python tools/experiments/exp_c2_step.py >> $O/piece.txt 2>&1
done
cat $O/piece.txt
