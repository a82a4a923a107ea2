O=gpurun_out; mkdir -p $O; : > $O/coop.txt
for i in 1 2; do
for c in 1 0; do
  echo "COOP=$c" >> $O/coop.txt
  PG_CHAIN_COOP=$c EXP_ONLY=o EXP_SHAPE="256 256 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py >> $O/coop.txt 2>&1
  PG_CHAIN_COOP=$c EXP_ONLY=o EXP_SHAPE="4096 4096 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py >> $O/coop.txt 2>&1
  PG_CHAIN_COOP=$c EXP_SHAPE="5120 5120 0.4" timeout 120 python tools/experiments/exp_c5_qkvo.py >> $O/coop.txt 2>&1
  PG_CHAIN_COOP=$c timeout 120 python tools/experiments/exp_c2_step.py >> $O/coop.txt 2>&1
done
done
PG_CHAIN_COOP=0 PG_CHAIN_DBG=1 EXP_ONLY=o EXP_SHAPE="256 256 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py 2>&1 | grep stamp >> $O/coop.txt
cat $O/coop.txt
