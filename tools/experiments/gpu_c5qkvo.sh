O=gpurun_out; mkdir -p $O; : > $O/c5sweep.txt
for sh in "4096 4096 0.6" "5120 5120 0.4"; do
  for env in "X=0" "EXP_R=1" "PG_CHAIN_L2HINT=0" "PG_CHAIN_STAGES=4" "PG_CHAIN_STAGES=6" "PG_CHAIN_GRID=132" "PG_CHAIN_GRID=144" "PG_CHAIN_CHUNK_DIV=4"; do
    echo "$env" >> $O/c5sweep.txt
    env $env EXP_ONLY=o EXP_SHAPE="$sh" timeout 120 python tools/experiments/exp_c5_qkvo.py >> $O/c5sweep.txt 2>&1
  done
done
cat $O/c5sweep.txt
