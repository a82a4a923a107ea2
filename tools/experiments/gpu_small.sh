O=gpurun_out; mkdir -p $O; : > $O/smemcap.txt
for kb in 227 200 160 100; do
  PG_CHAIN_SMEM_KB=$kb EXP_ONLY=o EXP_SHAPE="256 256 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py | sed "s/^/S$kb /" >> $O/smemcap.txt 2>&1
  PG_CHAIN_SMEM_KB=$kb EXP_ONLY=o EXP_SHAPE="4096 4096 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py | sed "s/^/S$kb /" >> $O/smemcap.txt 2>&1
done
for kb in 227 200; do
  PG_CHAIN_SMEM_KB=$kb timeout 120 python tools/experiments/exp_c2_step.py | sed "s/^/S$kb /" >> $O/smemcap.txt 2>&1
done
cat $O/smemcap.txt
