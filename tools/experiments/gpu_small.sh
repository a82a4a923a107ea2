O=gpurun_out; mkdir -p $O; : > $O/ctaep.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "chain or mlp or module or aggregated or decode or masked or peer or smoke" 2>&1 | tail -2 >> $O/ctaep.txt
for i in 1 2; do
for c in 1 0; do
  PG_CHAIN_CTA_EPOCH=$c EXP_ONLY=o EXP_SHAPE="256 256 0.6" timeout 120 python tools/experiments/exp_c5_qkvo.py | sed "s/^/E$c /" >> $O/ctaep.txt 2>&1
  PG_CHAIN_CTA_EPOCH=$c EXP_SHAPE="5120 5120 0.4" timeout 120 python tools/experiments/exp_c5_qkvo.py | sed "s/^/E$c /" >> $O/ctaep.txt 2>&1
  PG_CHAIN_CTA_EPOCH=$c timeout 120 python tools/experiments/exp_c2_step.py | sed "s/^/E$c /" >> $O/ctaep.txt 2>&1
done
done
cat $O/ctaep.txt
