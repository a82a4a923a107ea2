O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "chain or mlp or module or aggregated or decode or masked or config2" 2>&1 | tail -2 > $O/ec2.txt
for i in 1 2; do for a in 1 0; do echo "slices $a"; PG_CHAIN_SLICES=$a timeout 120 python tools/experiments/exp_decode.py 4 2048; done; done >> $O/ec2.txt 2>&1
cat $O/ec2.txt
