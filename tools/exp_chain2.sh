O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "chain or mlp or module or aggregated or decode or masked" 2>&1 | tail -2 > $O/ec2.txt
for a in 0 4 8 16; do echo "l2ahead $a"; PG_CHAIN_L2AHEAD=$a timeout 120 python tools/exp_decode.py 4 2048; done >> $O/ec2.txt 2>&1
cat $O/ec2.txt
