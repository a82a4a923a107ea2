O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "chain or mlp or module or aggregated or decode or masked or config2" 2>&1 | tail -2 > $O/ec2.txt
for a in 1 0; do echo "acttag $a"; PG_CHAIN_ACTTAG=$a EXP_ONLY=mlp timeout 120 python tools/exp_decode.py 4 2048; done >> $O/ec2.txt 2>&1
PG_CHAIN_DBG=1 EXP_ONLY=mlp timeout 120 python tools/exp_decode.py 4 512 >> $O/ec2.txt 2>&1
cat $O/ec2.txt
