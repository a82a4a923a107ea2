O=gpurun_out; mkdir -p $O
for R in 1 4; do echo "R=$R"; PG_CHAIN_DBG=1 EXP_ONLY=mlp timeout 120 python tools/exp_decode.py $R 512; done > $O/ec2.txt 2>&1
cat $O/ec2.txt
