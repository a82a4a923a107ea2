O=gpurun_out; mkdir -p $O
for ns in 0 20 50 100 200 400; do echo "pollns $ns"; PG_CHAIN_POLLNS=$ns EXP_ONLY=mlp timeout 120 python tools/exp_decode.py 4 2048; done > $O/ec2.txt 2>&1
cat $O/ec2.txt
