O=gpurun_out; mkdir -p $O
for i in 1 2; do for z in 0 1; do echo "ztag $z"; PG_CHAIN_ZTAG=$z timeout 120 python tools/exp_decode.py 4 2048; done; done > $O/ec2.txt 2>&1
cat $O/ec2.txt
