# decode-chain experiment: gpu tests, MLP step timing, per-phase stamps
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > $O/ec.txt
timeout 120 python tools/exp_decode.py 4 2048 >> $O/ec.txt 2>&1
for m in 1 3; do echo "mode $m" >> $O/ec.txt; PG_CHAIN_MODE=$m EXP_ONLY=mlp timeout 120 python tools/exp_decode.py 4 1024 >> $O/ec.txt 2>&1; done
PG_CHAIN_DBG=1 EXP_ONLY=mlp timeout 120 python tools/exp_decode.py 4 512 >> $O/ec.txt 2>&1
cat $O/ec.txt
