# decode-chain experiment: gpu tests (chain), MLP step timing, per-phase stamps
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "chain or mlp or module or aggregated or decode or masked" 2>&1 | tail -2 > $O/ec.txt
timeout 120 python tools/experiments/exp_decode.py 4 2048 >> $O/ec.txt 2>&1
PG_CHAIN_DBG=1 EXP_ONLY=mlp timeout 120 python tools/experiments/exp_decode.py 4 512 >> $O/ec.txt 2>&1
cat $O/ec.txt
