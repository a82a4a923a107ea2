O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > $O/ep.txt
timeout 300 python tools/experiments/exp_prefill.py >> $O/ep.txt 2>&1
timeout 300 python tools/experiments/exp_gemm.py >> $O/ep.txt 2>&1
cat $O/ep.txt
