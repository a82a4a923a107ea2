O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests -m gpu -x -q -k "prefill or gemm or config5 or masked_forward_bf16" 2>&1 | tail -2
timeout 300 python tools/experiments/exp_gemm.py 2>&1 | tail -7; timeout 300 python tools/experiments/exp_prefill.py 2>&1 | head -1
