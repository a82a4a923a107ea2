O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests -m gpu -x -q -k "prefill or gemm or config5 or masked_forward_bf16" 2>&1 | tail -2
for v in 1 0; do echo "PG_UMMA_2CTA=$v"; PG_UMMA_2CTA=$v timeout 300 python tools/exp_gemm.py; PG_UMMA_2CTA=$v timeout 300 python tools/exp_prefill.py | head -1; done 2>&1 | tail -40
