for d in 0 1; do echo "== PG_UMMA_EPI_DEEP=$d"; PG_UMMA_EPI_DEEP=$d timeout 300 python tools/experiments/exp_gemm.py 2>&1 | tail -8; done
timeout 400 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_routed.py -x -q 2>&1 | tail -2
for d in 0 1; do PG_UMMA_EPI_DEEP=$d timeout 600 python bench.py --steps 5 --warmup 3 --cpu 0 > gpurun_out/pf_$d.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/pf_$d.json')); p=d['prefill']; print('deep=$d prefill ms/layer', p['ms_per_layer'], 'frac', p['roofline']['frac'], 'tok/s', p['tokens_per_s'])"; done
